import time, json, numpy as np, sys
sys.path.insert(0, ".")
import paper_2510_05367_b200 as lc
B = {"run.frames":16,"run.height":512,"run.width":512,"codec.stages":3,"codec.width":128,"unet.base_channels":320,"unet.depth":3,"sampler.steps":4,"cache.n":2}
C = {"run.frames":25,"run.height":576,"run.width":1024,"codec.stages":3,"codec.width":128,"unet.base_channels":320,"unet.depth":3,"sampler.steps":25,"cache.n":2,"swap.mode":"async"}
ctx = lc.Context(0)
for name, over in [("B", B), ("C", C)]:
    t=time.time(); ctx.configure(lc.config_text(over, base=lc.DEFAULT_CONFIG)); print(name, "configure s", time.time()-t, flush=True)
    for i in range(3):
        t=time.time(); v, lat, rep = ctx.run_pipeline(); w=time.time()-t
        print(name, f"wall {w*1000:.1f} ms", json.dumps({k: rep[k] for k in ["device_ms","hbm_peak_bytes","cache_bytes","cache_bytes_physical","swap","kernel_launches"]}), rep["timeline"]["stall_ms"], flush=True)
    T=over["run.frames"]; print(name, "fps", T/(rep["device_ms"]["total"]/1000), "finite", np.isfinite(v).all(), float(np.abs(v).mean()))
