"""One warm resident pipeline step of a bench workload (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2510_05367_b200 as lc
wl = sys.argv[1] if len(sys.argv) > 1 else "B"
over = bench.WORKLOADS[wl]
text = lc.config_text(over, base=lc.DEFAULT_CONFIG)
ctx = lc.Context(0)
ctx.configure(text)
T = int(over.get("run.frames", 8))
ctx.set_decode_slice(2 if wl == "A" else max(d for d in range(1, 6) if T % d == 0))  # bench.py's default
kv = lc.parse_config(text)
n = ctx.latent_elems()
lat = lc.randn(lc.derive_seed(int(kv["run.seed"]), 1), n)
if wl == "D":  # the sliced decode alone (one lc_decode_sharded per run, world 1)
    s = 1 << int(kv["codec.stages"])
    lat = lat.reshape(1, T, 4, int(kv["run.height"]) // s, int(kv["run.width"]) // s)
    for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
        _, ms = ctx.decode_sharded(lat, 5)
    print("launches/decode", ctx.kernel_launches(), "device ms", ms)
    sys.exit(0)
ctx.upload_latent(lat)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    rep = ctx.run_resident()
print("launches/step", rep["kernel_launches"], "device ms", rep["device_ms"])
