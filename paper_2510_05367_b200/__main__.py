"""Command line of the reference (proj/tools/main.cpp) on the GPU engine:

    python -m paper_2510_05367_b200 [--config FILE] [--set key=value ...] [--out DIR]
        {run, compare, ablate, sweep-n [--n 1,2,4], export-plots [--n ...]}

Same subcommands, artifacts and exit codes: 0 ok, 1 error (ShapeError and
anything else), 2 ConfigError, 3 BudgetError, 4 InvariantError
(proj/tools/main.cpp:157-169).
"""
import argparse
import os
import sys

from . import BudgetError, ConfigError, Context, InvariantError, parse_config
from . import harness as H


def _n_list(s: str):
    ns = [int(x) for x in s.split(",") if x.strip()]
    if not ns:
        raise ConfigError("--n expects a comma-separated list such as 1,2,4")
    return ns


def _write(path: str, text: str):
    with open(path, "w") as f:
        f.write(text + "\n")


def _print_peaks(rep: dict):
    print(f"{'stage':<8s} {'fast peak (B)':>14s} {'slow peak (B)':>14s}")
    for s in H.STAGES:
        print(f"{s:<8s} {rep['peaks'][s]['fast']:>14d} {rep['peaks'][s]['slow']:>14d}")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2510_05367_b200",
                                 description="Staged latent-diffusion inference engine with feature caching, tier "
                                             "swapping, spatial chunking and sliced decoding (B200)")
    ap.add_argument("--config", default="", help="Key-value config file")
    ap.add_argument("--set", action="append", default=[], help="Override config keys (key=value, repeatable)")
    ap.add_argument("--out", default="", help="Output directory (overrides run.out_dir)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    sub.add_parser("run", help="Execute one pipeline run and write artifacts")
    sub.add_parser("compare", help="Run the cache-off baseline and this config, compare")
    sub.add_parser("ablate", help="Run {all-on, -swap, -slice, -chunk, cache-only}")
    for name in ("sweep-n", "export-plots"):
        p = sub.add_parser(name)
        p.add_argument("--n", default="1,2,3,4,8", help="Comma-separated N values")
    args = ap.parse_args(argv)
    try:
        text = H.build_config(args.config or None, args.set, args.out or None)
        out_dir = parse_config(text)["run.out_dir"]
        ns = _n_list(args.n) if args.cmd in ("sweep-n", "export-plots") else []
        if args.cmd == "sweep-n" and any(ns[i] <= ns[i - 1] for i in range(1, len(ns))):
            raise ConfigError("sweep-n: N values must be ascending")
        ctx = Context(0)
        try:
            if args.cmd == "run":
                res = H.run_pipeline(ctx, text, repeats=1)
                H.write_run_artifacts(ctx, res, out_dir)
                w, m = res.wall, res.rep["mac"]
                print(f"run complete: {res.video.shape[1]} frames, device {w['total']:.3f}s "
                      f"(denoise {w['denoise']:.3f}s, decode {w['decode']:.3f}s)")
                print(f"denoiser MACs {m['denoiser_total']} ({m['full_steps']} full + {m['cached_steps']} cached steps)")
                _print_peaks(res.rep)
                print(f"artifacts written to {out_dir}")
            elif args.cmd == "compare":
                row = H.compare(ctx, H.baseline_text(text), text)
                os.makedirs(out_dir, exist_ok=True)
                _write(os.path.join(out_dir, "compare.json"), H.dumps(row))
                print(f"{'speed_up':<10s} {'psnr':<8s} {'ssim':<8s} {'identical':<10s}")
                print(f"{row['speed_up']:<10.3f} {row['psnr_mean']:<8.3f} {row['ssim_mean']:<8.4f} "
                      f"{'yes' if row['identical_video'] else 'no':<10s}")
                print(f"wrote {out_dir}/compare.json")
            elif args.cmd == "ablate":
                rows = H.ablate(ctx, text)
                os.makedirs(out_dir, exist_ok=True)
                _write(os.path.join(out_dir, "ablate.json"), H.dumps(rows))
                print(f"{'row':<12s} {'time(s)':<8s} {'psnr':<8s} {'ssim':<8s} {'encode(B)':>12s} "
                      f"{'denoise(B)':>12s} {'decode(B)':>12s}")
                for r in rows:
                    pf = r["peak_fast"]
                    print(f"{r['label']:<12s} {r['wall_total']:<8.3f} {r['psnr_mean']:<8.3f} {r['ssim_mean']:<8.4f} "
                          f"{pf['encode']:>12d} {pf['denoise']:>12d} {pf['decode']:>12d}")
                print(f"wrote {out_dir}/ablate.json")
            elif args.cmd == "sweep-n":
                table = H.sweep_n(ctx, text, ns)
                os.makedirs(out_dir, exist_ok=True)
                _write(os.path.join(out_dir, "sweep.json"), H.dumps(table))
                print(f"{'N':<4s} {'speed_up':<10s} {'psnr':<8s} {'ssim':<8s} {'macs':>14s}")
                for r in table["rows"]:
                    print(f"{r['n']:<4d} {r['speed_up']:<10.3f} {r['psnr_mean']:<8.3f} {r['ssim_mean']:<8.4f} "
                          f"{r['macs']:>14d}")
                if not table["quality_monotone"]:
                    print("note: quality trend is not monotone over the requested Ns")
                print(f"wrote {out_dir}/sweep.json")
            elif args.cmd == "export-plots":
                for path in H.export_plots(ctx, text, ns, out_dir):
                    print(f"wrote {path}")
        finally:
            ctx.close()
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2
    except BudgetError as e:
        print(f"budget abort: {e}", file=sys.stderr)
        return 3
    except InvariantError as e:
        print(f"invariant failure: {e}", file=sys.stderr)
        return 4
    except Exception as e:  # noqa: BLE001 -- the reference maps every other exception to 1
        print(f"error: {e}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
