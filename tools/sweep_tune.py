"""Variant sweep of the sweep kernel on one GPU (LDC, device-timed, graphs on).

    python tools/sweep_tune.py [--n 256] [--steps 100] [--variants 0-7] [--aligns 128]

Prints one line per (precision, variant, align): MFLUPS and algorithmic GB/s
(2*19*sizeof(real) bytes per fluid cell update).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def parse_list(s):
    out = []
    for part in s.split(","):
        if "-" in part:
            a, b = part.split("-")
            out += list(range(int(a), int(b) + 1))
        else:
            out.append(int(part))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--patch", type=int, default=0)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--variants", default="0-7")
    ap.add_argument("--aligns", default="128")
    ap.add_argument("--precisions", default="8,4")
    ap.add_argument("--impls", default="tma,simt")
    ap.add_argument("--shapes", default="0-2")
    ap.add_argument("--layout", type=int, default=0)
    args = ap.parse_args()
    import torch
    from paper_1007_1388_b200 import inputs, lbm
    n = (args.n,) * 3
    patch = (args.patch,) * 3 if args.patch else n
    fl, wu = inputs.ldc_flags(n)
    results = []
    combos = []
    for impl in args.impls.split(","):
        for v in (parse_list(args.variants) if impl == "simt" else parse_list(args.shapes)):
            combos.append((impl, v))
    for prec in parse_list(args.precisions):
        for align in parse_list(args.aligns):
            for impl, v in combos:
                os.environ["LBM_SWEEP_IMPL"] = impl
                os.environ["LBM_SWEEP_VARIANT"] = str(v) if impl == "simt" else "7"
                os.environ["LBM_TMA_SHAPE"] = str(v) if impl == "tma" else "0"
                os.environ["LBM_ALIGN_BYTES"] = str(align)
                L = lbm.Lattice(n, patch, inputs.LDC_OMEGA, prec, device=0, layout=args.layout)
                L.set_flags(fl, wu)
                L.init_noise(1388)
                L.step(10)
                st = torch.cuda.ExternalStream(L.stream())
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(st)
                L.step_async(args.steps)
                e1.record(st)
                L.synchronize()
                ms = e0.elapsed_time(e1) / args.steps
                fluid = L.info()["fluid_cells_global"]
                L.close()
                mfl = fluid / (ms / 1e3) / 1e6
                gbs = mfl * 1e6 * 2 * 19 * prec / 1e9
                r = dict(prec=prec, impl=impl, variant=v, align=align, layout=args.layout, ms=ms, mflups=mfl,
                         alg_gbs=gbs)
                results.append(r)
                print(json.dumps(r), flush=True)
    best = {}
    for r in results:
        if r["prec"] not in best or r["mflups"] > best[r["prec"]]["mflups"]:
            best[r["prec"]] = r
    print("BEST", json.dumps(best))


if __name__ == "__main__":
    main()
