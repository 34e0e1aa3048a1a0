"""Time the device bin_scatter on HBM-resident points (CUDA events on the
context stream) and report algorithmic GB/s (8*d bytes per point read + the
count array written once) against the measured HBM peak.

    python tools/time_bin_scatter.py [--npts 100000000] [--reps 10]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_03298_b200 import kronglm as K  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--npts", type=int, default=100_000_000)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--cases", default="", help="comma-separated case names (default: all)")
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    ctx = K.default_context()
    stream = torch.cuda.ExternalStream(ctx.stream)
    g = torch.Generator(device="cuda").manual_seed(1)
    cases = [("d3_c2grid_uniform", 3, [100, 100, 120], "uniform"),
             ("d3_c1grid_uniform", 3, [40, 40, 40], "uniform"),
             ("d2_64x64_uniform", 2, [64, 64], "uniform"),
             ("d2_64x64_gauss", 2, [64, 64], "gauss"),
             ("d3_c5grid_uniform", 3, [977, 25, 25], "uniform"),
             ("d2_16x16_gauss", 2, [16, 16], "gauss")]
    keep = set(a.cases.split(",")) if a.cases else None
    for name, d, bins, dist in cases:
        if keep and name not in keep:
            continue
        if dist == "uniform":
            pts = torch.rand((a.npts, d), generator=g, device="cuda", dtype=torch.float64)
        else:
            pts = (torch.randn((a.npts, d), generator=g, device="cuda", dtype=torch.float64) * 0.1 + 0.5)
        cells = int(np.prod(bins))
        out = torch.empty(cells, device="cuda", dtype=torch.float64)
        bounds = [(0.0, 1.0)] * d
        for _ in range(a.warmup):
            K.bin_scatter(pts, bounds, bins, out=out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ms = []
        for _ in range(a.reps):
            e0.record(stream)
            r = K.bin_scatter(pts, bounds, bins, out=out)
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        med = float(np.median(ms))
        byts = 8.0 * d * a.npts + 8.0 * cells
        print(json.dumps({"case": name, "npts": a.npts, "cells": cells, "ms": round(med, 4),
                          "gbs": round(byts / med / 1e6, 1), "gpts_s": round(a.npts / med / 1e6, 2),
                          "dropped": r.dropped}))
        del pts, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
