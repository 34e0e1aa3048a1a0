"""kg_time_kernel on one config: which = 0 fused n-space pass, 1 largest banded
contraction, 2 stream-read reference; prints ms and GB/s."""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_03298_b200 import _lib, configs  # noqa: E402
from paper_1510_03298_b200 import kronglm as K  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--which", type=int, nargs="+", default=[0, 1, 2])
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
d = configs.make(args.config)
ctx = K.Context(0)
D = K.Design(d["design"], ctx)
O = K.Observation(D, d["y"])
for w in args.which:
    ms, b = C.c_double(), C.c_double()
    ctx.check(_lib.load().kg_time_kernel(ctx.h, D.h, O.h, w, args.reps, C.byref(ms), C.byref(b)))
    print(f"{args.config} which={w}: {ms.value * 1000:.1f} us, {b.value / 1e6:.1f} MB, "
          f"{b.value / (ms.value / 1000) / 1e9:.0f} GB/s", flush=True)
