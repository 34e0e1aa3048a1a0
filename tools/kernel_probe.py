"""Times the hot kernels and their debug variants on one config (CUDA events)."""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_03298_b200 import _lib, configs  # noqa: E402
from paper_1510_03298_b200 import kronglm as K  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--which", default="2,3,4,0,1")
args = ap.parse_args()
d = configs.make(args.config)
ctx = K.Context(0)
D = K.Design(d["design"], ctx)
O = K.Observation(D, d["y"])
names = {0: "fused full", 1: "largest H contraction", 2: "stream read v,z", 3: "fused copies only",
         4: "fused copies + phase A"}
for w in [int(x) for x in args.which.split(",")]:
    ms, b = C.c_double(), C.c_double()
    ctx.check(_lib.load().kg_time_kernel(ctx.h, D.h, O.h, w, 50, C.byref(ms), C.byref(b)))
    print(f"{args.config} {names[w]:26s} {ms.value * 1000:9.2f} us  {b.value / 1e6:8.1f} MB  "
          f"{b.value / ms.value / 1e6:8.1f} GB/s", flush=True)
