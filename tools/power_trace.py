"""Spectral-radius power iterations per factor (KG_POWER_TRACE=1) and the
design-creation wall time for each config."""
import os
import sys
import time

os.environ.setdefault("KG_DEV", "1")
os.environ.setdefault("KG_POWER_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_03298_b200 import configs  # noqa: E402
from paper_1510_03298_b200 import kronglm as K  # noqa: E402

for cfg in sys.argv[1:] or ["C2"]:
    d = configs.make(cfg)
    for rep in range(2):
        t0 = time.perf_counter()
        D = K.Design(d["design"])
        print(f"{cfg} rep {rep}: design {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
        D.close()
