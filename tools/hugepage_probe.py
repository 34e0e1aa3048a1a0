"""Host-side cost of writing a fresh 43 MB result array: 4 KB pages vs
transparent huge pages (MADV_HUGEPAGE), and the DMA into it."""
import mmap
import time

import numpy as np
import torch

for f in ("enabled", "defrag"):
    try:
        print(f, open(f"/sys/kernel/mm/transparent_hugepage/{f}").read().strip())
    except OSError as e:
        print(f, "unreadable", e)
n = 43_200_000 // 8
d = torch.rand(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()


def huge(nbytes):
    m = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    m.madvise(mmap.MADV_HUGEPAGE)
    return np.frombuffer(m, dtype=np.float64)


for rep in range(3):
    for name, alloc in (("np.zeros", lambda: np.zeros(n)), ("np.empty", lambda: np.empty(n)),
                        ("mmap+THP", lambda: huge(n * 8))):
        t0 = time.perf_counter()
        a = alloc()
        t1 = time.perf_counter()
        torch.from_numpy(a).copy_(d)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"rep {rep} {name}: alloc {1e3 * (t1 - t0):.2f} ms, D2H into it {1e3 * (t2 - t1):.2f} ms")
