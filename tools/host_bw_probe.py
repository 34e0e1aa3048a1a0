import time, torch, numpy as np
n = 43_200_000 // 8
a = np.random.rand(n)
d = torch.empty(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for name, src in (("pageable", torch.from_numpy(a)), ("pinned", torch.from_numpy(a).pin_memory())):
    for _ in range(2):
        t = time.perf_counter(); d.copy_(src); torch.cuda.synchronize(); h2d = time.perf_counter() - t
        t = time.perf_counter(); src.copy_(d); torch.cuda.synchronize(); d2h = time.perf_counter() - t
    print(name, "H2D ms", round(h2d*1e3, 2), "D2H ms", round(d2h*1e3, 2))
t = time.perf_counter(); b = a.copy(); print("host memcpy ms", round((time.perf_counter()-t)*1e3, 2))
t = time.perf_counter(); p = torch.empty(n, dtype=torch.float64).pin_memory(); print("pin alloc ms", round((time.perf_counter()-t)*1e3, 2))
