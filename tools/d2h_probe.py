import time, numpy as np, torch
from concurrent.futures import ThreadPoolExecutor
ex = ThreadPoolExecutor(8)
t = torch.randint(0, 2, (2333606, 34), dtype=torch.int8, device="cuda")
stage = torch.empty(t.numel(), dtype=torch.int8, pin_memory=True)
def a():
    return t.cpu().numpy()
def b(nt):
    stage.copy_(t.reshape(-1), non_blocking=True); torch.cuda.synchronize()
    out = np.empty(t.shape, np.int8); fo = out.reshape(-1); s = stage.numpy()
    n = fo.size; step = (n + nt - 1) // nt
    if nt == 1:
        np.copyto(fo, s)
    else:
        list(ex.map(lambda i: np.copyto(fo[i:i+step], s[i:i+step]), range(0, n, step)))
    return out
def c():
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True); h.copy_(t, non_blocking=True); torch.cuda.synchronize(); return h.numpy()
for name, f in [("pageable", a), ("stage1", lambda: b(1)), ("stage4", lambda: b(4)), ("stage8", lambda: b(8)), ("pinned_fresh", c)]:
    f(); torch.cuda.synchronize()
    ts = []
    keep = []
    for _ in range(5):
        t0 = time.perf_counter(); r = f(); ts.append(time.perf_counter() - t0); keep.append(r)
    print(name, " ".join(f"{x*1e3:.1f}" for x in ts))
