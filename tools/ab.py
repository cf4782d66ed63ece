"""Interleaved A/B timing of libfrr builds inside ONE process (removes the
process-to-process and box-to-box variance of separate runs).

    python tools/ab.py c2|c3 M lib1.so lib2.so ...

Every library gets the same device buffers (prepared by the default build)
and the same stream; launches alternate lib1, lib2, ... for R rounds; the
output of each build is compared bit-for-bit with the default build's.
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_07642_b200 as frr  # noqa: E402
from paper_2501_07642_b200 import _native as N  # noqa: E402
from paper_2501_07642_b200 import generation as G  # noqa: E402

shape, M, libs = sys.argv[1], int(sys.argv[2]), sys.argv[3:]
R = int(os.environ.get("AB_ROUNDS", "7"))
if shape == "c2":
    X = np.random.default_rng(2).standard_normal((1000, 64))
    design = frr.DesignSpec(1000, 500, accept_prob=1e-3, max_draws=M, batch_size=10_000, root_seed=42)
    kern = frr.precompute_precision(X, "exact")._kernel
else:
    X = np.random.default_rng(3).standard_normal((2000, 1024))
    design = frr.DesignSpec(2000, 1000, accept_prob=1e-4, max_draws=M, batch_size=10_000, root_seed=43,
                            precision_mode="ridge")
    kern = frr.precompute_precision(X, "ridge")._kernel
os.environ["FRR_MC_PATH"] = "tensor_core"
want = G.mc_stats_device(kern, design, 0, M).cpu().numpy()
s, keep = kern.device_struct(design.n_treated, limbs=True)
stream = torch.cuda.current_stream()
out = torch.empty(M, dtype=torch.float64, device="cuda")
handles = []
for p in libs:
    L = ctypes.CDLL(os.path.abspath(p), mode=ctypes.RTLD_LOCAL)
    f = L.frr_mc_stats_tc
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.POINTER(N.Balance), ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p,
                  ctypes.c_void_p]
    L.frr_last_error.restype = ctypes.c_char_p
    f.last_error = L.frr_last_error
    f.lib = p
    handles.append(f)


def launch(f):
    rc = f(ctypes.byref(s), design.root_seed, 0, M, ctypes.c_void_p(out.data_ptr()),
           ctypes.c_void_p(stream.cuda_stream))
    if rc:
        raise RuntimeError(f"{f.lib}: rc={rc}: {f.last_error().decode()}")


bad = []
for f in handles:
    out.zero_()
    launch(f)
    torch.cuda.synchronize()
    bad.append(int((out.cpu().numpy().view(np.uint64) != want.view(np.uint64)).sum()))
# warm-up: the first ~1-2 s of back-to-back tensor-heavy launches on a fresh
# box are erratic (power ramp); launch the first build until AB_WARM seconds pass
import time  # noqa: E402

t_warm = time.time() + float(os.environ.get("AB_WARM", "5"))
while time.time() < t_warm:
    launch(handles[0])
    torch.cuda.synchronize()
times = [[] for _ in handles]
for _ in range(R):
    for i, f in enumerate(handles):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        launch(f)
        e1.record(stream)
        torch.cuda.synchronize()
        times[i].append(e0.elapsed_time(e1))
if os.environ.get("AB_VERBOSE"):
    for p, t in zip(libs, times):
        print(os.path.basename(p), " ".join(f"{M / x * 1e3 / 1e6:.0f}" for x in t))
for p, t, b in zip(libs, times, bad):
    t = sorted(t)
    print(f"{os.path.basename(p):28s} mismatches={b:<8d} median={M / t[len(t) // 2] * 1e3:.3e} "
          f"best={M / t[0] * 1e3:.3e} worst={M / t[-1] * 1e3:.3e} cand/s", flush=True)
