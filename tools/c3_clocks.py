"""C3 pass-1 launches back to back for a few seconds with nvidia-smi sampling
clocks, power and throttle reasons (is launch-to-launch variance clocks?)."""
import os
import subprocess
import sys
import tempfile
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_07642_b200 as frr  # noqa: E402
from paper_2501_07642_b200 import generation as G  # noqa: E402

X = np.random.default_rng(3).standard_normal((2000, 1024))
design = frr.DesignSpec(2000, 1000, accept_prob=1e-4, max_draws=10**8, batch_size=10_000, root_seed=43,
                        precision_mode="ridge")
kern = frr.precompute_precision(X, "ridge")._kernel
M = 1 << 20
out = torch.empty(M, dtype=torch.float64, device="cuda")
G.mc_stats_device(kern, design, 0, M, out)
torch.cuda.synchronize()
log = tempfile.TemporaryFile(mode="w+")
q = "clocks.sm,power.draw,temperature.gpu,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown"
p = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "100"],
                     stdout=log, stderr=subprocess.DEVNULL, text=True)
rates = []
t_end = time.time() + 6
while time.time() < t_end:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    G.mc_stats_device(kern, design, 0, M, out)
    e1.record()
    torch.cuda.synchronize()
    rates.append(M / e0.elapsed_time(e1) * 1e3)
p.terminate()
p.wait()
log.seek(0)
lines = [l.strip() for l in log if l.strip()]
print("launches", len(rates), "rate min/med/max %.3e %.3e %.3e" % (min(rates), sorted(rates)[len(rates) // 2], max(rates)))
print("rates:", " ".join(f"{r / 1e6:.0f}" for r in rates[:60]))
from collections import Counter
print(Counter(lines).most_common(12))
