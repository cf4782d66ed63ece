"""Benchmark of the rerandomization hot path (BASELINE.json metric).

Workload (BASELINE.json configs[1], "C2"): Monte Carlo rerandomization,
n=1000 units, 500 treated, d=64 Gaussian covariates, 1e8 candidates per
GPU per step, prob_accept=1e-3.  One step = generate and balance-check
every candidate (fused sm_100a kernel) + exact global acceptance selection
(radix select + compaction; NCCL all-reduce of the histograms for N>1).
The GPU runs the steps strictly one after another; the host keeps up to 4
steps enqueued (each with its own statistics buffer) and reads a step's
selection back only before its buffer is reused, so host-thread stalls
shorter than three passes cost no GPU time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0.  `value` = candidates balance-checked per
second over all GPUs (device time, max over ranks, inputs resident in HBM);
`e2e` = the same metric through the public API (monte_carlo_pool with the
covariates in host memory, accepted pool returned to host memory).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_UNITS, N_TREATED, D_COV = 1000, 500, 64
M_PER_GPU = 10**8
ACCEPT = 1e-3
SEED = 42
X_SEED = 2  # X = default_rng(2).standard_normal((1000, 64))
FLOPS_PER_CAND = 2 * N_UNITS * D_COV  # algorithmic: treated-minus-control mean difference GEMV


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return j, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    # Sampling every 500 ms: each NVML query can stall this process's CUDA
    # calls for tens of ms (measured at 200 ms: 10% of the step time lost to
    # stalls of the select's host syncs; 500 ms: 0.5%, no sampling: 0).
    # nvidia-smi writes to a temporary file that is parsed after the timed
    # region: a reader thread in this interpreter would contend for the GIL
    # with the step's host orchestration and show up as ~5% step time.
    def __enter__(self):
        import tempfile

        self.log = tempfile.TemporaryFile(mode="w+")
        if os.environ.get("FRR_NO_CLOCKS"):  # diagnostics only
            self.proc = None
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", os.environ.get("FRR_CLOCK_MS", "500")], stdout=self.log, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        # let nvidia-smi finish its NVML start-up before the timed region:
        # its first samples stall CUDA API calls of this process (measured:
        # the timed step that overlapped the second sample took 12-100 ms
        # longer), so wait until two samples are written
        deadline = time.time() + 5.0
        while self.proc is not None and time.time() < deadline:
            self.log.flush()
            self.log.seek(0)
            if sum(1 for _ in self.log) >= 2:
                break
            time.sleep(0.01)
        self.log.seek(0, os.SEEK_END)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        self.log.seek(0)
        for line in self.log:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)
        self.log.close()

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


class NvmlStepSampler:
    """Clocks and throttle reasons read through NVML (the library nvidia-smi
    uses) from this process, once per step, right after the step's pass-1
    kernel is launched: the query runs while the GPU is busy with that
    kernel, so it cannot stall the step's later host syncs the way an
    asynchronous nvidia-smi sample landing in the select does (measured: a
    sample that lands there adds 1-10 ms, occasionally 60 ms, to a 100 ms
    step).  Falls back to ClockSampler when pynvml is unavailable."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.handle = None
        self.fallback = None

    def __enter__(self):
        try:
            import pynvml
            import torch

            pynvml.nvmlInit()
            self.nv = pynvml
            pr = torch.cuda.get_device_properties(self.index)
            try:
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                self.handle = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:  # noqa: BLE001
                self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.sample()
        except Exception:  # noqa: BLE001
            self.handle = None
            self.fallback = ClockSampler(self.index).__enter__()
        return self

    def sample(self):
        if self.handle is None:
            return
        nv = self.nv
        sm = nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(self.handle, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        self.samples.append([str(sm), str(mx)] + ["Active" if r & b else "Not Active" for b in bits])

    def __exit__(self, *a):
        if self.fallback is not None:
            self.fallback.__exit__(*a)
            self.samples = self.fallback.samples
            return
        try:
            self.nv.nvmlShutdown()
        except Exception:  # noqa: BLE001
            pass

    def summary(self):
        out = ClockSampler.summary(self)
        out["source"] = "nvidia-smi -lms" if self.fallback is not None else "NVML, once per timed step"
        return out


def _dist():
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return rank, world, local


def _max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def cpu_sample(budget_s: float = 15.0, threads: int | None = None):
    """The reference algorithm (numpy port, oracle/) on a bounded prefix of
    the same workload: batches of the C2 draws until ~budget_s seconds."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    threads = threads or (os.cpu_count() or 1)
    X = np.random.default_rng(X_SEED).standard_normal((N_UNITS, D_COV))
    bal = O.balance_setup(X, O.precision(X, "exact"))
    chunk = 10_000 * threads
    done, t0 = 0, time.perf_counter()
    all_stats = []
    while time.perf_counter() - t0 < budget_s:
        all_stats.append(O.np_mc_pass1(bal, N_TREATED, SEED, done, chunk, batch_size=10_000, workers=threads))
        done += chunk
    stats = np.concatenate(all_stats)
    O.np_select(stats, ACCEPT)
    el = time.perf_counter() - t0
    return {"value": done / el, "unit": "candidates/s", "cores": threads, "kind": "port",
            "sample": f"C2 draws [0, {done}) of seed {SEED}: numpy port of keys.batch_assignments + "
                      f"BalanceKernel.stats (OpenBLAS) + stable-argsort select, {threads} threads, {el:.1f} s",
            "seconds": el}


def run_reference(args):
    """Reference arm: the reference's CPU algorithm (oracle numpy port) on the
    box's host cores; under torchrun only rank 0 works."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    steps = []
    budget = max(2.0, 60.0 / max(1, args.warmup + args.steps))
    for i in range(args.warmup + args.steps):
        cb = cpu_sample(budget_s=budget)
        if i >= args.warmup:
            steps.append(cb)
    v = float(np.mean([s["value"] for s in steps]))
    cb = dict(steps[-1])
    cb["value"] = v
    line = {"metric": "candidate randomizations balance-checked/sec", "value": v, "unit": "candidates/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * float(np.mean([s["seconds"] for s in steps])), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64+f64", "data": "synthetic",
            "config": _config(args.gpus), "impl": "reference", "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "candidates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _config(gpus):
    return {"workload": "C2: monte_carlo n=1000 n_treated=500 d=64, 1e8 candidates per GPU, prob_accept=1e-3",
            "n_units": N_UNITS, "n_treated": N_TREATED, "d": D_COV, "candidates_per_gpu": M_PER_GPU,
            "candidates_total": M_PER_GPU * gpus, "accept_prob": ACCEPT, "precision": "exact (bit-exact stats)",
            "parallelism": f"candidate-index shards x{gpus}",
            "l2": "stats buffer 800 MB/GPU > 126 MB L2; the 384 KB int8-limb operand stays L2-resident by design"}


def run_ours(args):
    import torch

    import paper_2501_07642_b200 as frr
    from paper_2501_07642_b200 import _native as N
    from paper_2501_07642_b200 import generation as G
    from paper_2501_07642_b200._select import DeviceSelectOps, TorchComm, LocalComm, select_start

    rank, world, local = _dist()
    dev = torch.device("cuda", local)
    comm = TorchComm() if world > 1 else LocalComm()
    X = np.random.default_rng(X_SEED).standard_normal((N_UNITS, D_COV))
    total = M_PER_GPU * world
    design = frr.DesignSpec(N_UNITS, N_TREATED, accept_prob=ACCEPT, max_draws=total, batch_size=10_000,
                            root_seed=SEED)
    prec = frr.precompute_precision(X, "exact")
    kern = prec._kernel
    lo, hi = G._shard(total, comm)
    stats = torch.empty(hi - lo, dtype=torch.float64, device=dev)
    k = G._accepted_count(ACCEPT, total)
    ops = DeviceSelectOps()
    stream = torch.cuda.current_stream()

    # statistics buffers in flight: the host may stall for up to (depth - 1)
    # passes (~100 ms each) without leaving the GPU idle
    depth = max(2, int(os.environ.get("FRR_BENCH_DEPTH", "4")))
    bufs = [stats] + [torch.empty_like(stats) for _ in range(depth - 1)]

    def launch_pass1(i, ev=None, clk=None):
        if ev:
            ev[0].record(stream)
        G.mc_stats_device(kern, design, lo, hi - lo, out=bufs[i % depth])
        if ev:
            ev[1].record(stream)
        if clk is not None:
            clk.sample()  # while pass 1 runs (see NvmlStepSampler)

    def run_steps(n, evs=None, clk=None, end_ev=None):
        """n steps, each pass 1 over this GPU's candidates + the exact select.
        The stream runs them strictly in order.  The host keeps up to `depth`
        steps enqueued (each in its own statistics buffer) and reads a step's
        selection back only before its buffer is reused, so a host thread
        that stalls for less than depth - 1 passes (seen on these VMs: 10 ms
        to over 100 ms) leaves no gap on the GPU."""
        from collections import deque

        jobs, res = deque(), None
        dbg = [] if (evs and os.environ.get("FRR_BENCH_DEBUG")) else None
        for i in range(n):
            t0 = time.perf_counter()
            if len(jobs) == depth:
                res = jobs.popleft().finish()  # before pass 1 overwrites its buffer
            t1 = time.perf_counter()
            launch_pass1(i, evs[i] if evs else None, clk)
            t2 = time.perf_counter()
            jobs.append(select_start(bufs[i % depth], lo, k, ops, comm, m_total=total))
            if dbg is not None:
                dbg.append((round(1e3 * (t1 - t0), 1), round(1e3 * (t2 - t1), 1),
                            round(1e3 * (time.perf_counter() - t2), 1)))
        if dbg is not None:
            print("host ms per step (finish, pass-1 launch, select enqueue):", dbg, file=sys.stderr)
        if end_ev is not None:
            end_ev.record(stream)  # the GPU reaches it when the last select is done
        while jobs:
            res = jobs.popleft().finish()
        return res

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # no interpreter garbage collection inside the timed region (as timeit
    # does): a collection pass stalls the host between the select's kernels
    import gc

    gc.collect()
    gc.disable()
    with NvmlStepSampler(local) as clk:
        # warm-up under the same conditions as the timed steps
        run_steps(args.warmup, clk=clk)
        torch.cuda.synchronize()
        _barrier(world)
        torch.cuda.synchronize()
        launches0 = int(N.lib().frr_launch_count())
        import paper_2501_07642_b200._select as SEL

        fallbacks0 = SEL.FALLBACKS
        t_last = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        res = run_steps(args.steps, evs, clk, end_ev=t_last)
        t_end.record(stream)
        if SEL.FALLBACKS == fallbacks0:
            # no select fell back (which enqueues more work during the reads):
            # the timed region ends where the GPU finished the last select, not
            # where the host got round to recording an event after its reads
            t_end = t_last
        launches = int(N.lib().frr_launch_count()) - launches0  # libfrr kernels of the timed region
        torch.cuda.synchronize()
    gc.enable()
    if os.environ.get("FRR_BENCH_DEBUG"):
        print("pass1 ms:", [round(a.elapsed_time(b), 2) for a, b in evs],
              "gaps ms:", [round(evs[i][1].elapsed_time(evs[i + 1][0]), 2) for i in range(args.steps - 1)],
              file=sys.stderr)
    _barrier(world)
    torch.cuda.synchronize()
    ms = t_start.elapsed_time(t_end) / args.steps
    ms = _max_over_ranks(ms, world)
    kern_ms = float(np.mean([a.elapsed_time(b) for a, b in evs]))
    value = total / (ms / 1e3)
    n_acc = int(res[0].shape[0])

    # ---- end to end through the public API: host X in, host pool out
    e2e_steps = max(1, min(args.steps, 5))
    frr.monte_carlo_pool(X, design)  # warm-up (first-call kernel attributes, allocator)
    _barrier(world)
    torch.cuda.synchronize()
    gc.collect()
    gc.disable()  # as in the timed region (and timeit)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        pool = frr.monte_carlo_pool(X, design)
    torch.cuda.synchronize()
    e2e_s = _max_over_ranks((time.perf_counter() - t0) / e2e_steps, world)
    gc.enable()
    h2d = N_UNITS * D_COV * 8 + 2 * D_COV * 8 + 8 * 16  # Zq, colsum, cc, (seeds/state)
    # accepted draw indices + stats, the (seed, draw) keys built on the device,
    # and the select's result scalars
    d2h = pool.n_accepted * 16 + pool.n_accepted * 16 + 8 * 4
    assert pool.n_accepted == k and n_acc == k

    peaks, src = _peaks()
    peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    achieved = (hi - lo) * FLOPS_PER_CAND / (kern_ms / 1e3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("k_mc_stats_mma_bytes_per_launch")
    draw_peak = _draw_peak(N)
    issue = None
    ip = os.path.join(ROOT, "profiles", "issue.json")
    if os.path.exists(ip):
        with open(ip) as f:
            issue = json.load(f)
    if rank != 0:
        return
    cb = cpu_sample() if (world == 1 and not args.no_cpu) else None
    line = {
        "metric": "candidate randomizations balance-checked/sec", "value": value, "unit": "candidates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int8-limb tensor core + int64 + f64",
        "data": "synthetic", "config": _config(world),
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "k_mc_stats_mma", "kernel_ms_per_launch": kern_ms,
                     "algorithmic_flops_per_candidate": FLOPS_PER_CAND,
                     "peak_source": f"{src} bf16 dense sustained (MEASURED_PEAKS.json)",
                     "note": "binding resource is integer issue (bit-exact splitmix64 Fisher-Yates); see DESIGN.md"},
        "int_roofline": {"bound": "int-issue", "unit": "draws/s",
                         "achieved": (hi - lo) * N_TREATED / (kern_ms / 1e3), "peak": draw_peak,
                         "frac": (hi - lo) * N_TREATED / (kern_ms / 1e3) / draw_peak,
                         "peak_source": "k_microbench_draws in this run: splitmix64 + exact bounded reduction "
                                        "with constants in registers, full occupancy (include/frr.h)",
                         "ncu": issue},
        "cpu_baseline": cb,
        "e2e": {"value": total / e2e_s, "unit": "candidates/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "api": "paper_2501_07642_b200.monte_carlo_pool(X_host, design)"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "accepted_per_step": k,
    }
    print(json.dumps(line), flush=True)


def _draw_peak(N):
    """Generator arithmetic ceiling (draws/s) of this GPU, best of 4 launches."""
    torch = N.torch_mod()
    sink = torch.zeros(1, dtype=torch.int64, device="cuda")
    tot = N.ctypes.c_int64(0)
    best = 0.0
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        N.call("frr_microbench_draws", 1 << 14, N.ptr(sink), N.ctypes.byref(tot), N.stream_ptr())
        e1.record()
        torch.cuda.synchronize()
        best = max(best, tot.value / (e0.elapsed_time(e1) / 1e3))
    return best


def _self_launch(args) -> int:
    """--gpus N > 1 without a torchrun environment: re-launch this script as N
    ranks (one process per GPU, NCCL) through torch.distributed.run."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, this node has {have}", file=sys.stderr)
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # keep NCCL's init log (communicator size per rank)
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if world == 0 and args.gpus > 1:
        sys.exit(_self_launch(args))
    if world and world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
