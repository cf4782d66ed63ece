"""Full-size sharded pools (test infrastructure): C2 (1e8 Monte Carlo draws)
and C4 (2,333,606,220 exact ranks) built by the product's multi-rank path
with world sizes 1, 2 and 4, the ranks sharing this box's one GPU over a
gloo group (TorchComm stages CUDA tensors through the host; NCCL with one
GPU per rank is the production backend).  Every world size must give the
same accepted pool bit for bit -- SURVEY section 8 (e), the analogue of the
reference's worker-count invariance test (test_acceptance.py:247-267).

    python tests/parity/sharded_full.py > sharded_full.json"""
import hashlib
import json
import os
import socket
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def _digest(*arrays):
    h = hashlib.sha1()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()[:16]


def _case(name):
    import paper_2501_07642_b200 as frr

    t0 = time.perf_counter()
    if name == "C2":
        X = np.random.default_rng(2).standard_normal((1000, 64))
        d = frr.DesignSpec(1000, 500, accept_prob=1e-3, max_draws=10**8, batch_size=10_000, root_seed=42)
        p = frr.monte_carlo_pool(X, d)
        dig = _digest(p.accepted_indices, p.stats, np.array([p.threshold_value]), p.keys)
    else:
        X = np.random.default_rng(4).standard_normal((34, 5))
        d = frr.DesignSpec(34, 17, accept_prob=1e-3, mode="exact", enumeration_cap=10**10)
        p = frr.enumerate_exact(X, d)
        dig = _digest(p.accepted_indices, p.stats, np.array([p.threshold_value]), p.assignments)
    return {"digest": dig, "accepted": int(p.n_accepted), "threshold": float(p.threshold_value),
            "seconds": time.perf_counter() - t0}


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out[rank] = {c: _case(c) for c in ("C2", "C4")}
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    import torch.multiprocessing as mp

    res = {"world_1": {c: _case(c) for c in ("C2", "C4")}}
    for world in (2, 4):
        with mp.Manager() as man:
            out = man.dict()
            mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
            res[f"world_{world}"] = {f"rank_{r}": v for r, v in sorted(dict(out).items())}
    ref = {c: res["world_1"][c]["digest"] for c in ("C2", "C4")}
    equal = all(v[c]["digest"] == ref[c] for w, ranks in res.items() if w != "world_1"
                for v in ranks.values() for c in ("C2", "C4"))
    print(json.dumps({"all_world_sizes_equal": equal, "reference_digests": ref, "runs": res}))


if __name__ == "__main__":
    main()
