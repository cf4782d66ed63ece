"""bench.py's launch contract on a machine without enough GPUs (no GPU
needed): --gpus N > 1 outside torchrun self-launches N ranks only when N
GPUs exist, else it fails loudly; a torchrun world must match --gpus; the
warm-up floor is enforced."""

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          env=e, timeout=300)


def test_gpus_without_gpus_fails_loudly():
    r = _run(["--gpus", "2", "--steps", "1", "--warmup", "3"], {"CUDA_VISIBLE_DEVICES": ""})
    assert r.returncode == 2 and "needs 2 GPUs" in r.stderr


def test_world_must_match_gpus():
    r = _run(["--gpus", "4", "--steps", "1", "--warmup", "3"], {"WORLD_SIZE": "2"})
    assert r.returncode == 2 and "WORLD_SIZE=2 but --gpus 4" in r.stderr


def test_warmup_floor():
    r = _run(["--steps", "1", "--warmup", "1"])
    assert r.returncode != 0 and "--warmup must be >= 3" in r.stderr
