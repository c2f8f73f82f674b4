"""CPU (gloo) check of bench.py's N > 1 path (VERDICT r1 "make SCALE measurable"): `--gpus N`
spawns N ranks itself (torch.distributed.run on 127.0.0.1), every grouped call's y shards are
gathered with ONE collective (64 per Llama-3.2-1B token), the layer-sharded sketch is replicated;
the assembled outputs and sketch bytes are identical to N = 1.  A launcher whose WORLD_SIZE
disagrees with --gpus is refused."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(n, env_extra=None):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--dist-selftest"],
                          capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)


def _line(out):
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads([l for l in out.stdout.strip().splitlines() if l.startswith("{")][-1])


@pytest.mark.parametrize("n", [2, 3])
def test_spawned_ranks_match_single_rank(n):
    one, many = _line(_run(1)), _line(_run(n))
    assert one["n_gpus"] == 1 and many["n_gpus"] == n
    assert many["y_sha256"] == one["y_sha256"] and many["sketch_sha256"] == one["sketch_sha256"]
    assert one["y_exact"] and many["y_exact"]
    assert one["collectives_per_step"] == 0 and many["collectives_per_step"] == 64


def test_world_size_mismatch_refused():
    out = _run(2, {"WORLD_SIZE": "1", "RANK": "0"})
    assert out.returncode == 2 and "WORLD_SIZE" in out.stderr
