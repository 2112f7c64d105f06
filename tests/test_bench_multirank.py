"""bench.py --gpus N on CPU: the self-launch under torchrun, request sharding, max-over-ranks timing and
the aggregate / per-GPU arithmetic, with the kernels replaced by a host stub (tests/bench_stub) and gloo
in place of NCCL (MV_BENCH_DEVICE=cpu).  SURVEY.md §8e: requests shard with no collective."""
import json
import os
import pathlib
import subprocess
import sys

import pytest

REPO = pathlib.Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("gpus", [2])
def test_bench_gpus_flag_launches_ranks(gpus):
    env = dict(os.environ, MV_BENCH_DEVICE="cpu", PYTHONPATH=str(REPO / "tests" / "bench_stub"))
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, str(REPO / "bench.py"), "--gpus", str(gpus), "--steps", "5", "--warmup", "3",
                        "--requests", "1", "--extras", "none"], capture_output=True, text=True, env=env,
                       cwd=REPO, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    line = lines[0]
    assert line["n_gpus"] == gpus
    assert line["config"]["requests_per_gpu"] == 1 and line["config"]["branches_per_gpu"] == 8
    # aggregate = all ranks' branch tokens per step / the slowest rank's step time
    tokens = 8 * gpus
    assert line["value"] == pytest.approx(tokens / (line["ms_per_step"] / 1e3), rel=1e-6)
    assert line["value_per_gpu"] == pytest.approx(line["value"] / gpus, rel=1e-9)
    assert line["ms_per_step"] >= 2.0  # the stub kernel sleeps 2 ms per step on every rank
    assert line["config"]["parallelism"] == f"requests x{gpus}, no collective"


def test_bench_rejects_world_mismatch():
    env = dict(os.environ, MV_BENCH_DEVICE="cpu", PYTHONPATH=str(REPO / "tests" / "bench_stub"), WORLD_SIZE="1",
               RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, str(REPO / "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
                        "--requests", "1", "--extras", "none"], capture_output=True, text=True, env=env, cwd=REPO,
                       timeout=300)
    assert r.returncode != 0 and "WORLD_SIZE=1" in r.stderr
