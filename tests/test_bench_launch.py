"""CPU tests of bench.py's launch contract (VERDICT r1 "multi-GPU readiness"):
`--gpus N` without a launcher spawns N ranks itself (torch.distributed.run on
127.0.0.1) and rank 0 prints one JSON line with n_gpus = N; a launcher whose
WORLD_SIZE disagrees with --gpus is an error.  The reference arm (the CPU
oracle) runs on CPU, so the spawn path is exercised here without a GPU."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _env(**kw):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                           "MASTER_PORT")}
    env.update(kw)
    return env


def test_gpus_n_spawns_n_ranks_and_rank0_prints_one_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--config", "c1", "--steps", "2", "--warmup", "1"], cwd=ROOT, env=_env(),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["steps"] == 2
    assert d["ms_per_step"] > 0 and d["value"] > 0
    assert "spawning 2 ranks" in r.stderr


def test_world_size_mismatch_is_an_error():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "1",
                        "--config", "c1", "--steps", "1", "--warmup", "0"], cwd=ROOT,
                       env=_env(WORLD_SIZE="2", RANK="0", LOCAL_RANK="0"), capture_output=True, text=True,
                       timeout=300)
    assert r.returncode != 0
    assert "--gpus 1 but 2 rank(s)" in r.stderr
