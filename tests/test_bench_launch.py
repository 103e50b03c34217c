"""bench.py's launcher on CPU: `--gpus N` without a torchrun environment
re-launches itself under torch.distributed.run with N ranks (the driver's
multi-GPU path).  The reference arm runs on the host only, so the spawn, the
rank/world plumbing and the single JSON line of rank 0 are exercised here
without a GPU: rank 0 prints n_gpus = N, the other ranks exit 0 silently."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=600, env=e, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    return lines


def test_spawn_two_ranks_reference_arm():
    lines = _run(["--impl", "reference", "--gpus", "2", "--config", "1", "--steps", "2", "--warmup", "1"])
    assert len(lines) == 1                      # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["scaling"] == "strong" and d["config"]["t_per_gpu"] == 32   # 64 columns split in two
    assert d["config"]["parallelism"] == "columns/2"
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]


def test_single_rank_reference_arm_matches_config():
    lines = _run(["--impl", "reference", "--config", "1", "--steps", "2", "--warmup", "1"])
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["config"]["workload"].startswith("c1_")
    assert d["config"]["t_per_gpu"] == 64 and d["cpu_baseline"]["kind"] == "oracle"


def test_default_config_is_the_largest():
    """bench.py's default workload is configs[4] (C = 5), the largest config
    that fits one GPU (X = 51.5 GB)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    old = sys.argv
    try:
        sys.argv = ["bench.py"]
        a = mod.parse()
    finally:
        sys.argv = old
    assert a.config == 5 and a.scaling == "strong" and a.gpus == 1
