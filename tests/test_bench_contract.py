"""bench.py's reference arm runs on CPU: one JSON line with the contract's keys."""

import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "toy",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "impl", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["cores"] >= 1


def test_gpus_flag_spawns_ranks_dry_run():
    """``bench.py --gpus 2`` outside torchrun launches 2 ranks itself (gloo dry run: the
    rendezvous and the WORLD_SIZE == --gpus check, no GPU)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    # the two ranks share the launcher's stderr, so their lines may interleave mid-line
    ranks = sorted(set(re.findall(r"\[bench\] rank (\d+/\d+)", r.stderr)))
    assert ranks == ["0/2", "1/2"], r.stderr[-2000:]
    assert json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0]) == {"dry_run": True, "n_gpus": 2}


def test_world_size_must_match_gpus():
    env = {**os.environ, "WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=1" in (r.stderr + r.stdout)


def test_frozen_strategies_match_current_graphs():
    """Every committed StrategyFile under profiles/strategies/ still matches its workload's
    cost-annotated graph (else bench.py would re-plan at run time) and validates."""
    import glob

    sys.path.insert(0, ROOT)
    from bench import _workload
    from paper_2406_17145_b200.model import validate_strategy
    from paper_2406_17145_b200.runtime.api import plan_cached
    from paper_2406_17145_b200.workloads import b200_cluster

    files = glob.glob(os.path.join(ROOT, "profiles", "strategies", "*.json"))
    assert files
    for path in files:
        d = json.load(open(path))
        n, mode = d["n_gpus"], d["mode"]
        br = len([s for s in d["strategy"]["graph"]["ops"] if s["name"].endswith("_layer0")]) if d["workload"] == "mmt" else None
        wl = _workload(d["workload"], n, None, br)
        sg, meta = plan_cached(wl, n, mode, costs=d["costs"])
        assert meta["source"] == "frozen", path
        assert validate_strategy(wl.graph, b200_cluster(n), sg) == [], path
