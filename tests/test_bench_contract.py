"""CPU checks of bench.py's contract that need no GPU: the reference arm (the oracle)
prints one JSON line with the keys the driver reads, and the scenario sharding used
by the GPU arm partitions the scenarios."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "C1",
                          "--steps", "1", "--warmup", "1"], cwd=ROOT, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("C1:")
    assert "model" not in d["config"]


def test_scenario_blocks_cover_all_scenarios():
    sys.path.insert(0, ROOT)
    import importlib
    bench = importlib.import_module("bench")

    class A:
        scenarios = 10
        scaling = "strong"
    for world in (1, 2, 3, 4):
        got = []
        for rank in range(world):
            b0, b1 = bench.scenario_block(A, rank, world)
            got.extend(range(b0, b1))
        assert got == list(range(10)), world


def test_launcher_spawns_ranks_dry_run():
    """`bench.py --gpus 2` started directly re-launches itself as 2 ranks
    (torch.distributed.run, 127.0.0.1); the ranks rendezvous (gloo) and rank 0 reports
    n_gpus == --gpus (VERDICT r1 'runnable N-GPU path')."""
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run"], cwd=ROOT,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["dry_run"] and d["n_gpus"] == 2 and d["ranks_seen"] == 2


def test_reference_arm_levelize_config():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config",
                          "C2-tree", "--steps", "1", "--warmup", "0"], cwd=ROOT,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][0])
    assert d["config"]["workload"].startswith("C2-tree:") and d["value"] > 0
    assert d["paper_context"]["speedup"] == 7.7
