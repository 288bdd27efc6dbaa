"""bench.py output contract (reference arm, runnable without a GPU) — `-m "not gpu"`:
exactly one JSON line on stdout with the keys the driver reads."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 1 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["unit"] == d["unit"]
    assert "workload" in d["config"]


def test_gpus_n_self_launches_ranks():
    """`bench.py --gpus 2` outside torchrun starts 2 ranks itself (torchrun on 127.0.0.1;
    gloo without a GPU) and still prints exactly one JSON line, from rank 0, n_gpus = 2."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                           "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--config", "c1", "--steps", "1", "--warmup", "1"], capture_output=True, text=True,
                         timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference" and d["value"] > 0


def test_pair_roofline_arithmetic():
    """roofline.pair = (K1 + K2 algorithmic bytes) / (summed per-launch event times) / peak,
    None when either kernel did not run."""
    sys.path.insert(0, ROOT)
    import bench

    class FakeSolver:
        def kernel_bytes(self, name):
            return {"primal_step_AT": 3.79e9, "dual_step_A": 3.28e9}[name]

    kt = {"primal_step_AT": (69.0, 100), "dual_step_A": (82.7, 100)}   # (total ms, launches)
    p = bench.pair_roofline(FakeSolver(), kt, 6550.7)
    assert abs(p["ms"] - 1.517) < 1e-9
    assert abs(p["achieved"] - 7.07e9 / 1.517e-3 / 1e9) < 1e-6
    assert abs(p["frac"] - p["achieved"] / 6550.7) < 1e-12
    assert bench.pair_roofline(FakeSolver(), {"primal_step_AT": (69.0, 100)}, 6550.7) is None
