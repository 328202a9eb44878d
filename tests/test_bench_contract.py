"""bench.py's JSON-line contract, checked on the CPU.

The reference arm (`bench.py --impl reference`) times the oracle port of the
reference's `_train_pass` (trainer.py:184-207) on host cores; it runs here
without a GPU, so its line is checked end to end.  The GPU arm cannot run
here; its workload description comes from the same `workload_config()` /
`sharded_config()` functions the reference arm prints, which is what lets
the driver compare the two lines' `config` dicts key for key."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

REQUIRED = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
            "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"}


def test_reference_arm_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "3",
                          "--warmup", "3"], cwd=ROOT, capture_output=True, text=True,
                         timeout=600, env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout  # exactly one JSON line
    d = json.loads(lines[0])
    assert REQUIRED <= set(d), REQUIRED - set(d)
    assert d["impl"] == "reference"
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["metric"] == "sample-updates/sec" and d["unit"] == "updates/s"
    assert d["higher_is_better"] is True and d["value"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["sample"]
    assert cb["value"] == d["value"] and cb["unit"] == d["unit"]
    e2e = d["e2e"]
    assert e2e["value"] == d["value"] and e2e["unit"] == d["unit"]
    assert e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0
    import bench
    assert d["config"] == json.loads(json.dumps(bench.workload_config()))


def test_arms_share_the_config_builders():
    """Both arms of both workloads take `config` from the shared builders."""
    src = open(os.path.join(ROOT, "bench.py")).read()
    import bench
    for fn in ("run_reference", "run_ours"):
        body = src.split(f"def {fn}(")[1].split("\ndef ")[0]
        assert '"config": workload_config()' in body, fn
    for fn in ("run_sharded", "run_sharded_reference"):
        body = src.split(f"def {fn}(")[1].split("\ndef ")[0]
        assert '"config": sharded_config()' in body, fn
    cfg = bench.workload_config()
    assert cfg["workload"].startswith("C2") and cfg["dim"] == 128 and cfg["negatives"] == 3
    assert "workload" in bench.sharded_config()


def test_rejects_fewer_than_three_warmups():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                          "--warmup", "1"], cwd=ROOT, capture_output=True, text=True,
                         timeout=300, env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    assert out.returncode != 0 and "--warmup must be >= 3" in out.stderr
