"""CPU checks of bench.py's contract pieces that need no GPU: the reference arm (the oracle timed on
this host's cores on a bounded, extrapolated block sample) prints one valid JSON line with the keys
the driver reads; --gpus N against a different WORLD_SIZE is refused; the block sample is spread
evenly and covers every block when it is at least K."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          env=e, timeout=600)


def test_reference_arm_json_line():
    r = _bench(["--impl", "reference", "--config", "cfg2s", "--steps", "2", "--warmup", "1", "--cpu-blocks", "4"])
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["higher_is_better"] is True
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and "extrapolated" in cb["sample"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_gpus_must_match_world_size():
    r = _bench(["--gpus", "2", "--impl", "reference", "--config", "cfg1"], env={"WORLD_SIZE": "1", "RANK": "0"})
    assert r.returncode != 0
    assert "WORLD_SIZE" in r.stdout


def test_sample_blocks():
    sys.path.insert(0, ROOT)
    import bench
    assert bench._sample_blocks(64, 16) == list(range(0, 64, 4))
    assert bench._sample_blocks(4, 16) == [0, 1, 2, 3]
    b = bench._sample_blocks(1024, 16)
    assert len(b) == 16 and b[0] == 0 and b[-1] == 960
