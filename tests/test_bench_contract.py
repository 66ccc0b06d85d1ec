"""bench.py output contract: one JSON line with the keys the driver reads.

The reference arm runs on CPU (the oracle port on host cores), so its line is
checked in the CPU suite; our arm needs the GPU (marked gpu).
"""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=600):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0])


BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def test_reference_arm_line():
    d = _run("--impl", "reference", "--workload", "tiny", "--steps", "2", "--warmup", "1")
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(cb) and cb["kind"] in ("port", "reference")
    assert cb["value"] == d["value"] and cb["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert "workload" in d["config"]


@pytest.mark.gpu
def test_our_arm_line():
    d = _run("--workload", "tiny", "--steps", "3", "--warmup", "3")
    assert BASE_KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1.5 and r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    cb = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(cb)
    e = d["e2e"]
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(e)
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["value"] != d["value"]
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)
    assert d["gpu_launches"] >= 5 * d["steps"]
    assert d["config"]["workload"].startswith("tiny")


def test_reference_arm_loads_no_product_code():
    """The --impl reference arm must not touch the product library: its corpus
    comes from the oracle's generator and its chunk from the reference's own
    partition (or the oracle's restatement)."""
    code = (
        "import sys, runpy, json\n"
        f"sys.argv = ['bench.py', '--impl', 'reference', '--workload', 'tiny', '--steps', '1', '--warmup', '1']\n"
        f"runpy.run_path({os.path.join(ROOT, 'bench.py')!r}, run_name='__main__')\n"
        "maps = open('/proc/self/maps').read()\n"
        "print(json.dumps({'so': 'libgfb200' in maps,\n"
        "                  'pkg': any(m.startswith('paper_1803_04631_b200') for m in sys.modules)}))\n"
    )
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    verdict = json.loads(p.stdout.strip().splitlines()[-1])
    assert verdict == {"so": False, "pkg": False}


def test_both_arms_describe_the_same_config():
    """Same command, same `config` object (the driver compares the arms)."""
    sys.path.insert(0, ROOT)
    import bench

    ns = type("A", (), dict(workload="tiny", topics=None, seed=bench.CORPUS_SEED, scaling="strong", shard=None,
                            warmup=3, steps=5))()
    c1 = bench.make_config(ns, 1, bench.corpus_tokens_total(ns, 1))
    from paper_1803_04631_b200 import synth

    T = synth.generate(1000, 1000, 100.0, seed=bench.CORPUS_SEED).num_tokens
    assert c1 == bench.make_config(ns, 1, T)
