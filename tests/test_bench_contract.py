"""bench.py's JSON contract on the CPU-only reference arm (the oracle timed on
host cores): one line with the required keys, the reference markers, an e2e
object without host<->device bytes, and no libfrsvt loaded in that arm."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ref_line(*extra):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", *extra], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [x for x in out.stdout.splitlines() if x.strip().startswith("{")]
    assert len(lines) == 1
    return json.loads(lines[0])


@pytest.mark.parametrize("config,unit", [("c5", "iter/s"), ("c1", "calls/s")])
def test_reference_arm_json_line(config, unit):
    d = _ref_line("--config", config, *(["--ref-rows", "512"] if config == "c5" else []))
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == unit and d["higher_is_better"] is True
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith(config)


def test_reference_arm_does_not_load_the_library():
    """The oracle arm never maps libfrsvt.so (it must run without the build)."""
    code = ("import runpy, sys; sys.argv=['bench.py','--impl','reference','--steps','1','--warmup','0',"
            "'--config','c1']; runpy.run_path('bench.py', run_name='__main__'); "
            "maps=open('/proc/self/maps').read(); assert 'libfrsvt' not in maps, 'libfrsvt mapped'; "
            "assert 'paper_1509_00296_b200' not in sys.modules")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]


def test_gpus_flag_launches_ranks():
    """`--gpus 2` outside torchrun re-launches under torch.distributed.run: the
    reference arm then reports n_gpus 2 from rank 0 (gloo, no GPU needed)."""
    d = _ref_line("--config", "c1", "--gpus", "2")
    assert d["n_gpus"] == 2
