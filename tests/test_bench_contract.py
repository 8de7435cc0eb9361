"""bench.py's reference arm on the CPU (no GPU needed): the JSON line the driver parses —
metric / value / unit / higher_is_better / cpu_baseline / e2e keys — from the unmodified
reference (oracle/_ref) timed on a small sample."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    from oracle.bind import reference_available
    if not reference_available():
        pytest.skip("oracle/_ref not built")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1", "--ref-nodes", "4000",
                          "--ref-candidates", "8"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "config", "cpu_baseline",
              "e2e"):
        assert k in line, k
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["candidates"]["value"] > 0 and line["candidates"]["matches_golden"] is True
    assert line["host"]["cores"] >= 1


def test_reference_arm_maps_no_product_library():
    """The reference arm synthesises its inputs with oracle/_ref: libdagplace_b200.so must
    not be mapped in that process."""
    from oracle.bind import reference_available
    if not reference_available():
        pytest.skip("oracle/_ref not built")
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0', "
            "'--ref-nodes', '3000', '--candidates', '0']; "
            "runpy.run_path(sys.argv[0], run_name='__main__'); "
            "maps = open('/proc/self/maps').read(); "
            "assert 'libdagplace_b200' not in maps, 'product library mapped'; "
            "assert 'libdagplace_ref' in maps")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
