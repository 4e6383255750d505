"""The C++ consumer of the C ABI (tests/cabi/run_plan.cpp) runs the canonical plan on the GPU and
reproduces the reference's SF0.01 result (first group and group count)."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_program_runs_plan_through_c_abi(tmp_path):
    import subprocess
    from test_abi import _build_cabi_example
    exe = _build_cabi_example(tmp_path)
    golden = json.load(open(os.path.join(ROOT, "tests", "golden", "results.json")))
    plan = tmp_path / "plan.json"
    plan.write_text(json.dumps(golden["plans"]["canonical"]))
    data = str(tmp_path / "d")
    r = subprocess.run([exe, str(plan), data, "0.01"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    head = r.stdout.split()
    assert head[:4] == ["rows", "1145", "cols", "4"]
    raw = np.fromfile(os.path.join(ROOT, "tests", "golden", "q3_s001_rows.bin"), dtype="<u8")
    first = raw[2:6].tolist()
    i = head.index("first")
    assert [int(x) for x in head[i + 1:i + 5]] == first
