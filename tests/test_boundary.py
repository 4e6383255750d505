"""The drop-in boundary, compiled: the reference-side binding of INTEGRATION.md §1
(tests/cabi/gpu_pipeline_harness.cpp) builds against the UNMODIFIED reference headers
(/root/reference/proj/include) and the reference library (oracle/_ref/libpystachio_ref.a) plus
libpsg.so, and maps every psg status code onto its pystachio::Error class (errors.hpp:21-87).
The GPU run of the same binary is tests/test_gpu_boundary.py."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"
HARNESS = os.path.join(ROOT, "oracle", "_ref", "gpu_pipeline_harness")


@pytest.fixture(scope="module")
def harness():
    if not os.path.isdir(REF_INC) or not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libpystachio_ref.a")):
        pytest.skip("reference sources / oracle/_ref not present (development container only)")
    subprocess.run(["bash", os.path.join(ROOT, "oracle", "build_harness.sh")], check=True, capture_output=True)
    return HARNESS


def test_every_status_code_rethrows_its_reference_class(harness):
    r = subprocess.run([harness, "errors"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = r.stdout.splitlines()
    assert sum(1 for x in lines if " OK" in x) == 13 + 1 + 1, r.stdout
    assert "BAD" not in r.stdout


def test_status_enum_matches_reference_error_classes():
    """psg.h's codes name exactly the reference's exception classes (errors.hpp)."""
    if not os.path.isdir(REF_INC):
        pytest.skip("reference headers not present")
    classes = re.findall(r"class (\w+) : public Error", open(os.path.join(REF_INC, "pystachio", "errors.hpp")).read())
    hdr = open(os.path.join(ROOT, "include", "psg.h")).read()
    named = re.findall(r"PSG_ERR_\w+ = (\d+),\s*/\* (\w+)\s", hdr)
    assert [c for _n, c in named if int(_n) < 100] == classes
