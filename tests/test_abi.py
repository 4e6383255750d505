"""CPU-only checks of the product library: it loads, exports every psg.h symbol, and its host-side
pieces (generator, PSTO writer/reader, Eq. 1) match the reference. No GPU compute here."""
import hashlib
import os
import re

import numpy as np
import pytest

import paper_2512_02862_b200 as psg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "psg.h")).read()
    declared = set(re.findall(r"\b(psg_[a-z0-9_]+)\s*\(", hdr))
    assert declared == set(psg.EXPORTS)
    L = psg.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert L.psg_abi_version() == 2


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(psg.PsgError) as e:
        psg.Context(0)
    assert e.value.kind == "CudaError"


@pytest.mark.parametrize("idx", range(7))
def test_product_generator_matches_reference_bytes(idx, gen_hashes, tmp_path):
    spec = gen_hashes[idx]
    d = str(tmp_path / "g")
    psg.gen_workload("tpch", d, devices=spec["devices"], nodes=spec["nodes"], scale=spec["scale"], seed=spec["seed"],
                     codec=spec["codec"], row_group_bytes=spec["rg_bytes"])
    got = {}
    for root, _dirs, files in os.walk(d):
        for f in files:
            if not f.endswith(".psto"):  # the manifest names absolute paths (checked separately)
                continue
            p = os.path.join(root, f)
            got[os.path.relpath(p, d)] = hashlib.sha256(open(p, "rb").read()).hexdigest()
    assert got == spec["files"]


def test_tmin_worked_example():
    gib = 1024 ** 3
    size = int(12.8 * gib)
    assert psg.tmin(size, float(size), 0, 22.3 * gib) == 1.0
    assert psg.tmin(gib, 1.0 * gib, 10 * gib, 5.0 * gib) == 2.0
    with pytest.raises(psg.PsgError):
        psg.tmin(0, 1.0, 0, 1.0)


def test_table_round_trip_and_inspect(tmp_path):
    from oracle import plan_oracle as po
    path = str(tmp_path / "t.psto")
    cols = {"k": np.arange(100, dtype=np.int64), "v": np.arange(100) / 7.0}
    assert psg.write_table(path, cols, row_group_rows=32, codec="block") == 4
    info = psg.inspect(path)
    assert info["rows"] == 100 and info["row_groups"] == 4 and info["codec"] == "block"
    assert info["schema"] == [("k", "int64"), ("v", "float64")]
    back = po.read_table(path)  # independent reader (oracle)
    assert np.array_equal(back["k"].view(np.int64), cols["k"])
    assert np.array_equal(back["v"].view(np.float64), cols["v"])
    meta = po.parse_footer(path)
    assert meta.groups[0][1][0][3] == 0 and meta.groups[0][1][0][4] == 31  # zone min/max


def test_corrupt_footer_raises(tmp_path):
    path = str(tmp_path / "t.psto")
    psg.write_table(path, {"k": np.arange(10, dtype=np.int64)}, row_group_rows=4)
    data = bytearray(open(path, "rb").read())
    bad = str(tmp_path / "bad.psto")
    open(bad, "wb").write(bytes(data[:-1]) + b"X")
    with pytest.raises(psg.PsgError) as e:
        psg.inspect(bad)
    assert e.value.kind == "CorruptFooter"
    with pytest.raises(psg.PsgError) as e:
        psg.inspect(str(tmp_path / "missing.psto"))
    assert e.value.kind == "IoFailure"


def test_query_compiler_builds_every_sink_for_sm100a():
    """NVRTC specialisation of the fused scan (jit.cpp) compiles for sm_100a without a GPU."""
    failures, log = psg.jit_selftest()
    assert failures == 0, log


def test_gen_workload_defaults_and_manifest_match_reference(tmp_path):
    """gen_workload mirrors the reference's defaults (block codec, 1 MiB row groups,
    bench.hpp:42-52) and writes the same manifest.json (bench.cpp:85-114)."""
    import json as _json
    import subprocess
    d = str(tmp_path / "ours")
    mpath = psg.gen_workload("tpch", d, devices=2, nodes=3, scale=0.002, seed=7)
    m = _json.load(open(mpath))
    assert m["kind"] == "tpch-analog" and m["nodes"] == 3 and m["devices"] == 2 and m["seed"] == 7
    assert m["tables"]["customer"]["replicated"] and len(m["tables"]["lineitem"]["paths_per_node"]) == 3
    assert psg.inspect(m["tables"]["lineitem"]["paths_per_node"][0])["codec"] == "block"
    drv = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
    if os.path.exists(drv):
        r = str(tmp_path / "ref")
        subprocess.run([drv, "gen", "--out", r, "--scale", "0.002", "--nodes", "3", "--devices", "2", "--seed", "7",
                        "--codec", "block"], check=True, capture_output=True)
        ref = open(os.path.join(r, "manifest.json")).read().replace(r, "ROOT")
        assert open(mpath).read().replace(d, "ROOT") == ref


def test_synthetic_generator_matches_reference_bytes(tmp_path):
    """gen_workload(kind='synthetic') is byte-identical to the reference's synthetic-join tables
    (tests/golden/synthetic.json, made by the reference generator)."""
    import json as _json
    syn = _json.load(open(os.path.join(ROOT, "tests", "golden", "synthetic.json")))
    for spec in syn["gen"]:
        d = str(tmp_path / ("s%d" % spec["seed"]))
        m = psg.gen_workload("synthetic", d, devices=spec["devices"], nodes=spec["nodes"], seed=spec["seed"],
                             codec=spec["codec"])
        got = {}
        for root, _dirs, files in os.walk(d):
            for f in files:
                if f.endswith(".psto"):
                    p = os.path.join(root, f)
                    got[os.path.relpath(p, d)] = hashlib.sha256(open(p, "rb").read()).hexdigest()
        assert got == spec["files"]
        man = _json.load(open(m))
        assert man["kind"] == "synthetic-join" and man["tables"]["build"]["rows"] == 120000


def _build_cabi_example(tmp_path):
    import subprocess
    exe = str(tmp_path / "run_plan")
    libdir = os.path.join(ROOT, "paper_2512_02862_b200")
    subprocess.run(["g++", "-std=c++17", "-O1", os.path.join(ROOT, "tests", "cabi", "run_plan.cpp"),
                    "-I" + os.path.join(ROOT, "include"), "-L" + libdir, "-lpsg", "-Wl,-rpath," + libdir, "-o", exe],
                   check=True, capture_output=True)
    return exe


def test_cabi_example_compiles_links_and_fails_loudly_without_gpu(tmp_path):
    """A C++ program against include/psg.h links to libpsg.so (the reference-side binding of
    INTEGRATION.md); without a GPU, psg_ctx_create reports CudaError instead of computing."""
    import subprocess
    exe = _build_cabi_example(tmp_path)
    plan = tmp_path / "p.json"
    plan.write_text("{}")
    r = subprocess.run([exe, str(plan), str(tmp_path)], capture_output=True, text=True)
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        assert r.returncode == 2 and "psg error" in r.stderr
