"""ORACLE package — test infrastructure only (see oracle/plan_oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may import this package.
"""
import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def gen_lib():
    """ctypes handle to oracle/_build/liboracle_gen.so (built on demand with gcc)."""
    global _LIB
    if _LIB is None:
        so = os.path.join(_HERE, "_build", "liboracle_gen.so")
        if not os.path.exists(so):
            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        lib = ctypes.CDLL(so)
        lib.orc_gen_tpch.argtypes = [ctypes.c_char_p, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64]
        lib.orc_gen_tpch.restype = ctypes.c_int
        _LIB = lib
    return _LIB


def gen_tpch(out_dir, scale, nodes=1, devices=None, seed=42, codec="identity", rg_bytes=1 << 20):
    rc = gen_lib().orc_gen_tpch(out_dir.encode(), float(scale), int(nodes), int(devices or nodes), int(seed),
                                1 if codec == "block" else 0, int(rg_bytes))
    if rc != 0:
        raise RuntimeError("oracle generator failed rc=%d" % rc)
    return out_dir
