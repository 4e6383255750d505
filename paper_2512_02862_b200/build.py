"""Builds paper_2512_02862_b200/libpsg.so in-tree: sm_100a CUDA kernels (nvcc) + C++ host engine (g++).

    python -m paper_2512_02862_b200.build         # incremental
    python -m paper_2512_02862_b200.build --clean

The .so is git-ignored but travels to the GPU box with gpurun snapshots. cudart is linked
statically (version-consistent with nvcc 12.9); NCCL is the torch-bundled libnccl.so.2 (rpath).
"""
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_obj")
LIB = os.path.join(HERE, "libpsg.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
SITE = sysconfig.get_paths()["purelib"]
NCCL_DIR = os.path.join(SITE, "nvidia", "nccl")
JSON_DIR = os.path.join(SITE, "include", "cudnn_frontend", "thirdparty", "nlohmann")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed: %s\n%s%s" % (" ".join(cmd), r.stdout, r.stderr))
    return r.stderr


def _stale(obj, srcs):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(s) > t for s in srcs)


def build(verbose=False):
    os.makedirs(OBJ, exist_ok=True)
    headers = glob.glob(os.path.join(CSRC, "*.hpp")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "psg.h")]
    inc = ["-I" + os.path.join(ROOT, "include"), "-I" + CSRC, "-I" + os.path.join(CUDA, "include"),
           "-I" + os.path.join(NCCL_DIR, "include"), "-I" + JSON_DIR]
    jobs = []
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cu"))):
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        if _stale(obj, [src] + headers):
            jobs.append([os.path.join(CUDA, "bin", "nvcc"), *ARCH, "-O3", "-lineinfo", "-std=c++17",
                         "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3", *inc, "-c", src, "-o", obj])
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cpp"))):
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        if _stale(obj, [src] + headers):
            jobs.append(["g++", "-std=c++20", "-O2", "-g", "-fPIC", "-Wall", "-Wno-unused-function", *inc, "-c", src,
                         "-o", obj])
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for err in ex.map(_run, jobs):
            if verbose and err:
                sys.stderr.write(err)
    objs = sorted(glob.glob(os.path.join(OBJ, "*.o")))
    if jobs or not os.path.exists(LIB):
        nccl_lib = os.path.join(NCCL_DIR, "lib")
        _run(["g++", "-shared", "-o", LIB + ".tmp", *objs, "-L" + os.path.join(CUDA, "lib64"), "-lcudart_static",
              os.path.join(nccl_lib, "libnccl.so.2"), "-Wl,-rpath," + nccl_lib, "-lz", "-ldl", "-lrt", "-lpthread"])
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    if "--clean" in sys.argv:
        shutil.rmtree(OBJ, ignore_errors=True)
        if os.path.exists(LIB):
            os.remove(LIB)
    print(build(verbose="-v" in sys.argv))
