"""Build libipmg.so in-tree: nvcc for sm_100a (-gencode arch=compute_100a,code=sm_100a),
one translation unit per polynomial degree (each with its own __constant__
tables), compiled in parallel, linked with the static CUDA runtime.

    python -m paper_2405_18982_b200.build [--force] [--verbose]
"""
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libipmg.so")
INCLUDE = os.path.join(ROOT, "include")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                  "--expt-relaxed-constexpr", "-I" + INCLUDE, "-I" + CSRC]
CXXFLAGS = ["-O2", "-std=c++17", "-fPIC", "-I" + INCLUDE, "-I" + CSRC, "-I/usr/local/cuda/include"]

SOURCES_CU = (["kernels_k%d.cu" % k for k in range(1, 8)] + ["kernels_dir_k%d.cu" % k for k in range(1, 8)] +
              ["blas.cu", "peak.cu"])
SOURCES_CXX = ["fe1d.cpp", "comm.cpp", "ipmg.cpp"]
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h")))   # every header is a dependency


def _stale(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, log):
    p = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + p.stdout)
    if p.returncode != 0:
        raise RuntimeError("build failed: %s\n%s" % (" ".join(cmd), p.stdout[-4000:]))
    return p.stdout


def build(force=False, verbose=False, jobs=None, defines=(), tag=""):
    """defines: extra -D flags (tuning experiments); tag: build into _build<tag>/ and
    libipmg<tag>.so (load it with IPMG_LIB=...)."""
    obj_dir = OBJ + tag
    lib = LIB if not tag else os.path.join(HERE, "libipmg%s.so" % tag)
    os.makedirs(obj_dir, exist_ok=True)
    cuflags = CUFLAGS + ["-D" + d for d in defines]
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "ipmg.h")]
    tasks = []
    for s in SOURCES_CU:
        src = os.path.join(CSRC, s)
        obj = os.path.join(obj_dir, s + ".o")
        if force or _stale(obj, [src] + hdrs):
            tasks.append(([NVCC] + cuflags + ["-c", src, "-o", obj], obj + ".log"))
    for s in SOURCES_CXX:
        src = os.path.join(CSRC, s)
        obj = os.path.join(obj_dir, s + ".o")
        if force or _stale(obj, [src] + hdrs):
            tasks.append((["g++"] + CXXFLAGS + ["-c", src, "-o", obj], obj + ".log"))
    jobs = jobs or max(1, os.cpu_count() or 1)
    with cf.ThreadPoolExecutor(jobs) as ex:
        outs = list(ex.map(lambda t: _run(*t), tasks))
    if verbose:
        for o in outs:
            sys.stdout.write(o)
    objs = [os.path.join(obj_dir, s + ".o") for s in SOURCES_CU + SOURCES_CXX]
    if force or tasks or _stale(lib, objs):
        _run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", lib] + objs + ["-ldl", "-lpthread"], os.path.join(obj_dir, "link.log"))
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    tags = [a[6:] for a in sys.argv[1:] if a.startswith("--tag=")]
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv, defines=defs,
                tag=tags[0] if tags else ""))
