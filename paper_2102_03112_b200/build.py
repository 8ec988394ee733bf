"""Builds the in-tree CUDA library libgradpack_b200.so for sm_100a.

    python -m paper_2102_03112_b200.build        (or __graft_entry__.build())

One nvcc invocation per translation unit, then a shared link.  The library
exports only the C-ABI of include/gradpack_b200.h.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libgradpack_b200.so")
OBJ = os.path.join(HERE, "build_obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills"]
SOURCES = ["capi.cu", "topr.cu", "container.cu", "indexcodec.cu", "values.cu", "bloom.cu", "p2.cu", "p1.cu", "rle.cu", "sort.cu", "values_fit.cu", "values_quant.cu", "huffman.cu", "inflate.cu", "dense.cu", "topr64.cu", "deflate.cu", "volume.cpp", "dp_exchange.cpp"]


def _run(cmd):
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout)
        raise RuntimeError(f"command failed: {' '.join(cmd)}")
    return r.stdout


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    objs = []
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp"))]
    deps.append(os.path.join(HERE, "..", "include", "gradpack_b200.h"))
    newest_dep = max(os.path.getmtime(p) for p in deps)
    stale = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(OBJ, src.rsplit(".", 1)[0] + ".o")
        if (not os.path.exists(obj) or os.path.getmtime(obj) < os.path.getmtime(path)
                or os.path.getmtime(obj) < newest_dep):
            stale.append([NVCC, *ARCH, *FLAGS, "-c", path, "-o", obj])
        objs.append(obj)
    with ThreadPoolExecutor(max_workers=max(1, min(len(stale), os.cpu_count() or 1))) as pool:
        for out in pool.map(_run, stale):  # one nvcc per translation unit, in parallel
            if verbose and out.strip():
                print(out)
    if not os.path.exists(OUT) or any(os.path.getmtime(o) > os.path.getmtime(OUT) for o in objs):
        _run([NVCC, *ARCH, "-shared", "-o", OUT, *objs, "-Xlinker", "--exclude-libs,ALL"])
    build_cli()
    build_inputs()
    return OUT


def build_inputs() -> str:
    """libgp_inputs.so: the host generator of the benchmark gradients (inputs.py)."""
    src = os.path.join(CSRC, "inputs.c")
    out = os.path.join(HERE, "libgp_inputs.so")
    if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        _run(["gcc", "-std=c11", "-O2", "-fPIC", "-shared", "-ffp-contract=off", src, "-o", out, "-lm"])
    return out


CLI_SRC = os.path.join(HERE, "..", "tests", "cpp", "gp_cli.cpp")
CLI_OUT = os.path.join(HERE, "..", "tests", "cpp", "gp_cli")


CPP_TESTS = ["gp_cli", "dp_test"]  # tests/cpp/<name>.cpp → tests/cpp/<name>


def build_cli() -> str:
    """The C++ host programs over include/gradpack_b200.h(pp) (tests/test_gpu_cpp*.py)."""
    hdrs = [os.path.join(HERE, "..", "include", h) for h in ("gradpack_b200.hpp", "gradpack_b200.h")]
    for name in CPP_TESTS:
        src = os.path.join(HERE, "..", "tests", "cpp", name + ".cpp")
        out = os.path.join(HERE, "..", "tests", "cpp", name)
        if (os.path.exists(out) and all(os.path.getmtime(out) > os.path.getmtime(p) for p in [src, OUT, *hdrs])):
            continue
        _run(["g++", "-std=c++17", "-O2", "-pthread", "-I/usr/local/cuda/include", src, "-o", out, f"-L{HERE}",
              "-lgradpack_b200", "-L/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{HERE}",
              "-Wl,-rpath,/usr/local/cuda/lib64"])
    return CLI_OUT


if __name__ == "__main__":
    print(build(verbose=True))
