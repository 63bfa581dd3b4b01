"""Build helpers for the three native libraries (used by __graft_entry__.build()
and lazily by the Python wrappers / tests).

  bqgen/libbqgen.so                        — input generators (gcc)
  oracle/liboracle.so                      — the CPU oracle + std::sort ref (g++)
  paper_1604_06697_b200/libbq.so           — the CUDA path + C-ABI (nvcc, sm_100a)

Every build is an explicit compiler call producing an in-tree .so, so the
artefact travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")

GEN_SRC = [os.path.join(ROOT, "bqgen", "bqgen.c")]
GEN_SO = os.path.join(ROOT, "bqgen", "libbqgen.so")
ORACLE_SRC = [os.path.join(ROOT, "oracle", "bq_oracle.cpp"),
              os.path.join(ROOT, "oracle", "stdsort_ref.cpp")]
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
BQ_DIR = os.path.join(ROOT, "paper_1604_06697_b200")
BQ_SO = os.path.join(BQ_DIR, "libbq.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "-I", os.path.join(ROOT, "include"),
]


def _bq_sources():
    return sorted(glob.glob(os.path.join(BQ_DIR, "csrc", "*.cu")))


def _bq_deps():
    return (_bq_sources() + glob.glob(os.path.join(BQ_DIR, "csrc", "*.cuh"))
            + glob.glob(os.path.join(ROOT, "include", "*.h")))


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed: " + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r


def build_gen(force=False):
    if force or _stale(GEN_SO, GEN_SRC):
        _run(["gcc", "-O2", "-shared", "-fPIC", "-o", GEN_SO] + GEN_SRC)
    return GEN_SO


def build_oracle(force=False):
    if force or _stale(ORACLE_SO, ORACLE_SRC):
        _run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", ORACLE_SO] + ORACLE_SRC)
    return ORACLE_SO


def build_bq(force=False, verbose_ptxas=False, out=None, extra=()):
    srcs = _bq_sources()
    target = out or BQ_SO
    if not (force or _stale(target, _bq_deps())):
        return target
    flags = list(NVCC_FLAGS) + os.environ.get("BQ_NVCC_EXTRA", "").split() + list(extra)
    if verbose_ptxas:
        flags += ["-Xptxas", "-v"]
    objdir = os.path.join(ROOT, "build", "obj" if out is None else "obj_" + os.path.basename(target))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    # compile translation units in parallel (each kernel family is its own .cu)
    procs = []
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        objs.append(o)
        procs.append((s, subprocess.Popen([NVCC] + flags + ["-c", s, "-o", o],
                                          stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    logs = []
    for s, p in procs:
        out, err = p.communicate()
        logs.append(err)
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {s}\n{out}\n{err}")
    tmp = target + ".tmp"
    _run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp] + objs)
    os.replace(tmp, target)
    if verbose_ptxas:
        return "\n".join(logs)
    return target


def build_all(force=False):
    build_gen(force)
    build_oracle(force)
    build_bq(force)


if __name__ == "__main__":
    import sys
    print(build_bq(force=True, verbose_ptxas="-v" in sys.argv) if "bq" in sys.argv else build_all(True))
