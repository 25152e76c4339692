"""Build libdvc.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2601_20564_b200.build [--force]
    python -m paper_2601_20564_b200.build --experiments OUT.so   # A/B build: honours DVC_* knobs

The product library ignores every DVC_* environment variable; only an --experiments build
(-DDVC_EXPERIMENTS, written elsewhere than libdvc.so) reads the timing/debug knobs.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SO = os.path.join(PKG, "libdvc.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "-I", os.path.join(ROOT, "include"),
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "dvc.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, jobs: int = 8, experiments: str | None = None) -> str:
    so = SO
    extra = []
    if experiments:
        so, extra = os.path.abspath(experiments), ["-DDVC_EXPERIMENTS"]
    elif not force and not _stale():
        return SO
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    objdir = os.path.join(PKG, "build_exp" if experiments else "build")
    os.makedirs(objdir, exist_ok=True)
    objs, procs = [], []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        cmd = [nvcc, *NVCC_FLAGS, *extra, "-Xptxas", "-v" if verbose else "-O3", "-dc" if False else "-c", src, "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        if len(procs) >= jobs:
            _drain(procs, verbose)
    _drain(procs, verbose)
    link = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", so + ".tmp", *objs, "-ldl"]
    subprocess.check_call(link)
    os.replace(so + ".tmp", so)
    return so


def _drain(procs, verbose):
    while procs:
        cmd, p = procs.pop(0)
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out)
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
        if verbose and out:
            sys.stderr.write(out)


if __name__ == "__main__":
    exp = sys.argv[sys.argv.index("--experiments") + 1] if "--experiments" in sys.argv else None
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, experiments=exp))
