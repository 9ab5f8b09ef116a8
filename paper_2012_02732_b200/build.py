"""In-tree build of libsw_b200.so (planner C++ + runtime/kernels CUDA for sm_100a).

    python -m paper_2012_02732_b200.build          # incremental
    python -m paper_2012_02732_b200.build --force  # rebuild everything

Objects go to build/ (git-ignored); the shared library lands next to this
file so it travels to the GPU box with the repo snapshot.  nvcc
cross-compiles sm_100a without a GPU.  cudart is linked statically so the
library also loads (planner only) on a CPU-only host.
"""

from __future__ import annotations

import argparse
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
BUILD = os.path.join(ROOT, "build")
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsw_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CXX_FLAGS = ["-std=c++17", "-O3", "-fPIC", "-Wall", "-I", os.path.join(ROOT, "include")]
NVCC_FLAGS = ["-std=c++17", "-O3", "-lineinfo", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
              "-Xptxas", "-v,-warn-spills", "-I", os.path.join(ROOT, "include"), *ARCH]


def sources():
    out = []
    for sub in ("planner", "runtime", "kernels"):
        d = os.path.join(CSRC, sub)
        if not os.path.isdir(d):
            continue
        for fn in sorted(os.listdir(d)):
            if fn.endswith((".cpp", ".cu")):
                out.append(os.path.join(d, fn))
    return out


def headers():
    hs = [os.path.join(ROOT, "include", f) for f in os.listdir(os.path.join(ROOT, "include"))]
    for sub in ("planner", "runtime", "kernels"):
        d = os.path.join(CSRC, sub)
        if os.path.isdir(d):
            hs += [os.path.join(d, f) for f in os.listdir(d) if f.endswith((".h", ".cuh"))]
    return hs


def _run(cmd, log):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        log.write(" ".join(cmd) + "\n" + r.stdout + r.stderr + "\n")
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:6])} ...")


def build(force: bool = False, verbose: bool = False, probe: bool = False) -> str:
    """Build libsw_b200.so; ``probe=True`` builds the diagnostic variant
    libsw_b200_probe.so (-DSW_PROBE: kernel phase stamps, tools/phase_probe.py)."""
    BUILD = os.path.join(ROOT, "build", "probe") if probe else os.path.join(ROOT, "build")
    LIB = os.path.join(PKG, "libsw_b200_probe.so") if probe else globals()["LIB"]
    extra = ["-DSW_PROBE"] if probe else []
    os.makedirs(BUILD, exist_ok=True)
    newest_header = max(os.path.getmtime(h) for h in headers())
    objs = []
    log = open(os.path.join(BUILD, "build.log"), "a")
    jobs = []
    for src in sources():
        rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
        obj = os.path.join(BUILD, rel + ".o")
        objs.append(obj)
        stale = force or not os.path.exists(obj) or \
            os.path.getmtime(obj) < max(os.path.getmtime(src), newest_header)
        if not stale:
            continue
        if src.endswith(".cu"):
            cmd = [NVCC, *NVCC_FLAGS, *extra, "-c", src, "-o", obj]
        else:
            cmd = ["g++", *CXX_FLAGS, *extra, "-c", src, "-o", obj]
        jobs.append(cmd)
    # compile in parallel
    procs = []
    for cmd in jobs:
        if verbose:
            print(" ".join(cmd))
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                            text=True)))
    failed = []
    for cmd, p in procs:
        out, _ = p.communicate()
        log.write(" ".join(cmd) + "\n" + out + "\n")
        if p.returncode != 0:
            failed.append((cmd, out))
    if failed:
        for cmd, out in failed:
            sys.stderr.write(out)
        raise RuntimeError(f"{len(failed)} compile step(s) failed; see build/build.log")
    if jobs or force or not os.path.exists(LIB) or \
            any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        link = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-lcuda" if False else "-ldl"]
        _run(link, log)
    log.close()
    return LIB


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("--probe", action="store_true", help="diagnostic build with kernel phase stamps")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose, probe=a.probe))


if __name__ == "__main__":
    main()
