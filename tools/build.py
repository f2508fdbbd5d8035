"""Build libgeot.so (and the synth generator library) for sm_100a, in-tree.

    python tools/build.py [--force] [-j N]

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo, one object per
translation unit compiled in parallel, then a shared-library link.  Objects go
to build/ (git-ignored); the .so files land next to their Python loaders so
they travel to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))  # repo root (tools/..)
PKG = os.path.join(ROOT, "paper_2404_03019_b200")
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
                  "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]

LIBGEOT = os.path.join(PKG, "libgeot.so")
LIBSYNTH = os.path.join(ROOT, "synth", "libgeot_synth.so")


def _newest(paths):
    return max((os.path.getmtime(p) for p in paths if os.path.exists(p)), default=0.0)


def _compile(src, obj, deps, extra, force):
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= _newest([src] + deps):
        return obj, False
    os.makedirs(os.path.dirname(obj), exist_ok=True)
    cmd = [NVCC] + NVFLAGS + extra + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj, True


def _link(out, objs, force):
    if not force and os.path.exists(out) and os.path.getmtime(out) >= _newest(objs):
        return False
    tmp = out + f".tmp{os.getpid()}"
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-cudart=static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed for {out}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, out)
    return True


def build(force: bool = False, jobs: int | None = None, verbose: bool = True) -> list[str]:
    jobs = jobs or max(1, min(16, os.cpu_count() or 1))
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(CSRC, "*.inc")) + [os.path.join(ROOT, "include", "geot.h")]
    units = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    tasks = []
    with cf.ThreadPoolExecutor(jobs) as ex:
        for u in units:
            obj = os.path.join(BUILD, "geot", os.path.basename(u) + ".o")
            extra = ["-x", "cu"] if u.endswith(".cpp") else []
            tasks.append(ex.submit(_compile, u, obj, headers, extra, force))
        ssrc = os.path.join(ROOT, "synth", "csrc", "synth.cu")
        sobj = os.path.join(BUILD, "synth", "synth.cu.o")
        stask = ex.submit(_compile, ssrc, sobj, [], [], force)
        objs = [t.result()[0] for t in tasks]
        so = stask.result()[0]
    built = []
    if _link(LIBGEOT, objs, force):
        built.append(LIBGEOT)
    if _link(LIBSYNTH, [so], force):
        built.append(LIBSYNTH)
    if verbose and built:
        print("built:", ", ".join(os.path.relpath(b, ROOT) for b in built), file=sys.stderr)
    return [LIBGEOT, LIBSYNTH]


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    a = ap.parse_args()
    build(force=a.force, jobs=a.j)
