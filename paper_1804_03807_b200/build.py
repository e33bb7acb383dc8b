"""Build libnid.so in-tree for sm_100a.

    python -m paper_1804_03807_b200.build [--jobs J] [--sizes 4,7,10,14]

Compiles csrc/kernels_inst.cu once per system size n = 1..16 (each a fully
unrolled, register-resident instantiation) plus the C-ABI layer, in
parallel, and links them into paper_1804_03807_b200/libnid.so.  Objects go
to build/ (git-ignored); the .so travels to the GPU box with the snapshot.
"""

from __future__ import annotations

import argparse
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "nid")
LIB = os.path.join(PKG, "libnid.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")]
SIZES = list(range(1, 17))
if os.environ.get("NID_PHASE_TIMERS"):
    FLAGS = FLAGS + ["-DNID_PHASE_TIMERS"]
if os.environ.get("NID_LU_UNFUSED"):
    FLAGS = FLAGS + ["-DNID_LU_UNFUSED"]
if os.environ.get("NID_G10"):
    FLAGS = FLAGS + ["-DNID_G10=" + os.environ["NID_G10"]]
    OBJ = OBJ + "_G" + os.environ["NID_G10"]
# experiment variants: extra -D flags, objects in their own directory
# (NID_VARIANT_SIZES="10,...": only those sizes get the variant flags; the
# other sizes link the default objects)
EXTRA = os.environ.get("NID_EXTRA_DEFS", "").split()
OBJ_DEFAULT = OBJ
VARIANT_SIZES = [int(x) for x in os.environ.get("NID_VARIANT_SIZES", "").split(",") if x]
if EXTRA:
    FLAGS_DEFAULT = list(FLAGS)
    FLAGS = FLAGS + EXTRA
    OBJ = OBJ + "_" + "_".join(x.lstrip("-D").replace("=", "") for x in EXTRA)


def _sources():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh", ".h"))] + [
        os.path.join(ROOT, "include", "nid.h")]


def _stale(target: str) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in _sources())


def _run(cmd):
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout)
    return r.stdout


def build(jobs: int | None = None, verbose: bool = False, force: bool = False, out: str | None = None,
          sizes=None) -> str:
    lib = out or LIB
    os.makedirs(OBJ, exist_ok=True)
    jobs = jobs or max(1, min(16, os.cpu_count() or 4))
    cmds = []
    objs = []
    for n in sizes or SIZES:
        variant = not VARIANT_SIZES or n in VARIANT_SIZES
        o = os.path.join(OBJ if variant else OBJ_DEFAULT, f"inst_{n}.o")
        fl = FLAGS if variant or not EXTRA else FLAGS_DEFAULT
        objs.append(o)
        if force or _stale(o):
            os.makedirs(os.path.dirname(o), exist_ok=True)
            cmds.append([NVCC, *ARCH, *fl, f"-DNID_N={n}", "-c", os.path.join(CSRC, "kernels_inst.cu"), "-o", o])
    # the auxiliary tracker kernel (double-double tracking, step traces): always default flags
    for n in sizes or SIZES:
        o = os.path.join(OBJ_DEFAULT, f"aux_{n}.o")
        objs.append(o)
        if force or _stale(o):
            os.makedirs(os.path.dirname(o), exist_ok=True)
            fl = FLAGS_DEFAULT if EXTRA else FLAGS
            cmds.append([NVCC, *ARCH, *fl, f"-DNID_N={n}", "-c", os.path.join(CSRC, "kernels_aux.cu"), "-o", o])
    o = os.path.join(OBJ, "capi.o")
    objs.append(o)
    if force or _stale(o):
        cmds.append([NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, "capi.cu"), "-o", o])
    if cmds:
        with ThreadPoolExecutor(jobs) as ex:
            for out in ex.map(_run, cmds):
                if verbose and out.strip():
                    print(out)
    if cmds or force or not os.path.exists(lib) or any(os.path.getmtime(x) > os.path.getmtime(lib) for x in objs):
        _run([NVCC, *ARCH, "-shared", "-o", lib, *objs, "-lcudart"])
    return lib


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=None)
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    ap.add_argument("--out", default=None, help="library path (experiment variants)")
    a = ap.parse_args()
    print(build(a.jobs, a.v, a.force, a.out))
    sys.exit(0)
