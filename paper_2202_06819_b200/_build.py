"""Build libconvq.so in-tree with nvcc for sm_100a (no torch extension, no JIT).

The kernel instantiations live in sixteen translation units kern_b{8,4}_o{OUT}.cu,
one per (bits, output path) -- packed TMA / s32 / direct stores, ReLU, residual,
unsigned u8 codes --
compiled in parallel, plus the host library convq.cu and the host-only schedule
search search.cpp (NEXT-4); objects are linked into
one shared library with the CUDA runtime linked statically."""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# CONVQ_INSTRUMENT=1: the measurement build (wait-cycle trace + probe modes,
# scripts/trace.py / probe.py) -> libconvq_instr.so, loaded via CONV_Q_LIB
INSTR = os.environ.get("CONVQ_INSTRUMENT") == "1"
_SFX = ("_instr" if INSTR else "") + (f"_wg{os.environ['CONVQ_EPI_WG8']}" if os.environ.get("CONVQ_EPI_WG8") else "") + \
    (f"_wgi4{os.environ['CONVQ_EPI_WG4']}" if os.environ.get("CONVQ_EPI_WG4") else "") + \
    ("_tp" if os.environ.get("CONVQ_TMEM_PIPE") == "1" else "") + \
    ("_la" if os.environ.get("CONVQ_LATE_ACC") == "1" else "") + \
    ("_dual" if os.environ.get("CONVQ_DUAL_MMA") == "1" else "") + \
    ("_allw0" if os.environ.get("CONVQ_EPI_ALLW") == "0" else "")
OBJ = os.path.join(HERE, "build_obj" + _SFX)
LIB = os.path.join(HERE, f"libconvq{_SFX}.so")
SOURCES = ["convq.cu", "search.cpp"] + [f"kern_b{b}_o{o}.cu" for b in (8, 4) for o in (0, 1, 2, 4, 6, 8, 10)] + \
    ["kern_b8_o20.cu", "kern_b8_o22.cu"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden"] + \
    (["-DCONVQ_INSTRUMENT"] if INSTR else []) + \
    ([f"-DCONVQ_EPI_WG8={os.environ['CONVQ_EPI_WG8']}"] if os.environ.get("CONVQ_EPI_WG8") else []) + \
    ([f"-DCONVQ_EPI_WG4={os.environ['CONVQ_EPI_WG4']}"] if os.environ.get("CONVQ_EPI_WG4") else []) + \
    (["-DCONVQ_TMEM_PIPE=1"] if os.environ.get("CONVQ_TMEM_PIPE") == "1" else []) + \
    (["-DCONVQ_LATE_ACC=1"] if os.environ.get("CONVQ_LATE_ACC") == "1" else []) + \
    (["-DCONVQ_DUAL_MMA=1"] if os.environ.get("CONVQ_DUAL_MMA") == "1" else []) + \
    (["-DCONVQ_EPI_ALLW=0"] if os.environ.get("CONVQ_EPI_ALLW") == "0" else [])


def _deps():
    return [os.path.join(CSRC, s) for s in SOURCES] + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "convq.h"), __file__]


def _stale(target, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _compile(src, verbose):
    nvcc = os.environ.get("NVCC", "nvcc")
    obj = os.path.join(OBJ, os.path.splitext(os.path.basename(src))[0] + ".o")
    cmd = [nvcc, *NVCC_FLAGS, *(["-Xptxas", "-v"] if verbose else []), "-I", os.path.join(ROOT, "include"),
           "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-4000:]}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    deps = _deps()
    if not force and not _stale(LIB, deps):
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    # per-object staleness: an object is rebuilt when its source, any header or
    # this script is newer (a host-only change to convq.cu recompiles convq.o only)
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "convq.h"), __file__]

    def obj_of(src):
        return os.path.join(OBJ, os.path.splitext(os.path.basename(src))[0] + ".o")

    todo = [s for s in srcs if force or _stale(obj_of(s), [s] + headers)]
    jobs = max(1, min(len(todo), os.cpu_count() or 1))
    with cf.ThreadPoolExecutor(jobs) as ex:
        built = dict(zip(todo, ex.map(lambda s: _compile(s, verbose), todo)))
    results = [built.get(s, (obj_of(s), "")) for s in srcs]
    if verbose:
        for _, log in results:
            sys.stderr.write(log)
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([nvcc, *ARCH, "-shared", "--cudart", "static", *[o for o, _ in results], "-o", tmp])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
