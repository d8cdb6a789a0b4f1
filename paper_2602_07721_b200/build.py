"""Build libpariskv.so in-tree with nvcc for sm_100a (B200). No torch involvement.

    python -m paper_2602_07721_b200.build [-v]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
# PKV_LIB_TAG=x builds libpariskv_x.so from build_x/ (experiment variants; the binding loads it with PKV_LIB=x)
_TAG = os.environ.get("PKV_LIB_TAG", "")
OUT = os.path.join(HERE, f"libpariskv_{_TAG}.so" if _TAG else "libpariskv.so")
BUILD = os.path.join(HERE, f"build_{_TAG}" if _TAG else "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", f"-I{os.path.join(ROOT, 'include')}",
         "-Xptxas", "-v", "--expt-relaxed-constexpr"]


# PKV_PHASE_PROFILE=1: compile the globaltimer phase marks in (scripts/phase_profile.py); never for benchmarks
DEFS = ["-DPKV_PHASE_PROFILE"] if os.environ.get("PKV_PHASE_PROFILE") == "1" else []
DEFS += [f"-D{d}" for d in os.environ.get("PKV_BUILD_DEFS", "").split()]  # experiment switches
STAMP = os.path.join(BUILD, "defs.txt")


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _compile(src: str) -> tuple[str, str]:
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    cmd = [NVCC, *ARCH, *FLAGS, *DEFS, "-c", src, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [NVCC, *ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC,-O3", f"-I{os.path.join(ROOT, 'include')}",
               "-x", "cu", "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    try:
        with open(STAMP) as f:
            if f.read() != " ".join(DEFS):
                return False
    except OSError:
        return False
    t = os.path.getmtime(OUT)
    deps = sources() + [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "pariskv.h"),
                                                                              os.path.abspath(__file__)]
    return all(os.path.getmtime(d) <= t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(_compile, sources()))
    if verbose:
        for obj, log in results:
            if log.strip():
                print(f"== {os.path.basename(obj)}\n{log}")
    objs = [o for o, _ in results]
    tmp = OUT + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lnccl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, OUT)
    with open(STAMP, "w") as f:
        f.write(" ".join(DEFS))
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
