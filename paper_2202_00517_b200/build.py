"""Build libknnd.so (sm_100a) in-tree with nvcc.

The library is a plain C ABI (include/knnd.h) with the CUDA runtime linked
statically, so it does not depend on which libcudart torch happens to load.
Objects are rebuilt only when a source or header is newer than the .so.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG_DIR)
CSRC = os.path.join(PKG_DIR, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB_PATH = os.path.join(PKG_DIR, "libknnd.so")
# the checked build (-DKNND_CHECKED: device-side bounds checks, knnd_check_failures),
# used by tests/test_checked.py in place of compute-sanitizer; never by the product
CHECKED_LIB_PATH = os.path.join(PKG_DIR, "libknnd_checked.so")
OBJ_DIR = os.path.join(PKG_DIR, "_obj")

# (the join's kernel families are three translation units so that they compile in parallel)
SOURCES = ["abi.cu", "prep.cu", "csr.cu", "join.cu", "join_f32k2.cu", "join_q23.cu", "rng.cu", "exact.cu"]
HEADERS = ["common.cuh", "score.cuh", "join_impl.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
    f"-I{INCLUDE}",
]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the knnd CUDA library cannot be built")


def _newest_input() -> float:
    paths = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.join(INCLUDE, "knnd.h"), __file__]
    return max(os.path.getmtime(p) for p in paths)


def needs_build(path: str = LIB_PATH) -> bool:
    return not os.path.exists(path) or os.path.getmtime(path) < _newest_input()


def build(force: bool = False, verbose: bool = False, checked: bool = True) -> str:
    """Build libknnd.so (and, unless checked=False, libknnd_checked.so) in-tree."""
    targets = [(LIB_PATH, OBJ_DIR, ())]
    if checked:
        targets.append((CHECKED_LIB_PATH, OBJ_DIR + "_checked", ("-DKNND_CHECKED",)))
    targets = [t for t in targets if force or needs_build(t[0])]
    if not targets:
        return LIB_PATH
    nvcc = nvcc_path()
    for _, obj_dir, _ in targets:
        os.makedirs(obj_dir, exist_ok=True)

    def compile_one(job) -> tuple[str, str]:
        src, obj_dir, extra = job
        obj = os.path.join(obj_dir, src.replace(".cu", ".o"))
        cmd = [nvcc, *NVCC_FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src} {' '.join(extra)}:\n{res.stdout}\n{res.stderr}")
        return obj, res.stderr

    jobs = [(src, obj_dir, extra) for _, obj_dir, extra in targets for src in SOURCES]
    # the join's translation units first (their template instantiations dominate the build), then by size
    jobs.sort(key=lambda j: (not j[0].startswith("join"), -os.path.getsize(os.path.join(CSRC, j[0]))))
    with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as pool:
        results = dict(zip(jobs, pool.map(compile_one, jobs)))
    for lib_path, obj_dir, extra in targets:
        objs = [results[(src, obj_dir, extra)][0] for src in SOURCES]
        tmp = lib_path + ".tmp"
        cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
        os.replace(tmp, lib_path)
        with open(os.path.join(obj_dir, "ptxas.log"), "w") as fh:
            for src in SOURCES:
                fh.write(results[(src, obj_dir, extra)][1])
    if verbose:
        for _, log in results.values():
            sys.stderr.write(log)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
