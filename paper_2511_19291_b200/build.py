"""Build libtqd.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libtqd.so")
SOURCES = ["kernels.cu", "sweep_f32_fwd.cu", "sweep_f32_bwd.cu", "sweep_f64_fwd.cu", "sweep_f64_bwd.cu",
           "dense_tc.cu", "plan.cpp", "comm.cpp", "abi.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    try:
        import nvidia.nccl as m  # torch's bundled NCCL (the one torch.distributed loads)
        base = list(m.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and glob.glob(os.path.join(lib, "libnccl.so*")):
            return inc, lib
    except Exception:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _inputs():
    files = [os.path.join(CSRC, s) for s in SOURCES]
    files += glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.cpp")) + [os.path.join(ROOT, "include", "tqd.h")]
    return files


def up_to_date() -> bool:
    if not os.path.exists(SO):
        return False
    t = os.path.getmtime(SO)
    return all(os.path.getmtime(f) <= t for f in _inputs())


def build(force: bool = False, verbose: bool = False) -> str:
    """nvcc -c every source in parallel (sm_100a), then link the shared library."""
    if not force and up_to_date():
        return SO
    from concurrent.futures import ThreadPoolExecutor
    inc, lib = _nccl_dirs()
    nccl_so = sorted(glob.glob(os.path.join(lib, "libnccl.so*")))[0]
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    common = ["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
              "-Xcompiler", "-fPIC,-O3", f"-I{inc}"]
    if verbose:
        common.append("-Xptxas=-v")
    common += os.environ.get("TQD_NVCC_EXTRA", "").split()  # experiment knobs, e.g. -DTQD_SWEEP_R=3

    def compile_one(src):
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        cmd = common + ["-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
        if r.returncode != 0 or verbose:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}")
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = SO + f".tmp{os.getpid()}"
    cmd = ["nvcc", *ARCH, "-shared", "-o", tmp, *objs, f"-L{lib}", f"-l:{os.path.basename(nccl_so)}",
           "-Xlinker", f"-rpath,{lib}"]
    subprocess.check_call(cmd, cwd=CSRC)
    os.replace(tmp, SO)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(SO)
