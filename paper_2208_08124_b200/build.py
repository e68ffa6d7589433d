"""Build libub.so (sm_100a) in-tree with nvcc.  `python -m paper_2208_08124_b200.build`."""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(HERE, "libub.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir() -> str:
    import nvidia.nccl  # torch-bundled NCCL (headers + libnccl.so.2)
    return os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]


def _cublas_dir() -> str:
    """cuBLASLt for the encoder's plain GEMMs: the torch-bundled copy (the one torch itself
    loads into the process), else the toolkit's."""
    try:
        import nvidia.cublas
        d = os.path.join(list(nvidia.cublas.__path__)[0], "lib")
        if os.path.exists(os.path.join(d, "libcublasLt.so.12")):
            return d
    except ImportError:
        pass
    return "/usr/local/cuda/lib64"


def _flags():
    nccl = _nccl_dir()
    return nccl, ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
                  "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(nccl, "include")] + ARCH


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _headers():
    return glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "ub.h")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, trace: bool = False, variant: str = "",
          defines=()) -> str:
    """trace=True builds libub_trace.so with -DUB_TRACE (debug timelines; not the product).
    variant="x", defines=["A=1"] builds libub_x.so with -DA=1 (dev A/B experiments only)."""
    tag = "trace" if trace else variant
    build_dir = BUILD + ("_" + tag if tag else "")
    lib = LIB.replace("libub.so", f"libub_{tag}.so") if tag else LIB
    os.makedirs(build_dir, exist_ok=True)
    nccl, flags = _flags()
    if trace:
        flags = flags + ["-DUB_TRACE"]
    flags = flags + ["-D" + d for d in defines]
    hdrs = _headers()
    jobs = []
    objs = []
    for src in _sources():
        obj = os.path.join(build_dir, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + hdrs):
            jobs.append([NVCC] + flags + ["-c", src, "-o", obj])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        if verbose:
            sys.stderr.write(r.stdout + r.stderr)
        return r

    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(lib, objs):
        nccl_lib = os.path.join(nccl, "lib")
        # export only the C ABI (ub_*): visibility=hidden + explicit default in ub.h users
        blas_lib = _cublas_dir()
        cmd = [NVCC] + ARCH + ["-shared", "-o", lib] + objs + [
            "-L" + nccl_lib, "-l:libnccl.so.2", "-L" + blas_lib, "-l:libcublasLt.so.12", "-lcudart",
            "-Xlinker", "-rpath," + nccl_lib, "-Xlinker", "-rpath," + blas_lib,
            "-Xlinker", "--version-script=" + os.path.join(CSRC, "exports.map")]
        run(cmd)
    return lib


if __name__ == "__main__":
    var = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")]
    defs = [a[2:] for a in sys.argv if a.startswith("-D")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, trace="--trace" in sys.argv,
                variant=var[0] if var else "", defines=defs))
