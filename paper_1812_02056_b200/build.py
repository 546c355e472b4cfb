"""Build libstepfact.so in-tree with nvcc for sm_100a (B200).  No GPU needed to build."""
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libstepfact.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir():
    """The NCCL that torch itself loads (nvidia-nccl wheel, libnccl.so.2: same soname, so one
    copy per process), else the system one."""
    if os.environ.get("SF_NCCL_DIR"):
        return os.environ["SF_NCCL_DIR"]
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        return list(spec.submodule_search_locations)[0]
    return "/usr"


NCCL_DIR = _nccl_dir()
NCCL_INC = os.path.join(NCCL_DIR, "include")
NCCL_LIB = os.path.join(NCCL_DIR, "lib") if NCCL_DIR != "/usr" else "/usr/lib/x86_64-linux-gnu"
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr",
         "-Xptxas", "-v"]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    return hs + [os.path.join(ROOT, "include", "stepfact.h")]


def stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in sources() + headers())


def build(force=False, verbose=False):
    if not force and not stale():
        return LIB
    os.makedirs(os.path.join(PKG, "build"), exist_ok=True)

    newest_header = max(os.path.getmtime(h) for h in headers())

    def compile_one(src):
        obj = os.path.join(PKG, "build", os.path.basename(src) + ".o")
        # incremental: an object newer than its source and every header is reused
        if not force and os.path.exists(obj) and os.path.getmtime(obj) > max(os.path.getmtime(src), newest_header):
            return src, obj, subprocess.CompletedProcess([], 0, "", "")
        cmd = [NVCC, *ARCH, *[f for f in FLAGS if f != "-shared"], "-c",
               "-I", os.path.join(ROOT, "include"), "-I", NCCL_INC, "-o", obj, src]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, r

    from concurrent.futures import ThreadPoolExecutor
    objs = []
    with ThreadPoolExecutor(max_workers=max(1, min(8, os.cpu_count() or 1))) as ex:
        for src, obj, r in ex.map(compile_one, sources()):
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            if verbose:
                sys.stderr.write(r.stderr)
            objs.append(obj)
    cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", LIB, *objs, "-lcudart_static", "-ldl", "-lrt", "-lpthread",
           "-L" + NCCL_LIB, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + NCCL_LIB]
    subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
