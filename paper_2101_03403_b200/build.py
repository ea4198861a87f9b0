"""Build libcvm_b200.so in-tree (sm_100a only), plus the test/oracle helpers.

    python -m paper_2101_03403_b200.build            # product library
    python -m paper_2101_03403_b200.build --all      # + oracle (+ oracle/_ref)

nvcc cross-compiles for sm_100a without a GPU.  Objects go to _build/, the
shared library to _lib/ (both git-ignored; the .so travels to the GPU box).
"""
import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libcvm_b200.so")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# (#pragma unroll in the shared __host__ __device__ FFT header is device-only)
HOST_FLAGS = ["-O2", "-fPIC", "-ffp-contract=off", "-fvisibility=hidden", "-Wall",
              "-Wno-unknown-pragmas"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++20", "-Xptxas", "-v",
                     "--expt-relaxed-constexpr",
                     "-Xcompiler", ",".join(HOST_FLAGS)]
# developer instrumentation builds only (e.g. CVM_NVCC_EXTRA=-DCVM_PHASE_PROF)
NVCC_FLAGS += os.environ.get("CVM_NVCC_EXTRA", "").split()
CXX_FLAGS = ["-std=c++20"] + HOST_FLAGS + ["-I/usr/local/cuda/include"]

SOURCES = ["blind_rotate.cu", "blind_rotate_v4.cu", "key_switch.cu", "device_misc.cu", "context.cu", "keys.cpp",
           "backend.cpp", "schedule.cpp", "clear_backend.cpp", "dag.cpp", "capi.cpp"]
HEADERS = ["tfhe_params.h", "fft512.cuh", "fft512w.cuh", "br_common.cuh", "schedule.hpp", "sm100.cuh", "kernels.cuh", "cvm_internal.hpp"]


def _newer(src_list, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in src_list)


def _compile(src):
    path = os.path.join(CSRC, src)
    obj = os.path.join(BUILD, src + ".o")
    deps = [path] + [os.path.join(CSRC, h) for h in HEADERS] + \
        [os.path.join(REPO, "include", "cvm_gpu.h")]
    if not _newer(deps, obj):
        return obj, ""
    if src.endswith(".cu"):
        cmd = [NVCC] + NVCC_FLAGS + ["-c", path, "-o", obj]
    else:
        cmd = [shutil.which("g++") or "g++"] + CXX_FLAGS + ["-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(verbose=False):
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(_compile, SOURCES))
    objs = [o for o, _ in results]
    if verbose:
        for o, log in results:
            if log:
                print(f"--- {os.path.basename(o)}\n{log}")
    if _newer(objs, LIB):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


def build_oracle(with_ref=True):
    """Test infrastructure: the CPU oracle and, when /root/reference exists, the
    reference core + golden driver (oracle/_ref)."""
    subprocess.run(["make", "-s", "-C", os.path.join(REPO, "oracle")], check=True)
    if with_ref and os.path.isdir("/root/reference/proj/core/src"):
        subprocess.run(["make", "-s", "-C", os.path.join(REPO, "oracle"), "ref"], check=True)
        # the cryptovm::Backend shim + demo over the reference's own ALU/emulator
        subprocess.run(["make", "-s", "-C", os.path.join(REPO, "integration")], check=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--all", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(verbose=a.verbose))
    if a.all:
        build_oracle()


if __name__ == "__main__":
    sys.exit(main())
