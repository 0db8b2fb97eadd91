"""Build the tgp C-ABI shared library (libtgp.so) in-tree for sm_100a.

    python -m paper_2004_09910_b200.build        (or __graft_entry__.build())

nvcc cross-compiles without a GPU.  The CUDA runtime is linked statically and the driver API is
resolved at run time (cudaGetDriverEntryPoint), so the .so loads on a machine without a driver.
"""
import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(os.path.dirname(HERE), "include")
OUT = os.path.join(HERE, "libtgp.so")
OBJ = os.path.join(os.path.dirname(HERE), "build", "obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I", CSRC, "-I", INC, "-Xptxas", "-v"] if os.environ.get("TGP_PTXAS_V") else \
        ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-I", CSRC, "-I", INC]

SOURCES = ["plan.cpp", "runtime.cu", "kernels_ew.cu", "kernels_ln.cu", "gemm_simt.cu", "gemm_tc.cu", "task_stream.cu", "gemm_dw.cu", "gemm_dw_sgd.cu", "kernels_attn.cu", "gemm_wide.cu"]


def _deps_hash(src):
    h = hashlib.sha1()
    for f in sorted(os.listdir(CSRC)):
        if f.endswith((".h", ".cuh", ".inc")) or f == src:
            h.update(open(os.path.join(CSRC, f), "rb").read())
    h.update(open(os.path.join(INC, "tgp.h"), "rb").read())
    h.update(" ".join(FLAGS + ARCH).encode())
    return h.hexdigest()[:16]


def _compile(src):
    obj = os.path.join(OBJ, src + "." + _deps_hash(src) + ".o")
    if os.path.exists(obj):
        return obj
    for f in os.listdir(OBJ):  # drop stale objects of this source
        if f.startswith(src + ".") and f.endswith(".o"):
            os.remove(os.path.join(OBJ, f))
    cmd = [NVCC] + ARCH + FLAGS + ["-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    if os.environ.get("TGP_PTXAS_V"):
        sys.stderr.write(r.stderr)
    return obj


def build(verbose=True):
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    tmp = OUT + ".tmp"
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lrt", "-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, OUT)
    if verbose:
        print(f"built {OUT}")
    return OUT


if __name__ == "__main__":
    build()
