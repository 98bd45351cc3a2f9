"""Build tool libraries (not on the hot path): FP64 peak probe, microbenchmarks."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def build(force=False):
    out = os.path.join(HERE, "libpeak.so")
    src = os.path.join(HERE, "peak.cu")
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-Xcompiler", "-fPIC",
                               "-shared", "-o", out, src])
    mb = os.path.join(HERE, "microbench")
    msrc = os.path.join(HERE, "microbench.cu")
    if force or not os.path.exists(mb) or os.path.getmtime(mb) < os.path.getmtime(msrc):
        subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", mb, msrc])
    return out


def dfma_rate(reps=5):
    import ctypes
    lib = ctypes.CDLL(build())
    lib.tool_dfma_rate.restype = ctypes.c_double
    lib.tool_dfma_rate.argtypes = [ctypes.c_int]
    return lib.tool_dfma_rate(reps)
