"""Build paper_1509_01149_b200/libmppi_probe.so (FP32 peak probe, sm_100a)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "probe", "fp32_probe.cu")
LIB = os.path.join(HERE, "libmppi_probe.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def build(force=False):
    hdr = os.path.join(ROOT, "include", "mppi_probe.h")
    if not force and os.path.exists(LIB) and all(
            os.path.getmtime(p) <= os.path.getmtime(LIB) for p in (SRC, hdr)):
        return LIB
    tmp = LIB + ".tmp%d" % os.getpid()
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-Xcompiler",
           "-fPIC", "-cudart", "static", "-I", os.path.join(ROOT, "include"), "-shared", "-o", tmp, SRC]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libmppi_probe.so")
    os.replace(tmp, LIB)
    return LIB


def probe(packed, blocks=148 * 8, threads=256, iters=4096):
    import ctypes as C
    L = C.CDLL(build())
    L.mppi_probe_fp32.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double),
                                  C.POINTER(C.c_double)]
    tf, ms = C.c_double(), C.c_double()
    rc = L.mppi_probe_fp32(int(packed), blocks, threads, iters, C.byref(tf), C.byref(ms))
    if rc:
        raise RuntimeError("mppi_probe_fp32 failed: cuda error %d" % rc)
    return tf.value, ms.value


if __name__ == "__main__":
    print(build(force=True))
