"""Build paper_1509_01149_b200/libmppi_probe.so (FP32 peak probe and the BM32 sweep probe, sm_100a)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRCS = [os.path.join(HERE, "probe", "fp32_probe.cu"), os.path.join(HERE, "probe", "bm32_probe.cu")]
NOISE = os.path.join(HERE, "csrc", "noise.cuh")
LIB = os.path.join(HERE, "libmppi_probe.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def build(force=False):
    hdr = os.path.join(ROOT, "include", "mppi_probe.h")
    if not force and os.path.exists(LIB) and all(
            os.path.getmtime(p) <= os.path.getmtime(LIB) for p in SRCS + [hdr, NOISE]):
        return LIB
    tmp = LIB + ".tmp%d" % os.getpid()
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-Xcompiler",
           "-fPIC", "-cudart", "static", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(HERE, "csrc"), "-shared", "-o", tmp] + SRCS
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


def bm32(kind, packed, first, count, out0, out1=None):
    """mppi_probe_bm32 on device tensors (see include/mppi_probe.h)."""
    import ctypes as C
    L = C.CDLL(build())
    L.mppi_probe_bm32.argtypes = [C.c_int, C.c_int, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p]
    rc = L.mppi_probe_bm32(int(kind), int(packed), int(first), int(count), out0.data_ptr(),
                           out1.data_ptr() if out1 is not None else None)
    if rc:
        raise RuntimeError("mppi_probe_bm32 failed: %d" % rc)


if __name__ == "__main__":
    print(build(force=True))
