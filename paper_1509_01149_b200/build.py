"""Build paper_1509_01149_b200/libmppi_b200.so with nvcc for sm_100a (in-tree, so the built
library travels to the GPU box with the repo snapshot).

cudart is linked statically (nvcc 12.9 here, torch ships a 12.8 runtime); the library shares
the device's primary context with torch, so torch-allocated pointers and streams work as-is.
"""
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmppi_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "-cudart", "static",
         "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def nccl_include():
    """nccl.h of the NCCL torch ships (types only; the library resolves NCCL at run time)."""
    try:
        import nvidia.nccl
        d = os.path.join(list(nvidia.nccl.__path__)[0], "include")
        if os.path.exists(os.path.join(d, "nccl.h")):
            return d
    except Exception:
        pass
    return "/usr/include"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + \
        sorted(glob.glob(os.path.join(CSRC, "*.h"))) + [os.path.join(ROOT, "include", "mppi.h")]


def _elf_text_sections(blob):
    """{name: bytes} of the .text.* sections (machine code) of an ELF64 image."""
    import struct
    shoff, = struct.unpack_from("<Q", blob, 0x28)
    shentsize, shnum, shstrndx = struct.unpack_from("<HHH", blob, 0x3A)
    secs = []
    for i in range(shnum):
        name, typ, flags, addr, off, size = struct.unpack_from("<IIQQQQ", blob, shoff + i * shentsize)
        secs.append((name, off, size))
    stroff = secs[shstrndx][1]
    out = {}
    for name, off, size in secs:
        end = blob.index(b"\0", stroff + name)
        nm = blob[stroff + name:end].decode()
        if nm.startswith(".text."):
            out[nm] = blob[off:off + size]
    return out


def source_hash(lib=None):
    """sha256 of the rollout kernels' machine code: the .text sections (SASS bytes, no line tables
    or paths) of every rollout_kernel* in the sm_100a cubin compiled from mppi_kernels.cu, extracted
    from libmppi_b200.so with cuobjdump.  The key that ties a committed ncu capture
    (profiles/roofline_constants.json: per-sample-step instruction, FLOP and byte counts of the
    rollout kernels) to the code it measured: host-only changes leave it unchanged, any change to
    a kernel's instructions moves it."""
    import hashlib
    import shutil
    import tempfile
    lib = lib or LIB
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    with tempfile.TemporaryDirectory() as d:
        name = "mppi_kernels.sm_100a.cubin"
        r = subprocess.run([cuobjdump, "-xelf", name, lib], cwd=d, capture_output=True, text=True)
        path = os.path.join(d, name)
        if r.returncode != 0 or not os.path.exists(path):
            raise RuntimeError("cuobjdump -xelf failed: " + r.stderr[-300:])
        with open(path, "rb") as f:
            blob = f.read()
    h = hashlib.sha256()
    for nm, code in sorted(_elf_text_sections(blob).items()):
        if "rollout_kernel" in nm:          # the kernels the constants describe
            h.update(nm.encode())
            h.update(code)
    return h.hexdigest()[:16]


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in deps())


def build(force=False, verbose=False, out=None, defines=()):
    """Build the library (out/defines: an experimental variant, e.g. -DMPPI_X2_MINB=3)."""
    lib = out or LIB
    if not force and out is None and up_to_date():
        return LIB
    tmp = lib + ".tmp%d" % os.getpid()
    cmd = [NVCC] + ARCH + FLAGS + list(defines) + ["-I", os.path.join(ROOT, "include"), "-I", CSRC,
                                                   "-I", nccl_include(), "-shared", "-o", tmp] + sources() + ["-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libmppi_b200.so")
    if out is None:
        with open(os.path.join(HERE, "ptxas_report.txt"), "w") as f:
            f.write(r.stderr)
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    defs = [a for a in args if a.startswith("-D")] + [a[len("--flag="):] for a in args if a.startswith("--flag=")]
    outs = [a[len("--out="):] for a in args if a.startswith("--out=")]
    print(build(force=True, verbose="-v" in args, out=outs[0] if outs else None, defines=defs))
