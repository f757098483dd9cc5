"""The C ABI used from plain C (examples/cartpole_mpc.c): compiled with gcc against
include/mppi.h and libmppi_b200.so, no Python in the loop.  Config C2's receding-horizon
cart-pole must swing the pole up."""
import os
import shutil
import subprocess

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_example_swings_up(tmp_path):
    gcc = shutil.which("gcc") or shutil.which("cc")
    if gcc is None:
        pytest.skip("no C compiler")
    from paper_1509_01149_b200 import build
    lib = build.build()
    exe = str(tmp_path / "cartpole_mpc")
    libdir = os.path.dirname(lib)
    subprocess.run([gcc, "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "examples", "cartpole_mpc.c"),
                    "-L", libdir, "-lmppi_b200", "-Wl,-rpath," + libdir, "-lm", "-o", exe], check=True)
    r = subprocess.run([exe, "200"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    fields = r.stdout.split()
    final = float(fields[fields.index("1+cos(theta)") + 1])
    mean_q = float(fields[fields.index("q") + 1])
    assert final < 0.05, r.stdout          # upright at the end of 4 s (hanging = 2)
    assert mean_q < 1000.0, r.stdout
