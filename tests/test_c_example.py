"""The C ABI used from plain C (examples/solve_c1.c): no Python, no PyTorch on
the call path.  CPU: it compiles and links against libms2g.so.  GPU: it runs a
C1-shaped solve and reduces the data residual."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _build(tmp_path):
    from paper_2203_07308_b200 import build as B
    B.build()
    exe = str(tmp_path / "solve_c1")
    libdir = os.path.join(ROOT, "paper_2203_07308_b200")
    cmd = ["gcc", "-O2", "-std=c99", "-D_DEFAULT_SOURCE", os.path.join(ROOT, "examples", "solve_c1.c"),
           f"-I{os.path.join(ROOT, 'include')}", f"-I{CUDA}/include", f"-L{libdir}", "-lms2g",
           f"-L{CUDA}/lib64", "-lcudart", "-lm", f"-Wl,-rpath,{libdir}", "-o", exe]
    subprocess.check_call(cmd)
    return exe


def test_c_example_links(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run(["ldd", exe], capture_output=True, text=True).stdout
    assert "libms2g.so" in out


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    exe = _build(tmp_path)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "steps 20" in res.stdout and "residual" in res.stdout
