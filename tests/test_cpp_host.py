"""The C++ host layer (include/absp.hpp) as a reference-style call site: compiled with g++
against libabsp.so and run as a separate process (tests/cpp/test_host_cpp.cpp)."""
from __future__ import annotations

import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CUDA = Path("/usr/local/cuda")


def _compile(tmp_path: Path) -> Path:
    from oracle import oracle as O
    from paper_2605_12110_b200 import build as B
    lib = B.build()
    O.build_oracle()
    gxx = shutil.which("g++") or "/usr/bin/g++"
    exe = tmp_path / "test_host_cpp"
    cmd = [gxx, "-std=c++17", "-O1", "-Wall", "-I", str(ROOT / "include"), "-I", str(CUDA / "include"),
           str(ROOT / "tests" / "cpp" / "test_host_cpp.cpp"), "-o", str(exe),
           "-L", str(lib.parent), "-labsp", "-L", str(ROOT / "oracle"), "-loracle",
           "-L", str(CUDA / "lib64"), "-lcudart",
           f"-Wl,-rpath,{lib.parent}:{ROOT / 'oracle'}:{CUDA / 'lib64'}"]
    subprocess.run(cmd, check=True)
    return exe


def test_cpp_host_layer_cpu(tmp_path):
    exe = _compile(tmp_path)
    r = subprocess.run([str(exe), "cpu", str(tmp_path)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "OK cpu" in r.stdout


@pytest.mark.gpu
def test_cpp_host_layer_gpu(tmp_path):
    exe = _compile(tmp_path)
    r = subprocess.run([str(exe), "gpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "OK gpu" in r.stdout


def _compile_engine(tmp_path: Path) -> Path:
    from oracle import oracle as O
    from paper_2605_12110_b200 import build as B
    lib = B.build()
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    ref_dir = O.LIB_REF.parent
    gxx = shutil.which("g++") or "/usr/bin/g++"
    exe = tmp_path / "test_engine_cpp"
    cmd = [gxx, "-std=c++17", "-O1", "-Wall", "-I", str(ROOT / "include"),
           str(ROOT / "tests" / "cpp" / "test_engine_cpp.cpp"), "-o", str(exe),
           "-L", str(lib.parent), "-labsp", str(O.LIB_REF),
           f"-Wl,-rpath,{lib.parent}:{ref_dir}:{CUDA / 'lib64'}"]
    subprocess.run(cmd, check=True)
    return exe


def test_cpp_engine_compiles(tmp_path):
    """The C++ DecodeEngine call site builds against absp.hpp with g++ and no CUDA headers."""
    from oracle import oracle as O
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    assert _compile_engine(tmp_path).exists()


@pytest.mark.gpu
def test_cpp_engine_vs_reference_engine(tmp_path):
    """absp::DecodeEngine (no PyTorch) against the reference's DecodeEngine over 130 steps:
    store bit-exact after every step, selections equal, outputs in tolerance."""
    exe = _compile_engine(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "OK engine" in r.stdout
