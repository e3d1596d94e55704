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


def _compile_calib(tmp_path: Path) -> Path:
    from paper_2605_12110_b200 import build as B
    lib = B.build()
    gxx = shutil.which("g++") or "/usr/bin/g++"
    exe = tmp_path / "test_calib_cpp"
    cmd = [gxx, "-std=c++17", "-O1", "-Wall", "-I", str(ROOT / "include"),
           str(ROOT / "tests" / "cpp" / "test_calib_cpp.cpp"), "-o", str(exe),
           "-L", str(lib.parent), "-labsp", f"-Wl,-rpath,{lib.parent}:{CUDA / 'lib64'}"]
    subprocess.run(cmd, check=True)
    return exe


def test_cpp_trace_io_vs_reference(tmp_path):
    """absp_calib.hpp's load_trace / save_trace on a reference-written trace: byte-identical
    round trip, and the reference's error messages (workload.cpp:277-309)."""
    import numpy as np
    from oracle import oracle as O
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    exe = _compile_calib(tmp_path)
    rng = np.random.default_rng(3)
    k = rng.standard_normal((2, 19, 8)).astype(np.float32)
    v = rng.standard_normal((2, 19, 8)).astype(np.float32)
    q = rng.standard_normal((2, 8)).astype(np.float32)
    src, dst = tmp_path / "ref.absp", tmp_path / "cpp.absp"
    O.ref_save_trace(src, k, v, q, seed=77)
    r = subprocess.run([str(exe), "roundtrip", str(src), str(dst)], capture_output=True, text=True, timeout=60)
    assert "OK roundtrip" in r.stdout, r.stdout + r.stderr
    assert dst.read_bytes() == src.read_bytes()
    bad = tmp_path / "bad.absp"
    bad.write_bytes(src.read_bytes() + b"x")
    r = subprocess.run([str(exe), "load", str(bad)], capture_output=True, text=True, timeout=60)
    assert r.stdout.strip() == "error load_trace: trailing bytes after queries section"
    bad.write_bytes(src.read_bytes()[:30])
    r = subprocess.run([str(exe), "load", str(bad)], capture_output=True, text=True, timeout=60)
    assert r.stdout.strip() == "error load_trace: truncated file in section 'header'"


@pytest.mark.gpu
def test_cpp_calibration_vs_reference(tmp_path):
    """absp_calib.hpp's profile_sensitivity / assign_block_sizes / transfer_check (GPU samples)
    on reference-written traces against the reference calibrator: recalls within 1e-9,
    assignment and matched candidate equal."""
    import numpy as np
    from oracle import oracle as O
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    exe = _compile_calib(tmp_path)
    H, d, P, T, n, S, tau = 4, 64, 8, 256, 3000, 2, 0.9
    cands = [8, 16, 32]
    profiles = [("clustered", 2, 48), ("scattered", 20), ("clustered", 4, 16), ("uniform",)]
    ks, vs, qs = [], [], []
    for s in range(S):
        k, v, q = O.ref_generate_synthetic(n, H, d, profiles, seed=100 + s)
        k, v, q = (O.bf16_to_f32(O.f32_to_bf16(x)) for x in (k, v, q))
        O.ref_save_trace(tmp_path / f"s{s}.absp", k, v, q, seed=s)
        ks.append(k)
        vs.append(v)
        qs.append(q)
    k, v, q = np.stack(ks), np.stack(vs), np.stack(qs)
    r = subprocess.run([str(exe), "calib", str(tmp_path), str(S), str(H), str(d), str(P), str(T), str(tau)]
                       + [str(c) for c in cands], capture_output=True, text=True, timeout=300)
    assert "OK calib" in r.stdout, r.stdout + r.stderr
    lines = {ln.split()[0]: ln.split()[1:] for ln in r.stdout.splitlines() if ln}
    got = np.array([float(x) for x in lines["recalls"]]).reshape(H, len(cands))
    want = O.ref_profile_sensitivity(k, v, q, P, cands, T)
    assert np.all(np.abs(got - want) <= 1e-9)
    a = [int(x) for x in lines["assignment"]]
    assert a == O.ref_assign_block_sizes(want, cands, tau)
    tr = [float(x) for x in lines["transfer"]]
    ref = O.ref_transfer_check(a, k, v, q, P, cands, T)
    assert abs(tr[0] - ref["adaptive_recall"]) <= 1e-9 and abs(tr[1] - ref["delta"]) <= 1e-9
    assert int(tr[3]) == ref["matched_candidate"]
    assert np.all(np.abs(np.array(tr[4:]) - np.array(ref["uniform_recalls"])) <= 1e-9)
