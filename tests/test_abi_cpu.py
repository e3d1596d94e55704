"""CPU-side checks of the drop-in boundary: libabsp.so loads, exports every entry point
include/absp.h declares, validates configs with the reference's semantics, and fails
loudly (no CPU fallback) when no GPU is present."""
import ctypes as C
import re
from pathlib import Path

import pytest

from oracle import oracle as O
from paper_2605_12110_b200 import _abi
from paper_2605_12110_b200.absparse import EngineConfig, QuantSpec

HEADER = Path(__file__).resolve().parents[1] / "include" / "absp.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:absp_status|int|const char\*|uint64_t)\s+(absp_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _abi.load()
    syms = declared_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_abi.EXPORTED)
    assert lib.absp_abi_version() == 1


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(_abi.LIB_PATH)], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def _cfg(**kw):
    base = dict(num_heads=8, head_dim=128, page_size=16, candidate_block_sizes=(16, 32, 64), token_budget=2048,
                quant=QuantSpec(4), num_q_heads=32, max_batch=16, max_seq_len=131072)
    base.update(kw)
    return EngineConfig(**base)


CASES = [
    dict(),
    dict(num_heads=0),
    dict(page_size=0),
    dict(candidate_block_sizes=()),
    dict(candidate_block_sizes=(16, 24)),
    dict(candidate_block_sizes=(32, 16)),
    dict(candidate_block_sizes=(16, 16)),
    dict(token_budget=32),
    dict(quant=QuantSpec(3)),
]


@pytest.mark.parametrize("kw", CASES)
def test_config_validation_matches_reference(kw):
    cfg = _cfg(**kw)
    try:
        cfg.validate()
        mine = None
    except _abi.InvalidArgument as e:
        mine = str(e)
    if O.ref_available():
        L = O.ref()
        cands = (C.c_size_t * max(1, len(cfg.candidate_block_sizes)))(*cfg.candidate_block_sizes)
        rc = L.ref_config_validate(cfg.num_heads, cfg.head_dim, cfg.page_size, cands,
                                   len(cfg.candidate_block_sizes), cfg.token_budget,
                                   cfg.quant.bits if cfg.quant else 0)
        theirs = L.ref_last_error().decode() if rc else None
        assert (rc == 0) == (mine is None)
        if rc:
            assert rc == 1  # std::invalid_argument
            assert mine == theirs
    else:
        assert (mine is None) == (kw == {})


def test_gpu_build_limits():
    with pytest.raises(_abi.InvalidArgument):
        _cfg(head_dim=96).validate()
    with pytest.raises(_abi.InvalidArgument):
        _cfg(num_q_heads=36).validate()
    with pytest.raises(_abi.InvalidArgument):
        _cfg(candidate_block_sizes=(16, 256), token_budget=4096).validate()


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2605_12110_b200 import DecodeAttention
    with pytest.raises(_abi.CudaError):
        DecodeAttention(_cfg())
    from paper_2605_12110_b200 import BlockAssignment, DecodeEngine
    with pytest.raises(_abi.CudaError):  # the engine object has no CPU path either
        DecodeEngine(_cfg(max_batch=1), BlockAssignment.cycled(8, (16, 32, 64)), 4096)
