"""TEST INFRASTRUCTURE ONLY. numpy twin of absp_fill_synthetic_bf16 (csrc/synth.cu):
element i of stream s = RNE-bf16( fp32(IrwinHall4(splitmix64(seed + golden*(s<<40 | i) + golden))) * 2.6429e-5 ).
Used to prove the benchmark's device-generated inputs are the bytes the oracle sees."""
from __future__ import annotations

import numpy as np

_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def synth_bf16(count: int, seed: int, stream_id: int, start: int = 0) -> np.ndarray:
    with np.errstate(over="ignore"):
        i = np.arange(start, start + count, dtype=np.uint64)
        z = np.uint64(seed) + _GOLD * ((np.uint64(stream_id) << np.uint64(40)) + i + np.uint64(1))
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    m = np.uint64(0xFFFF)
    s = ((z & m).astype(np.int64) + ((z >> np.uint64(16)) & m).astype(np.int64)
         + ((z >> np.uint64(32)) & m).astype(np.int64) + (z >> np.uint64(48)).astype(np.int64) - 131070)
    f = s.astype(np.float32) * np.float32(2.6429e-05)
    u = f.view(np.uint32).astype(np.uint64)
    u = u + 0x7FFF + ((u >> 16) & 1)
    return (u >> 16).astype(np.uint16)
