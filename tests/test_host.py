"""Host-side mirror of the reference API (no GPU): assignment file format, quant spec
names, offsets, and the multi-GPU unit sharding."""
import numpy as np
import pytest

from oracle.oracle import lib
from paper_2605_12110_b200 import BlockAssignment, EngineConfig, InvalidArgument, QuantMode, QuantSpec, build_offsets
from paper_2605_12110_b200.sharding import shard_units


def test_quant_spec_names_roundtrip():
    for bits in (2, 4, 8):
        for mode in QuantMode:
            s = QuantSpec(bits, mode)
            assert QuantSpec.parse(s.name) == s
    assert QuantSpec.parse("int4xasym") == QuantSpec(4, QuantMode.ASYMMETRIC)
    with pytest.raises(InvalidArgument):
        QuantSpec.parse("int3xasym")


def test_build_offsets_matches_oracle():
    rng = np.random.default_rng(99)
    for _ in range(20):
        H = 1 + int(rng.integers(6))
        bs = [int(rng.choice([16, 32, 64])) for _ in range(H)]
        n = int(rng.integers(500))
        out = np.zeros(H + 1, np.uint64)
        lib().absp_oracle_offsets(n, np.array(bs, np.uint32), H, out)
        assert build_offsets(n, BlockAssignment(bs)) == out.tolist()


def test_assignment_file(tmp_path):
    """read/write_assignment_file semantics (calibrator.cpp:277-311)."""
    p = tmp_path / "assignment.txt"
    BlockAssignment([16, 64, 32]).save(p)
    assert p.read_text() == "0 16\n1 64\n2 32\n"
    p.write_text("0 16\n\n1 64\n2 32\n")
    a = BlockAssignment.load(p)
    assert a.block_sizes == [16, 64, 32]
    cfg = EngineConfig(num_heads=3)
    a.validate(cfg)
    with pytest.raises(InvalidArgument):
        BlockAssignment([16, 48, 32]).validate(cfg)
    for bad in ("0 16\n0 32\n", "1 16\n", "0 16 7\n", "", "0 x\n", "# c\n0 16\n"):
        p.write_text(bad)
        with pytest.raises(RuntimeError):
            BlockAssignment.load(p)
    with pytest.raises(RuntimeError):
        BlockAssignment.load(tmp_path / "missing.txt")


@pytest.mark.parametrize("batch,heads,world", [(16, 8, 1), (16, 8, 2), (16, 8, 8), (64, 8, 8), (1, 8, 8), (1, 8, 2), (3, 8, 2)])
def test_shard_units_partition(batch, heads, world):
    seen = {}
    for r in range(world):
        s = shard_units(batch, heads, world, r)
        for b in range(s.batch_start, s.batch_start + s.batch_count):
            for h in range(s.head_start, s.head_start + s.head_count):
                seen[(b, h)] = seen.get((b, h), 0) + 1
    assert seen == {(b, h): 1 for b in range(batch) for h in range(heads)}
