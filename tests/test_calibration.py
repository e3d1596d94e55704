"""Trace I/O (workload.cpp:260-309) and the host side of calibration (calibrator.cpp:116-249)
against the unmodified reference (oracle/_ref), CPU only: byte-identical trace files both
ways, the reference's load errors, the Eq.-2 assignment rule, normalized recall, report and
top-k page recall."""
import numpy as np
import pytest

from oracle.oracle import (RefError, ref_assign_block_sizes, ref_available, ref_load_trace, ref_save_trace,
                           ref_write_min_block_csv, ref_write_recall_csv)
from paper_2605_12110_b200 import (InvalidArgument, RecallTable, Trace, assign_block_sizes, load_trace,
                                   make_report, normalized_recall, save_trace, topk_page_recall,
                                   topk_page_recall_per_head, write_min_block_csv, write_recall_csv)

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


def _trace(rng, H=3, n=37, d=16, seed=11):
    k = rng.standard_normal((H, n, d)).astype(np.float32)
    v = rng.standard_normal((H, n, d)).astype(np.float32)
    q = rng.standard_normal((H, d)).astype(np.float32)
    k[0, 0, 0] = -0.0
    v[1, 2, 3] = np.float32(np.inf)
    return Trace(H, d, n, seed, k, v, q)


@needs_ref
def test_trace_files_identical_to_reference(tmp_path):
    t = _trace(np.random.default_rng(1))
    ours, theirs = tmp_path / "ours.absp", tmp_path / "ref.absp"
    save_trace(t, ours)
    ref_save_trace(theirs, t.keys, t.values, t.queries, seed=t.seed)
    assert ours.read_bytes() == theirs.read_bytes()
    k, v, q, seed = ref_load_trace(ours)  # the reference reads our file
    assert seed == t.seed
    assert np.array_equal(k.view(np.uint32), t.keys.view(np.uint32))
    assert np.array_equal(q.view(np.uint32), t.queries.view(np.uint32))
    back = load_trace(theirs)  # we read the reference's file
    assert back == t
    assert back.keys.size == t.keys.size


@needs_ref
@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"ABSQ" + b[4:], "load_trace: format error, bad magic bytes"),
    (lambda b: b[:4] + (2).to_bytes(4, "little") + b[8:], "load_trace: version mismatch (file 2, expected 1)"),
    (lambda b: b + b"\x00", "load_trace: trailing bytes after queries section"),
    (lambda b: b[:-3], "load_trace: truncated file in section 'queries'"),
    (lambda b: b[:10], "load_trace: truncated file in section 'header'"),
    (lambda b: b[:8] + (0).to_bytes(4, "little") + b[12:], "load_trace: dimension inconsistency in header"),
])
def test_trace_errors_match_reference(tmp_path, mutate, msg):
    t = _trace(np.random.default_rng(2))
    good = tmp_path / "good.absp"
    save_trace(t, good)
    bad = tmp_path / "bad.absp"
    bad.write_bytes(mutate(good.read_bytes()))
    with pytest.raises(RuntimeError) as ours:
        load_trace(bad)
    with pytest.raises(RefError) as theirs:
        ref_load_trace(bad)
    assert str(ours.value) == msg
    assert theirs.value.kind == "runtime_error" and str(theirs.value).endswith(msg)


@needs_ref
@pytest.mark.parametrize("tau", [0.5, 0.9, 0.95, 0.99, 1.0, 1.5])
def test_assign_block_sizes_matches_reference(tau):
    rng = np.random.default_rng(int(tau * 100))
    cands = [4, 8, 16, 32, 64]
    rec = np.sort(rng.uniform(0.2, 1.0, (16, len(cands))), axis=1)[:, ::-1].copy()
    rec[3, 2] = rec[3, 0] * tau  # exactly at the threshold (>= keeps it)
    table = RecallTable(16, cands, rec, 4)
    assert assign_block_sizes(table, tau).block_sizes == ref_assign_block_sizes(rec, cands, tau)
    rep = make_report(table, tau)
    assert rep.min_block_sizes == rep.assignment.block_sizes
    assert np.allclose(normalized_recall(table).recalls[:, 0], 1.0)


def test_calibration_host_errors():
    with pytest.raises(InvalidArgument):
        assign_block_sizes(RecallTable(0, [], np.zeros((0, 0)), 0), 0.9)
    with pytest.raises(InvalidArgument):
        assign_block_sizes(RecallTable(1, [16, 8], np.ones((1, 2)), 1), 0.9)
    with pytest.raises(InvalidArgument):
        assign_block_sizes(RecallTable(1, [8, 16], np.zeros((1, 2)), 1), 0.9)
    assert topk_page_recall_per_head([[1, 2, 3], [5]], [[1, 2], [4]]) == [1.0, 0.0]
    assert topk_page_recall([[1, 2, 3], [5]], [[1, 2], [4]]) == 0.5
    with pytest.raises(InvalidArgument):
        topk_page_recall([[1]], [[]])


@needs_ref
def test_csv_reports_identical_to_reference(tmp_path):
    rng = np.random.default_rng(9)
    cands = [8, 16, 32, 64]
    rec = rng.uniform(0.0, 1.0, (5, 4))
    rec[0, 0], rec[1, 1], rec[2, 2] = 1.0, 1.0 / 3.0, 1e-12
    table = RecallTable(5, cands, rec, 3)
    write_recall_csv(tmp_path / "ours.csv", table, "0")
    ref_write_recall_csv(tmp_path / "ref.csv", rec, cands, "0")
    assert (tmp_path / "ours.csv").read_bytes() == (tmp_path / "ref.csv").read_bytes()
    sizes = [8, 64, 16, 32, 8]
    write_min_block_csv(tmp_path / "ours_m.csv", sizes, "layer3")
    ref_write_min_block_csv(tmp_path / "ref_m.csv", sizes, "layer3")
    assert (tmp_path / "ours_m.csv").read_bytes() == (tmp_path / "ref_m.csv").read_bytes()
