"""Regenerate tests/golden/golden_v1.npz from the UNMODIFIED reference.

Runs only in the build container (needs oracle/_ref/libabsparse_ref.so, compiled from
/root/reference/proj/src by `make -C oracle ref`). Inputs are not stored: they are
re-created bit-exactly from the integer-only generator in oracle/synth.py, so the
fixture holds only the reference's outputs:

  per case: store (values / codes / scales / zps [+ _min]), estimate_scores of the
  group-summed query, select_topk, the GQA decode outputs (sparse_attention per
  group member) and full_attention_oracle per member.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import RefSeq, bf16_to_f32, group_sum  # noqa: E402
from oracle.synth import synth_bf16  # noqa: E402

# name: (H, G, d, P, block sizes (cycled), seq_len, T, method, bits, mode, key_mode)
CASES = {
    "mean_int4asym": (4, 2, 64, 16, (16, 32, 64), 1000, 256, 0, 4, 1, "rand"),
    "mean_int4sym": (4, 2, 64, 16, (16, 32, 64), 1000, 256, 0, 4, 0, "rand"),
    "mean_int8asym": (4, 2, 64, 16, (16, 32, 64), 1000, 256, 0, 8, 1, "rand"),
    "mean_int2asym": (4, 2, 64, 16, (16, 32, 64), 1000, 256, 0, 2, 1, "rand"),
    "mean_f32": (4, 2, 64, 16, (16, 32, 64), 1000, 256, 0, 0, 1, "rand"),
    "maxmin_int4asym": (4, 2, 64, 16, (16, 32, 64), 1000, 256, 1, 4, 1, "rand"),
    "maxmin_f32": (4, 2, 64, 16, (16, 32, 64), 1000, 256, 1, 0, 1, "rand"),
    "mean_int4asym_d128_g4": (8, 4, 128, 8, (8, 16, 32), 2100, 512, 0, 4, 1, "rand"),
    "ties_constant_keys": (4, 2, 64, 16, (16, 32, 64), 700, 128, 0, 4, 1, "const"),
    "short_seq_le_budget": (4, 2, 64, 16, (16, 32, 64), 200, 256, 0, 4, 1, "rand"),
    "single_token": (4, 1, 64, 16, (16, 32, 64), 1, 64, 0, 4, 1, "rand"),
    "p4_small_blocks": (4, 8, 64, 4, (4, 8, 16, 32), 900, 128, 0, 4, 1, "rand"),
}
SEED = 42


def case_inputs(name: str):
    """Deterministic inputs of a case: bf16 pools [H][pages][P][d], page table, q [H*G][d]."""
    H, G, d, P, cands, n, T, method, bits, mode, key_mode = CASES[name]
    pages = (n + P - 1) // P
    pool_pages = pages + 2
    sid = sum(ord(c) for c in name) * 16
    k = synth_bf16(H * pool_pages * P * d, SEED, sid + 0).reshape(H, pool_pages, P, d)
    if key_mode == "const":
        k = np.full_like(k, 0x3F80)  # 1.0 everywhere: every centroid and score ties
    v = synth_bf16(H * pool_pages * P * d, SEED, sid + 1).reshape(H, pool_pages, P, d)
    q = synth_bf16(H * G * d, SEED, sid + 2).reshape(H * G, d)
    # a fixed scatter of the pages: page i of the sequence lives at physical (7*i + 3) % pool_pages
    pt = ((7 * np.arange(pages) + 3) % pool_pages).astype(np.uint32)
    assert len(set(pt.tolist())) == pages
    bs = [cands[h % len(cands)] for h in range(H)]
    return dict(H=H, G=G, d=d, P=P, n=n, T=T, method=method, bits=bits, mode=mode, block_sizes=bs,
                k_pool=k, v_pool=v, page_table=pt, q=q)


def logical(pool, pt, n, P):
    t = np.arange(n)
    return np.ascontiguousarray(bf16_to_f32(pool[:, pt[t // P], t % P, :]))


def main() -> None:
    out = {}
    for name in CASES:
        c = case_inputs(name)
        keys = logical(c["k_pool"], c["page_table"], c["n"], c["P"])
        vals = logical(c["v_pool"], c["page_table"], c["n"], c["P"])
        r = RefSeq(keys, vals, c["P"], c["block_sizes"], c["method"], c["bits"], c["mode"])
        st = r.store()
        for k_, v_ in st.items():
            out[f"{name}/{k_}"] = v_
        out[f"{name}/offsets"] = r.offsets
        qf = bf16_to_f32(c["q"])
        qs = group_sum(qf, c["H"], c["G"])
        sc = r.scores(qs)
        out[f"{name}/scores"] = sc
        sel = r.select(sc, c["T"])
        out[f"{name}/sel_counts"] = np.array([len(s) for s in sel], np.uint32)
        out[f"{name}/sel_blocks"] = np.concatenate(sel).astype(np.uint32)
        out[f"{name}/attn_out"] = r.decode_gqa(qf, c["G"], c["T"])
        fulls = np.zeros_like(qf)
        for g in range(c["G"]):
            fulls.reshape(c["H"], c["G"], -1)[:, g] = r.full_attention(
                np.ascontiguousarray(qf.reshape(c["H"], c["G"], -1)[:, g]))
        out[f"{name}/full_out"] = fulls
    dst = Path(__file__).with_name("golden_v1.npz")
    np.savez_compressed(dst, **out)
    print(f"wrote {dst} ({dst.stat().st_size} bytes, {len(CASES)} cases)")


if __name__ == "__main__":
    main()
