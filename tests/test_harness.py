"""bench-memory / bench-attention drivers: the reference's synthetic stream
and CSV schema over the device caches."""
import io

import numpy as np
import pytest

import oracle as O
import paper_2506_08018_b200 as K
from paper_2506_08018_b200 import harness as Hn


def test_rng_stream_matches_reference():
    """kvmix::Rng + round_through_half == the oracle's random_h16 (same splitmix64 stream)."""
    for seed, shape in ((1, (1, 4, 7, 32)), (1234, (2, 3, 5, 64)), (99, (1, 1, 1, 2))):
        got = Hn.random_kv_tensor(Hn.Rng(seed), *shape)
        assert np.array_equal(got.view(np.uint32), O.random_h16(seed, shape).view(np.uint32))
    r = Hn.Rng(7)
    a = [r.uniform_int(1, 128) for _ in range(5)]
    assert all(1 <= x <= 128 for x in a)


def test_csv_schema():
    rep = K.MemoryReport(1, 2, 3, 6, 12, 2.0)
    s = io.StringIO()
    Hn.write_memory_csv(s, [Hn.BenchMemoryRow(0, 0, rep), Hn.BenchMemoryRow(-1, 0, rep)])
    assert s.getvalue().splitlines()[0] == "layer,step,payload_bits,metadata_bits,tail_bits,ratio,manifest"
    assert s.getvalue().splitlines()[2] == "-1,0,1,2,3,2,manifest.json"
    s = io.StringIO()
    Hn.write_attention_csv(s, [Hn.AttentionTrialRow(2, 0, 0.5, 0.25, 10.0, 20.0)])
    assert s.getvalue().splitlines() == ["bits,trial,mse_vs_fp,fused_ref_maxdev,fused_us,reference_us,manifest",
                                         "2,0,0.5,0.25,10,20,manifest.json"]


@pytest.mark.gpu
def test_bench_memory_rows_match_oracle(cuda):
    cfg = K.tiered_config(4, 1)
    opt = Hn.BenchMemoryOptions(batch=1, heads=2, head_dim=64, prefill=300, decode_steps=40, seed=3, emit_every=16)
    rows = Hn.bench_memory(cfg, opt)
    oras = [O.CacheOracle(l.key_bits, l.value_bits, l.key_rpc_ratio, l.value_rpc_ratio, l.group_size, 1, 2, 64)
            for l in cfg.layers]
    rng = Hn.Rng(3)
    for o in oras:
        o.append(Hn.random_kv_tensor(rng, 1, 2, 300, 64), Hn.random_kv_tensor(rng, 1, 2, 300, 64))
    expect = {}
    for step in range(0, 41):
        if step:
            for o in oras:
                o.append(Hn.random_kv_tensor(rng, 1, 2, 1, 64), Hn.random_kv_tensor(rng, 1, 2, 1, 64))
        if step % 16 == 0 or step == 40:
            for l, o in enumerate(oras):
                expect[(l, step)] = o.memory_usage()
    got = {(r.layer, r.step): r.report for r in rows if r.layer >= 0}
    assert set(got) == set(expect)
    for key, m in expect.items():
        assert got[key].total_bits == m["total_bits"] and got[key].tail_bits == m["tail_bits"], key
    agg = [r for r in rows if r.layer == -1]
    assert len(agg) == len({s for _, s in expect}) and agg[-1].step == 40


@pytest.mark.gpu
def test_bench_attention_monotone(cuda):
    rows = Hn.bench_attention(Hn.BenchAttentionOptions(trials=3, seed=1, heads=4, head_dim=64, tokens=512))
    assert len(rows) == 9
    mse = {b: np.mean([r.mse_vs_fp for r in rows if r.bits == b]) for b in (2, 3, 4)}
    assert mse[2] >= mse[3] >= mse[4] > 0
    # elementwise relative deviation (the reference's column): near-zero outputs dominate it;
    # the stated tolerance (max|V|-scaled, test_attention_gpu.py) is checked there
    assert max(r.fused_ref_maxdev for r in rows) < 1e-2
