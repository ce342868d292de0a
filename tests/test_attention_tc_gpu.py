"""GPU parity of the tcgen05 decode-attention kernel (attention_tc.cu) against the CPU oracle.

attend_tc_kernel serves the packed groups of D = 128, gs = 32 caches with 2/3/4-bit Keys,
2/4-bit Values and up to four query rows per KV head; the window launch of attend_mma_kernel
merges its partials. Every case asserts the tcgen05 kernel ran, and compares with the fp64
evaluation over the bit-exact snapshot (tolerances of test_attention_gpu.py), covering:
stream-K splits of a (b, kv-head) across CTAs, tiles with 1-3 valid groups, more CTAs than
tiles, GQA G = 2 / 4 in one pass, several query tokens, forced accumulator folds, fp16 windows,
and the fused append (kvmix_append_attend) over many decode steps.
"""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2506_08018_b200 as K
from test_attention_gpu import ATTN_TOL_F64, CHECKSUM_RTOL, abs_score_sum, build

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def tc_on():
    K.set_knob("KVMIX_TC", 1)
    yield
    K.set_knob("KVMIX_TC", 0)
    K.set_knob("KVMIX_TEST_FLUSH_BLOCKS", 0)


def run(dev, ora, q, G=1, expect_tc=True):
    ks, vs = ora.snapshot()
    B, Hq, t, D = q.shape
    qr = q.reshape(B, Hq // G, G * t, D) if G > 1 else q
    o64, cs64 = O.attend_f64(qr, ks, vs)
    o64 = o64.reshape(q.shape)
    n0 = K.launch_count_of("attend_tc_kernel")
    res = K.attend(torch.from_numpy(q).cuda(), dev)
    ran = K.launch_count_of("attend_tc_kernel") - n0
    assert (ran > 0) == expect_tc, f"attend_tc_kernel launches: {ran}"
    out = res.output.cpu().numpy()
    err = float(np.abs(out - o64).max()) / float(np.abs(vs).max())
    assert err <= ATTN_TOL_F64, err
    l1 = abs_score_sum(q, ks, G)
    assert abs(res.scores_checksum - cs64) <= CHECKSUM_RTOL * l1 + 1e-9, (res.scores_checksum, cs64)
    return err


@pytest.mark.parametrize("kb,vb", [(2, 2), (3, 4), (4, 4), (2, 4), (4, 2), (3, 2)])
@pytest.mark.parametrize("groups", [1, 3, 4, 6, 13, 64])
def test_tc_tiers_and_partial_tiles(cuda, kb, vb, groups):
    """Fast-group counts that are / are not multiples of the 4-group tile."""
    T = groups * 32 + 40
    dev, ora = build(kb, vb, 0.05, 0.05, 32, 2, 3, 128, [T] + [1] * 3, seed=kb * 10 + vb + groups, cap=T + 64)
    run(dev, ora, O.random_h16(groups, (2, 3, 1, 128)))


@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("kb,vb", [(2, 2), (3, 4)])
def test_tc_gqa_one_pass(cuda, G, kb, vb):
    dev, ora = build(kb, vb, 0.1, 0.1, 32, 2, 2, 128, [1500] + [1] * 5, seed=G * 31 + kb, cap=1600)
    run(dev, ora, O.random_h16(G + 70, (2, 2 * G, 1, 128)), G=G)


def test_tc_several_query_tokens(cuda):
    dev, ora = build(2, 2, 0.1, 0.1, 32, 1, 4, 128, [900], seed=5, cap=1000)
    run(dev, ora, O.random_h16(81, (1, 4, 2, 128)))
    run(dev, ora, O.random_h16(82, (1, 4, 4, 128)))


def test_tc_rows_beyond_four_use_the_imma_path(cuda):
    dev, ora = build(2, 2, 0.1, 0.1, 32, 1, 2, 128, [600], seed=6, cap=700)
    run(dev, ora, O.random_h16(83, (1, 2, 5, 128)), expect_tc=False)


@pytest.mark.parametrize("flush", [4, 8])
def test_tc_forced_folds(cuda, flush):
    """Accumulator folds every flush/4 tiles (the int32 overflow guard path)."""
    K.set_knob("KVMIX_TEST_FLUSH_BLOCKS", flush)
    dev, ora = build(2, 4, 0.1, 0.1, 32, 1, 2, 128, [3000], seed=flush, cap=3100)
    run(dev, ora, O.random_h16(84, (1, 2, 1, 128), sigma=3.0))


def test_tc_scale_ramp_moves_the_max(cuda):
    """Scores that keep growing along the context move the lazy reference max many times."""
    B, H, D, T = 1, 2, 128, 2048
    ramp = np.linspace(0.1, 6.0, T, dtype=np.float32)[None, None, :, None]
    k = (O.random_h16(1, (B, H, T, D)) * ramp).astype(np.float16).astype(np.float32)
    v = O.random_h16(2, (B, H, T, D))
    dev = K.KVLayerCache(K.LayerQuantConfig(0, 2, 2, 0.1, 0.1, 32), B, H, D, capacity_tokens=T + 16)
    ora = O.CacheOracle(2, 2, 0.1, 0.1, 32, B, H, D)
    dev.append(k, v)
    ora.append(k, v)
    q = O.random_h16(3, (B, H, 1, D))
    run(dev, ora, q)


def test_tc_fused_append_decode_steps(cuda):
    """kvmix_append_attend over 70 decode steps (Key-group age-outs included) vs the oracle."""
    B, H, D = 2, 4, 128
    dev, ora = build(3, 4, 0.2, 0.2, 32, B, H, D, [1000], seed=9, cap=1200, tail_dtype=torch.float16)
    worst = 0.0
    for s in range(70):
        k1 = O.random_h16(500 + 2 * s, (B, H, 1, D))
        v1 = O.random_h16(501 + 2 * s, (B, H, 1, D))
        q = O.random_h16(900 + s, (B, H, 1, D))
        n0 = K.launch_count_of("attend_tc_kernel")
        res = K.append_attend(dev, torch.from_numpy(k1).cuda().half(), torch.from_numpy(v1).cuda().half(),
                              torch.from_numpy(q).cuda())
        assert K.launch_count_of("attend_tc_kernel") > n0
        ora.append(k1, v1)
        if s % 7 == 0 or s == 69:
            ks, vs = ora.snapshot()
            o64, _ = O.attend_f64(q, ks, vs)
            worst = max(worst, float(np.abs(res.output.cpu().numpy() - o64).max()) / float(np.abs(vs).max()))
    assert dev.dump() == ora.dump()
    assert worst <= ATTN_TOL_F64, worst


def test_tc_matches_imma_path_closely(cuda):
    """Both tensor-core formulations agree far inside the tolerance (same fixed point)."""
    dev, ora = build(2, 2, 0.1, 0.1, 32, 4, 8, 128, [2500] + [1] * 20, seed=12, cap=2600)
    q = torch.from_numpy(O.random_h16(85, (4, 8, 1, 128))).cuda()
    a = K.attend(q, dev).output
    K.set_knob("KVMIX_TC", 0)
    b = K.attend(q, dev).output
    K.set_knob("KVMIX_TC", 1)
    _, vs = ora.snapshot()
    assert float((a - b).abs().max()) / float(np.abs(vs).max()) < 1e-6
