"""GPU parity: decode attention over the packed cache vs the CPU oracle.

Tolerance (stated): elementwise relative error is meaningless for
near-zero outputs at long contexts, so errors are scaled by max|V|:
  * primary, vs an fp64 evaluation over the reference's bit-exact snapshot:
        max |out - out64| <= ATTN_TOL_F64 * max|V|
  * secondary, vs the reference's own fp32 attend order (oracle attend_f32):
        max |out - out32| <= ATTN_TOL_F32 * max|V|
  * scores_checksum: |delta| <= CHECKSUM_RTOL * sum_j |score_j| (the checksum is a signed
    sum of ~B*H*t*T scores, so its error scales with the L1 norm, not with the sum).
"""
import threading

import numpy as np
import pytest
import torch

import oracle as O
import paper_2506_08018_b200 as K

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["tc", "ws", "single"])
def tc_kernel(request):
    """Every parity test runs on the three tensor-core paths: tcgen05 over the packed groups
    (default where it applies: D = 128, gs = 32, 2/4-bit Values, <= 4 query rows), the
    warp-specialized IMMA kernel and the single-warp IMMA kernel."""
    K.set_knob("KVMIX_TC", 1 if request.param == "tc" else 0)
    K.set_knob("KVMIX_WS", {"tc": 1, "ws": 2, "single": 0}[request.param])
    yield request.param
    K.set_knob("KVMIX_TC", 0)
    K.set_knob("KVMIX_WS", 1)

ATTN_TOL_F64 = 2e-6
ATTN_TOL_F32 = 4e-6
CHECKSUM_RTOL = 2e-7


def build(kb, vb, rk, rv, gs, B, H, D, chunks, seed=0, tail_dtype=torch.float32, cap=None):
    cap = cap or sum(chunks) + 16
    dev = K.KVLayerCache(K.LayerQuantConfig(0, kb, vb, rk, rv, gs), B, H, D, capacity_tokens=cap, tail_dtype=tail_dtype)
    ora = O.CacheOracle(kb, vb, rk, rv, gs, B, H, D)
    for i, t in enumerate(chunks):
        k = O.random_h16(seed + 2 * i, (B, H, t, D))
        v = O.random_h16(seed + 2 * i + 1, (B, H, t, D))
        dev.append(k, v)
        ora.append(k, v)
    return dev, ora


def abs_score_sum(q, ks, G=1):
    B, Hq, t, D = q.shape
    qr = q.reshape(B, Hq // G, G * t, D).astype(np.float64)
    return float(np.abs(np.einsum("bhtd,bhjd->bhtj", qr, ks.astype(np.float64))).sum() / np.sqrt(D))


def check_attend(dev, ora, q, G=1, expect_mma=None):
    ks, vs = ora.snapshot()
    l1 = abs_score_sum(q, ks, G)
    if G > 1:  # GQA: KV head h serves query heads h*G .. h*G+G-1 (= reference t=G rows)
        B, Hq, t, D = q.shape
        qr = q.reshape(B, Hq // G, G * t, D)
        o64, cs64 = O.attend_f64(qr, ks, vs)
        o32, cs32 = O.attend_f32(qr, ks, vs)
        o64, o32 = o64.reshape(q.shape), o32.reshape(q.shape)
    else:
        o64, cs64 = O.attend_f64(q, ks, vs)
        o32, cs32 = O.attend_f32(q, ks, vs)
    n_mma, n_gen = K.tensor_core_launches(), K.launch_count_of("attend_generic_kernel")
    res = K.attend(torch.from_numpy(q).cuda(), dev)
    out = res.output.cpu().numpy()
    used_mma = K.tensor_core_launches() - n_mma
    used_gen = K.launch_count_of("attend_generic_kernel") - n_gen
    assert (used_mma > 0) != (used_gen > 0)  # one path serves the call (the IMMA path in passes of rows)
    if expect_mma is not None:
        assert (used_mma > 0) == bool(expect_mma), "tensor-core path expected" if expect_mma else "generic path expected"
    vmax = float(np.abs(vs).max())
    e64 = float(np.abs(out - o64).max()) / vmax
    e32 = float(np.abs(out - o32).max()) / vmax
    assert e64 <= ATTN_TOL_F64, e64
    assert e32 <= ATTN_TOL_F32, e32
    assert abs(res.scores_checksum - cs64) <= CHECKSUM_RTOL * l1 + 1e-9, (res.scores_checksum, cs64, l1)
    return e64


@pytest.mark.parametrize("kb,vb", [(2, 2), (3, 4), (4, 4), (3, 3), (2, 4), (4, 2), (2, 3), (4, 3)])
def test_attend_fill_states(cuda, kb, vb):
    rng = np.random.default_rng(kb * 7 + vb)
    for trial in range(4):
        r = float(rng.uniform(0.0, 0.5))
        chunks = [int(x) for x in rng.integers(1, 96, size=int(rng.integers(1, 8)))]
        dev, ora = build(kb, vb, r, r, 32, 1, 2, 64, chunks, seed=trial * 100)
        q = O.random_h16(999 + trial, (1, 2, 1 + trial % 3, 64))
        check_attend(dev, ora, q)


@pytest.mark.parametrize("sigma", [1.0, 3.0])
def test_attend_long_context_config1(cuda, sigma):
    """Config 1: B1, H32, D128, K2/V2 gs32 r=0.1, 4096 tokens (prefill + decode steps)."""
    dev, ora = build(2, 2, 0.1, 0.1, 32, 1, 32, 128, [4032] + [1] * 64, seed=7, cap=4200)
    q = O.random_h16(5, (1, 32, 1, 128), sigma=sigma)
    check_attend(dev, ora, q, expect_mma=True)


def test_attend_right_after_prefill(cuda):
    dev, ora = build(2, 2, 0.1, 0.1, 32, 1, 8, 128, [4096], seed=3, cap=4200)
    assert dev.key_tail_tokens() == 416 and dev.value_tail_tokens() == 409
    check_attend(dev, ora, O.random_h16(6, (1, 8, 1, 128)), expect_mma=True)


def test_attend_mixed_tier_fp16(cuda):
    dev, ora = build(3, 4, 0.2, 0.2, 32, 2, 4, 128, [2000] + [1] * 40, seed=11, tail_dtype=torch.float16)
    q = O.random_h16(8, (2, 4, 1, 128))
    check_attend(dev, ora, q, expect_mma=True)
    # fp16 queries give the same result as their fp32 copy
    a = K.attend(torch.from_numpy(q).cuda(), dev).output
    b = K.attend(torch.from_numpy(q).cuda().half(), dev).output
    assert torch.equal(a, b)


@pytest.mark.parametrize("G", [2, 4, 8])
def test_attend_gqa(cuda, G):
    """GQA: G query heads per KV head run as passes of two query rows over the cache."""
    dev, ora = build(2, 2, 0.1, 0.1, 32, 2, 4, 128, [1500] + [1] * 33, seed=21)
    q = O.random_h16(12, (2, 4 * G, 1, 128), sigma=2.0)
    check_attend(dev, ora, q, G=G, expect_mma=True)


@pytest.mark.parametrize("kb,vb,G,tq", [(3, 4, 2, 1), (4, 2, 4, 1), (2, 4, 1, 3), (2, 2, 4, 5), (3, 2, 2, 5), (4, 4, 8, 3)])
def test_attend_multi_pass_rows(cuda, kb, vb, G, tq):
    """More than two query rows per KV head (GQA and/or several query tokens): row passes
    (two rows per pass, 3-bit Keys included) inside one launch, up to 8 per launch (20 rows: two
    launches), a last pass with one row, checksums summed over the passes."""
    dev, ora = build(kb, vb, 0.2, 0.2, 32, 1, 4, 128, [900] + [1] * 12, seed=27)
    q = O.random_h16(28, (1, 4 * G, tq, 128), sigma=1.5)
    check_attend(dev, ora, q, G=G, expect_mma=True)


@pytest.mark.parametrize("kb,vb,G,tq,D", [(2, 2, 4, 1, 128), (3, 4, 4, 1, 128), (4, 2, 2, 2, 128), (2, 4, 4, 1, 64),
                                          (3, 2, 3, 1, 128), (4, 4, 8, 1, 64)])
def test_four_row_passes_match_two_row_passes(cuda, kb, vb, G, tq, D):
    """Four query rows per pass (two IMMA column tiles over one unpacked A fragment, the
    default for > 2 rows) against the two-row passes (KVMIX_R4 = 0) on the same cache: both
    within the fp64 tolerance, and within 4e-7 max|V| of each other (only the fp32 merge and
    min-term summation orders differ)."""
    dev, ora = build(kb, vb, 0.2, 0.2, 32, 2, 2, D, [700] + [1] * 9, seed=61)
    q = O.random_h16(62, (2, 2 * G, tq, D), sigma=1.5)
    outs = []
    try:
        for r4 in (1, 0):
            K.set_knob("KVMIX_R4", r4)
            check_attend(dev, ora, q, G=G, expect_mma=True)
            outs.append(K.attend(torch.from_numpy(q).cuda(), dev).output.cpu().numpy())
    finally:
        K.set_knob("KVMIX_R4", 1)
    vmax = float(np.abs(ora.snapshot()[1]).max())
    assert float(np.abs(outs[0] - outs[1]).max()) / vmax <= 4e-7


@pytest.mark.parametrize("gs", [64, 128])
def test_attend_group_sizes(cuda, gs):
    dev, ora = build(2, 4, 0.1, 0.1, gs, 1, 4, 128, [1200, 1, 1, 300] + [1] * 20, seed=31)
    check_attend(dev, ora, O.random_h16(13, (1, 4, 2, 128)), expect_mma=True)


def test_attend_scale_ramp(cuda):
    """Magnitudes growing 1000x along the context and a late dominant key: the Value
    fixed-point exponent and the lazy softmax reference move several times per segment."""
    B, H, D, T = 2, 4, 128, 3000
    ramp = np.exp(np.linspace(0.0, np.log(1000.0), T)).astype(np.float32)[None, None, :, None]
    k = (O.random_h16(41, (B, H, T, D)) * ramp).astype(np.float16).astype(np.float32)
    v = (O.random_h16(42, (B, H, T, D)) * ramp).astype(np.float16).astype(np.float32)
    q = O.random_h16(43, (B, H, 1, D), sigma=0.01)
    k[:, :, 2500] = (q[:, :, 0] * 50.0).astype(np.float16).astype(np.float32)
    for kb, vb in ((2, 2), (4, 4), (2, 4)):
        dev = K.KVLayerCache(K.LayerQuantConfig(0, kb, vb, 0.05, 0.05, 32), B, H, D, capacity_tokens=T + 16)
        ora = O.CacheOracle(kb, vb, 0.05, 0.05, 32, B, H, D)
        for a, z in ((0, 2900), (2900, 3000)):
            dev.append(k[:, :, a:z], v[:, :, a:z])
            ora.append(np.ascontiguousarray(k[:, :, a:z]), np.ascontiguousarray(v[:, :, a:z]))
        check_attend(dev, ora, q, expect_mma=True)


def test_attend_forced_folds(cuda):
    """The int32 Value accumulators are folded every N blocks (N = 1024 in production,
    lowered here so that path runs): same result within the stated tolerance."""
    from paper_2506_08018_b200 import _lib
    dev, ora = build(2, 2, 0.1, 0.1, 32, 1, 2, 128, [2000] + [1] * 5, seed=17)
    q = O.random_h16(18, (1, 2, 1, 128), sigma=2.0)
    try:
        for n in (1, 3):
            _lib.set_knob("KVMIX_TEST_FLUSH_BLOCKS", n)
            check_attend(dev, ora, q, expect_mma=True)
    finally:
        _lib.set_knob("KVMIX_TEST_FLUSH_BLOCKS", 0)


def test_attend_d64_two_rows(cuda):
    """IMMA path at D = 64 (lanes 16..31 mirror the Key channel quads) with two query rows."""
    dev, ora = build(4, 2, 0.1, 0.1, 32, 2, 4, 64, [900] + [1] * 9, seed=19)
    check_attend(dev, ora, O.random_h16(20, (2, 4, 2, 64), sigma=1.5), expect_mma=True)
    dev, ora = build(2, 4, 0.1, 0.1, 32, 1, 3, 64, [700, 3, 1], seed=23)
    check_attend(dev, ora, O.random_h16(24, (1, 6, 1, 64)), G=2, expect_mma=True)


def test_full_precision_cache_exact_dot(cuda):
    """test_attention.cpp:73-87: r=1 cache -> scores are plain scaled dot products."""
    dev, ora = build(2, 2, 1.0, 1.0, 32, 1, 2, 64, [50], seed=1)
    q = O.random_h16(2, (1, 2, 1, 64))
    s = K.fused_qk_scores(q, dev).cpu().numpy()
    ks, _ = ora.snapshot()
    ref = np.einsum("bhtd,bhjd->bhtj", q.astype(np.float64), ks.astype(np.float64)) / np.sqrt(64.0)
    assert np.abs(s - ref).max() < 1e-5


def test_zero_query_uniform(cuda):
    dev, ora = build(4, 4, 0.2, 0.2, 32, 1, 1, 64, [200], seed=2)
    q = np.zeros((1, 1, 1, 64), np.float32)
    s = K.fused_qk_scores(q, dev)
    assert torch.count_nonzero(s) == 0
    p = K.softmax_rows(s).cpu().numpy()
    assert np.allclose(p, 1.0 / 200, rtol=1e-6)


def test_separate_kernels_compose_to_attend(cuda):
    dev, ora = build(3, 4, 0.2, 0.2, 32, 1, 2, 64, [150, 7, 1], seed=8)
    q = O.random_h16(3, (1, 2, 3, 64))
    p = K.softmax_rows(K.fused_qk_scores(q, dev))
    assert torch.allclose(p.sum(-1), torch.ones(1, 2, 3, device="cuda"), atol=1e-6)
    out = K.fused_pv(p, dev).cpu().numpy()
    ks, vs = ora.snapshot()
    o64, _ = O.attend_f64(q, ks, vs)
    assert np.abs(out - o64).max() / np.abs(vs).max() < ATTN_TOL_F64


def test_one_hot_tail_token_exact(cuda):
    """test_attention.cpp:131-143."""
    dev, ora = build(2, 2, 0.25, 0.25, 32, 1, 1, 64, [60, 40], seed=4)
    total = dev.total_tokens()
    j = total - dev.value_tail_tokens() + 1
    probs = torch.zeros(1, 1, 1, total, device="cuda")
    probs[0, 0, 0, j] = 1.0
    out = K.fused_pv(probs, dev)
    _, vs = dev.snapshot_dequantized()
    assert torch.equal(out[0, 0, 0], vs[0, 0, j])


def test_reference_attend_matches_oracle(cuda):
    dev, ora = build(2, 3, 0.3, 0.2, 32, 1, 2, 64, [333, 1, 1], seed=5)
    q = O.random_h16(4, (1, 2, 2, 64))
    ref = K.reference_attend(q, dev)
    ks, vs = ora.snapshot()
    o64, cs = O.attend_f64(q, ks, vs)
    assert np.abs(ref.output.cpu().numpy() - o64).max() / np.abs(vs).max() < ATTN_TOL_F64
    assert abs(ref.scores_checksum - cs) <= CHECKSUM_RTOL * abs_score_sum(q, ks) + 1e-9


def test_bits_monotone_error(cuda):
    """test_attention.cpp:251-275 / acceptance criterion 9, fewer trials."""
    err = {}
    for bits in (2, 3, 4):
        tot = 0.0
        for trial in range(6):
            qd, _ = build(bits, bits, 0.1, 0.1, 32, 1, 2, 64, [160, 1, 1], seed=1000 + trial)
            fp, _ = build(bits, bits, 1.0, 1.0, 32, 1, 2, 64, [160, 1, 1], seed=1000 + trial)
            q = O.random_h16(trial, (1, 2, 1, 64))
            tot += float((K.attend(q, qd).output - K.attend(q, fp).output).abs().mean())
        err[bits] = tot
    assert err[2] >= err[3] >= err[4] > 0


def test_concurrent_readers_identical(cuda):
    dev, _ = build(2, 2, 0.2, 0.2, 32, 1, 2, 64, [300], seed=9)
    q = torch.from_numpy(O.random_h16(1, (1, 2, 1, 64))).cuda()
    serial = K.attend(q, dev).output.clone()
    outs = [None, None]

    def run(i):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            outs[i] = K.attend(q, dev).output
        s.synchronize()

    th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert torch.equal(outs[0], serial) and torch.equal(outs[1], serial)


def test_errors(cuda):
    dev, _ = build(2, 2, 0.2, 0.2, 32, 1, 2, 64, [40], seed=10)
    with pytest.raises(K.KvmixInvalidArgument):
        K.fused_qk_scores(np.zeros((1, 2, 1, 32), np.float32), dev)
    with pytest.raises(K.KvmixInvalidArgument):
        K.fused_pv(torch.zeros(1, 2, 1, 39), dev)
    empty = K.KVLayerCache(K.LayerQuantConfig(0, 2, 2, 0.2, 0.2, 32), 1, 1, 64, capacity_tokens=8)
    with pytest.raises(K.KvmixInvalidArgument):
        K.attend(np.zeros((1, 1, 1, 64), np.float32), empty)
    with pytest.raises(K.KvmixInvalidArgument):
        K.attend(np.zeros((1, 3, 1, 64), np.float32), dev)


@pytest.mark.parametrize("kb,vb,D,G,tail", [(2, 2, 128, 1, torch.float16), (3, 4, 128, 1, torch.float32),
                                             (4, 2, 64, 2, torch.float16), (2, 4, 128, 1, torch.float32),
                                             (2, 2, 128, 4, torch.float16), (3, 4, 128, 4, torch.float32)])
def test_append_attend_matches_separate_calls(cuda, kb, vb, D, G, tail):
    """kvmix_append_attend (the append fused into the attention launch when it is a decode
    step) == append() then attend(): identical outputs, identical cache state, and the fused
    path is the one that runs in the steady state."""
    B, H = 2, 3
    fused = K.KVLayerCache(K.LayerQuantConfig(0, kb, vb, 0.1, 0.1, 32), B, H, D, capacity_tokens=700, tail_dtype=tail)
    sep = K.KVLayerCache(K.LayerQuantConfig(0, kb, vb, 0.1, 0.1, 32), B, H, D, capacity_tokens=700, tail_dtype=tail)
    pre = torch.from_numpy(O.random_h16(70, (B, H, 500, D))).cuda()
    pre_v = torch.from_numpy(O.random_h16(71, (B, H, 500, D))).cuda()
    fused.append(pre, pre_v)
    sep.append(pre, pre_v)
    n_fused = 0
    for s in range(80):
        k = torch.from_numpy(O.random_h16(100 + s, (B, H, 1, D))).cuda().half()
        v = torch.from_numpy(O.random_h16(300 + s, (B, H, 1, D))).cuda().half()
        q = torch.from_numpy(O.random_h16(500 + s, (B, H * G, 1, D))).cuda()
        a0 = K.launch_count_of("append_decode_kernel") + K.launch_count_of("append_kernel")
        r1 = K.append_attend(fused, k, v, q)
        n_fused += (K.launch_count_of("append_decode_kernel") + K.launch_count_of("append_kernel")) == a0
        sep.append(k, v)
        r2 = K.attend(q, sep, checksum=False)
        assert torch.equal(r1.output, r2.output), s
    assert fused.dump() == sep.dump()
    assert n_fused >= 60  # steady-state steps ran as one launch


def test_append_attend_from_an_empty_cache(cuda):
    """The first decode step of an empty cache: the append makes it non-empty, so
    append_attend must not raise the empty-softmax error (attend alone does)."""
    k = torch.from_numpy(O.random_h16(90, (1, 2, 1, 64))).cuda()
    v = torch.from_numpy(O.random_h16(91, (1, 2, 1, 64))).cuda()
    q = torch.from_numpy(O.random_h16(92, (1, 2, 1, 64))).cuda()
    for kb, vb, r in ((2, 2, 0.1), (4, 4, 1.0)):
        mk = lambda: K.KVLayerCache(K.LayerQuantConfig(0, kb, vb, r, r, 32), 1, 2, 64, capacity_tokens=64)
        c, sep = mk(), mk()
        with pytest.raises(K.KvmixInvalidArgument):
            K.attend(q, c)
        out = K.append_attend(c, k, v, q).output
        sep.append(k, v)
        assert torch.equal(out, K.attend(q, sep, checksum=False).output)
        assert c.total_tokens() == 1
        if r == 1.0:  # one full-precision token: softmax weight 1, out == v
            assert torch.equal(out, v.float())


@pytest.mark.parametrize("kb,vb,gs,rk,rv,tail", [(2, 2, 32, 0.1, 0.1, torch.float32), (3, 4, 32, 0.2, 0.2, torch.float16),
                                                 (2, 4, 64, 0.1, 0.1, torch.float16), (4, 2, 32, 0.1, 0.3, torch.float32),
                                                 (2, 3, 32, 0.1, 0.1, torch.float16), (3, 3, 32, 0.2, 0.2, torch.float32)])
def test_attend_window_blocks_through_a_cycle(cuda, kb, vb, gs, rk, rv, tail):
    """The Key window (full precision, Values already packed) runs through the IMMA Value
    path in 32-token window blocks. Walk a whole Key age-out cycle one decode step at a time
    with many (b, kv-head) so warps mix fast groups, window blocks and window tokens."""
    B, H, D = 1, 32, 128
    dev, ora = build(kb, vb, rk, rv, gs, B, H, D, [1500], seed=61, tail_dtype=tail, cap=1600)
    q = O.random_h16(62, (B, H, 1, D), sigma=1.5)
    for s in range(40):
        k = O.random_h16(700 + s, (B, H, 1, D))
        v = O.random_h16(800 + s, (B, H, 1, D))
        dev.append(k, v)
        ora.append(k, v)
        if s % 3 == 0 or s > 34:
            check_attend(dev, ora, q, expect_mma=True if vb != 3 else None)


@pytest.mark.parametrize("kb,D,G,tq,gs", [(2, 128, 1, 1, 32), (3, 128, 1, 1, 32), (4, 64, 2, 1, 32), (2, 128, 4, 1, 32),
                                         (3, 128, 1, 3, 32), (2, 64, 1, 2, 64), (4, 128, 2, 1, 128)])
def test_attend_3bit_values_tensor_core(cuda, tc_kernel, kb, D, G, tq, gs):
    """3-bit Values (Mixed3 in the reference, 4-bit fields on the device) run on the tensor cores
    in the warp-specialized kernel: the IMMA sums code * scale and the narrow slots (stream index
    % 11 == 10, decoded with scale * 7/3, quant.cpp:36-53) are corrected on the CUDA cores --
    same tolerance as every other tier. The single-warp kernel leaves them to the generic one."""
    H = 4
    dev, ora = build(kb, 3, 0.15, 0.1, gs, 2, H, D, [1000, 37] + [1] * 25, seed=91 + kb)
    q = O.random_h16(92, (2, H * G, tq, D), sigma=1.7)
    check_attend(dev, ora, q, G=G, expect_mma=tc_kernel in ("ws", "tc"))


@pytest.mark.parametrize("kb,vb", [(2, 2), (3, 4), (2, 3)])
def test_scratch_independent_of_token_count(cuda, tc_kernel, kb, vb):
    """The reference's scratch contract (scratch.hpp:14-21, test_attention.cpp:182-205): the
    fused path's scratch does not grow with the cached tokens. kvmix_scratch_allocated counts
    the bytes requested per call (split-K partials, counters, flags) -- equal at 128 and 32768
    tokens, for attend and for the fused append + attend."""
    from paper_2506_08018_b200 import _lib
    B, H, D = 2, 4, 128
    sizes = []
    for T in (128, 32768):
        dev = K.KVLayerCache(K.LayerQuantConfig(0, kb, vb, 0.1, 0.1, 32), B, H, D, capacity_tokens=T + 8,
                             tail_dtype=torch.float16)
        dev.append(torch.randn(B, H, T, D, device=cuda, dtype=torch.float16),
                   torch.randn(B, H, T, D, device=cuda, dtype=torch.float16))
        q = torch.randn(B, H, 1, D, device=cuda)
        _lib.scratch_reset()
        K.attend(q, dev, checksum=False)
        a = _lib.scratch_allocated()
        _lib.scratch_reset()
        K.append_attend(dev, torch.randn(B, H, 1, D, device=cuda), torch.randn(B, H, 1, D, device=cuda), q)
        sizes.append((a, _lib.scratch_allocated()))
    assert sizes[0] == sizes[1] and sizes[0][0] > 0, sizes
