"""GPU parity: the device KVLayerCache vs the CPU cache oracle (and the compiled reference
when oracle/_ref exists). Bar: identical counters and MemoryReport, bit-exact snapshot,
byte-identical segment words/meta and KVCD dump. Mirrors test_cache.cpp and acceptance
criteria 6/7."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2506_08018_b200 as K

pytestmark = pytest.mark.gpu


def make_pair(kb, vb, rk, rv, gs, B, H, D, cap, tail_dtype=torch.float32):
    dev = K.KVLayerCache(K.LayerQuantConfig(0, kb, vb, rk, rv, gs), B, H, D, capacity_tokens=cap, tail_dtype=tail_dtype)
    ora = O.CacheOracle(kb, vb, rk, rv, gs, B, H, D)
    return dev, ora


def assert_same(dev, ora, check_segments=True):
    c = ora.counters()
    assert dev.total_tokens() == c["total"]
    assert dev.key_tail_tokens() == c["key_tail"]
    assert dev.value_tail_tokens() == c["value_tail"]
    assert dev.quantized_key_tokens() == c["quant_keys"]
    assert dev.quantized_value_tokens() == c["quant_values"]
    m = dev.memory_usage()
    om = ora.memory_usage()
    for f in ("packed_payload_bits", "metadata_bits", "tail_bits", "total_bits", "fp16_baseline_bits"):
        assert getattr(m, f) == om[f], f
    assert m.compression_ratio == om["compression_ratio"]
    ks, vs = dev.snapshot_dequantized()
    ok, ov = ora.snapshot()
    assert np.array_equal(ks.cpu().numpy().view(np.uint32), ok.view(np.uint32))
    assert np.array_equal(vs.cpu().numpy().view(np.uint32), ov.view(np.uint32))
    if check_segments:
        for segs, osegs in ((dev.key_segments(), ora.key_segs), (dev.value_segments(), ora.value_segs)):
            assert len(segs) == len(osegs)
            for qg, (n, w, mm) in zip(segs, osegs):
                assert qg.shape.t == n
                assert np.array_equal(qg.codes.words_u32(), w)
                assert np.array_equal(qg.meta.cpu().numpy().view(np.uint16).reshape(-1, 2), mm)


@pytest.mark.parametrize("kb,vb", [(2, 2), (3, 4), (4, 3), (3, 3), (4, 4), (2, 4)])
@pytest.mark.parametrize("gs", [32, 64])
def test_random_append_sequences(cuda, kb, vb, gs):
    rng = np.random.default_rng(kb * 100 + vb * 10 + gs)
    B, H, D = 2, 3, 64
    rk, rv = float(rng.uniform(0.05, 0.6)), float(rng.uniform(0.05, 0.6))
    dev, ora = make_pair(kb, vb, rk, rv, gs, B, H, D, cap=2048)
    seed = 1
    for step in range(25):
        t = int(rng.integers(1, 96)) if step % 3 else 1
        k = O.random_h16(seed, (B, H, t, D))
        v = O.random_h16(seed + 1, (B, H, t, D), sigma=2.0)
        seed += 2
        dev.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
        ora.append(k, v)
        assert_same(dev, ora, check_segments=(step % 6 == 5))
    assert_same(dev, ora)
    assert dev.dump() == ora.dump()


def test_prefill_decode_counts(cuda):
    """test_cache.cpp:50-70: 1000-token prefill then one decode step."""
    dev, ora = make_pair(2, 2, 0.2, 0.2, 32, 1, 1, 64, cap=2048)
    k, v = O.random_h16(1, (1, 1, 1000, 64)), O.random_h16(2, (1, 1, 1000, 64))
    dev.append(k, v)
    ora.append(k, v)
    assert dev.quantized_key_tokens() == 800 and dev.key_tail_tokens() == 200
    assert dev.quantized_value_tokens() == 800 and dev.value_tail_tokens() == 200
    assert len(dev.key_segments()) == 1 and dev.key_segments()[0].group_count() == 64 * 800 // 32
    k, v = O.random_h16(3, (1, 1, 1, 64)), O.random_h16(4, (1, 1, 1, 64))
    dev.append(k, v)
    ora.append(k, v)
    assert dev.quantized_key_tokens() == 960 and dev.key_tail_tokens() == 41
    assert dev.value_tail_tokens() == 40 and dev.total_tokens() == 1001
    assert_same(dev, ora)


def test_shrink_rule_long_trace(cuda):
    """acceptance criterion 6: 1000 prefill + 500 decode steps, both tiers, exact replay."""
    for bits, r in ((3, 0.2), (2, 0.1)):
        vb = 4 if bits == 3 else 2
        dev, ora = make_pair(bits, vb, r, r, 32, 1, 2, 64, cap=1600)
        k, v = O.random_h16(10, (1, 2, 1000, 64)), O.random_h16(11, (1, 2, 1000, 64))
        dev.append(k, v)
        ora.append(k, v)
        for s in range(500):
            k, v = O.random_h16(100 + 2 * s, (1, 2, 1, 64)), O.random_h16(101 + 2 * s, (1, 2, 1, 64))
            dev.append(k, v)
            ora.append(k, v)
            if s % 50 == 0:
                assert dev.key_tail_tokens() == ora.counters()["key_tail"]
        assert dev.total_tokens() == 1500
        assert_same(dev, ora)


def test_r1_never_quantizes_and_r0_fully(cuda):
    dev = K.KVLayerCache(K.LayerQuantConfig(0, 2, 2, 1.0, 1.0, 32), 1, 2, 64, capacity_tokens=64)
    for s in range(40):
        dev.append(O.random_h16(s, (1, 2, 1, 64)), O.random_h16(s + 99, (1, 2, 1, 64)))
    assert dev.quantized_key_tokens() == 0 and dev.key_tail_tokens() == 40
    assert dev.memory_usage().packed_payload_bits == 0
    # fully quantized 2-bit gs32 cache: 16/3 compression (test_cache.cpp:171-184)
    dev = K.KVLayerCache(K.LayerQuantConfig(0, 2, 2, 0.0, 0.0, 32), 1, 1, 64, capacity_tokens=128)
    dev.append(O.random_h16(1, (1, 1, 128, 64)), O.random_h16(2, (1, 1, 128, 64)))
    r = dev.memory_usage()
    assert dev.key_tail_tokens() == 0 and dev.value_tail_tokens() == 0
    assert abs(r.compression_ratio - 16.0 / 3.0) < 1e-12


def test_fp16_tail_and_fp16_input(cuda):
    """f16 tail + f16 inputs on the binary16 grid are lossless w.r.t. the fp32 reference."""
    dev, ora = make_pair(3, 4, 0.2, 0.2, 32, 1, 4, 128, cap=1024, tail_dtype=torch.float16)
    for s, t in enumerate([300, 1, 1, 17, 1, 64, 1, 1]):
        k, v = O.random_h16(s, (1, 4, t, 128)), O.random_h16(s + 50, (1, 4, t, 128))
        dev.append(torch.from_numpy(k).cuda().half(), torch.from_numpy(v).cuda().half())
        ora.append(k, v)
    assert_same(dev, ora)


def test_huge_prefill_split_launch(cuda):
    """Append larger than the device ring forces the two-launch path."""
    dev, ora = make_pair(2, 2, 0.1, 0.1, 32, 1, 2, 64, cap=4096)
    k, v = O.random_h16(5, (1, 2, 3000, 64)), O.random_h16(6, (1, 2, 3000, 64))
    dev.append(k, v)
    ora.append(k, v)
    for s in range(40):
        k, v = O.random_h16(7 + s, (1, 2, 1, 64)), O.random_h16(70 + s, (1, 2, 1, 64))
        dev.append(k, v)
        ora.append(k, v)
    assert_same(dev, ora)


def test_snapshot_token_order(cuda):
    """test_cache.cpp:124-153: values constant per token, keys constant per channel."""
    D = 64
    dev = K.KVLayerCache(K.LayerQuantConfig(0, 4, 4, 0.2, 0.2, 32), 1, 1, D, capacity_tokens=1024)
    rng = np.random.default_rng(9)
    appended = 0
    for _ in range(12):
        t = int(rng.integers(1, 81))
        k = np.tile(np.arange(D, dtype=np.float32), (1, 1, t, 1))
        v = np.repeat((appended + np.arange(t, dtype=np.float32)).reshape(1, 1, t, 1), D, axis=3)
        dev.append(k, v)
        appended += t
    ks, vs = dev.snapshot_dequantized()
    ks, vs = ks.cpu().numpy(), vs.cpu().numpy()
    assert ks.shape[2] == appended
    assert np.array_equal(vs[0, 0, :, 0], np.arange(appended, dtype=np.float32))
    assert np.array_equal(ks[0, 0, 5], np.arange(D, dtype=np.float32))


def test_dump_load_roundtrip(cuda):
    dev, ora = make_pair(3, 4, 0.2, 0.2, 32, 2, 2, 64, cap=1024)
    rng = np.random.default_rng(0xD1CE)
    for s in range(6):
        t = int(rng.integers(1, 100))
        k, v = O.random_h16(s, (2, 2, t, 64)), O.random_h16(s + 9, (2, 2, t, 64))
        dev.append(k, v)
        ora.append(k, v)
    blob = dev.dump()
    assert blob == ora.dump()
    back = K.KVLayerCache.load(blob, capacity_tokens=2048)
    assert back.total_tokens() == dev.total_tokens()
    k0, v0 = dev.snapshot_dequantized()
    k1, v1 = back.snapshot_dequantized()
    assert torch.equal(k0, k1) and torch.equal(v0, v1)
    assert back.dump() == blob
    # a loaded cache keeps appending identically
    k, v = O.random_h16(77, (2, 2, 40, 64)), O.random_h16(78, (2, 2, 40, 64))
    back.append(k, v)
    ora.append(k, v)
    assert_same(back, ora)
    with pytest.raises(K.KvmixRuntimeError):
        K.KVLayerCache.load(b"nope")


def test_errors(cuda):
    c = K.KVLayerCache(K.LayerQuantConfig(0, 2, 2, 0.1, 0.1, 32), 1, 2, 64, capacity_tokens=16)
    with pytest.raises(K.KvmixInvalidArgument):
        c.append(torch.zeros(1, 1, 4, 64), torch.zeros(1, 1, 4, 64))
    with pytest.raises(K.KvmixInvalidArgument):
        c.append(torch.zeros(1, 2, 4, 64), torch.zeros(1, 2, 5, 64))
    c.append(torch.zeros(1, 2, 17, 64), torch.zeros(1, 2, 17, 64))  # past the reservation: grows
    assert c.capacity_tokens() >= 17 and c.total_tokens() == 17
    for bad in (K.LayerQuantConfig(0, 5, 2), K.LayerQuantConfig(0, 2, 2, -0.1), K.LayerQuantConfig(0, 2, 2, group_size=0)):
        with pytest.raises(K.KvmixInvalidArgument):
            K.KVLayerCache(bad, 1, 1, 64)
    assert K.rpc_target(201, 0.2) == 40
    with pytest.raises(K.KvmixInvalidArgument):
        K.rpc_target(-1, 0.2)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_against_compiled_reference(cuda):
    """Direct check against the unmodified reference KVLayerCache (oracle/_ref)."""
    dev = K.KVLayerCache(K.LayerQuantConfig(0, 3, 2, 0.3, 0.15, 32), 2, 2, 64, capacity_tokens=2048)
    ref = O.RefCache(3, 2, 0.3, 0.15, 32, 2, 2, 64)
    rng = np.random.default_rng(3)
    for s in range(20):
        t = int(rng.integers(1, 120))
        k, v = O.random_h16(s, (2, 2, t, 64)), O.random_h16(s + 400, (2, 2, t, 64))
        dev.append(k, v)
        ref.append(k, v)
    assert dev.dump() == ref.dump()


def _special_token(rng, B, H, D, step):
    """One [B,H,1,D] token on the binary16 grid with NaN / +-0 / inf / tiny values placed at
    the group first element and at the first element of a non-leader lane's slice."""
    x = O.random_h16(1000 + step, (B, H, 1, D))
    kind = step % 6
    for h in range(H):
        if kind == 0:
            x[0, h, 0, 4] = np.nan          # first element of lane 1's slice (channels 4..7)
            x[0, h, 0, 5] = -30.0           # only visible if the fold skips the NaN and goes on
        elif kind == 1:
            x[0, h, 0, 0] = np.nan          # group first element: meta NaN
        elif kind == 2:
            x[0, h, 0, :32] = 0.0
            x[0, h, 0, 3] = -0.0            # zero extrema: the first occurrence's sign wins
            x[0, h, 0, 9] = -0.0
        elif kind == 3:
            x[0, h, 0, 0] = -0.0
            x[0, h, 0, 1:32] = np.abs(x[0, h, 0, 1:32])
        elif kind == 4:
            x[0, h, 0, 36] = np.inf
            x[0, h, 0, 40] = np.nan
        else:
            x[0, h, 0, 64] = np.nan
            x[0, h, 0, 65] = -np.inf
    return x.astype(np.float32)


@pytest.mark.parametrize("vb", [2, 3, 4])
@pytest.mark.parametrize("fused", [False, True])
def test_decode_append_special_values(cuda, vb, fused):
    """Single-token decode appends whose aged Value tokens hold NaN at a group's first element
    or at the start of a non-leader lane's slice, +-0 extrema and infinities: meta and codes
    equal the reference's sequential fold (quant.hpp:170-182) -- through the decode-append
    kernel and through the attention kernel's fused prologue (append_attend)."""
    B, H, D = 1, 2, 128
    rng = np.random.default_rng(vb)
    dev, ora = make_pair(2, vb, 0.1, 0.1, 32, B, H, D, cap=512)
    k = O.random_h16(7, (B, H, 64, D))
    v = O.random_h16(8, (B, H, 64, D))
    dev.append(k, v)
    ora.append(k, v)
    q = torch.from_numpy(O.random_h16(9, (B, H, 1, D))).cuda()
    for step in range(40):
        kn = O.random_h16(2000 + step, (B, H, 1, D))
        vn = _special_token(rng, B, H, D, step)
        if fused:
            K.append_attend(dev, torch.from_numpy(kn).cuda(), torch.from_numpy(vn).cuda(), q)
        else:
            dev.append(torch.from_numpy(kn).cuda(), torch.from_numpy(vn).cuda())
        ora.append(kn, vn)
    torch.cuda.synchronize()
    assert dev.dump() == ora.dump()
    if O.ref_available():
        ref = O.RefCache(2, vb, 0.1, 0.1, 32, B, H, D)
        ref.append(k, v)
        rng = np.random.default_rng(vb)
        for step in range(40):
            ref.append(O.random_h16(2000 + step, (B, H, 1, D)), _special_token(rng, B, H, D, step))
        assert dev.dump() == ref.dump()


@pytest.mark.parametrize("kb,vb,r", [(2, 2, 0.1), (3, 4, 0.2), (3, 3, 0.15)])
def test_append_grows_the_reservation(cuda, kb, vb, r):
    """append() past capacity_tokens re-creates the device store (segments and tails
    re-imported): state, counters and KVCD dump equal the oracle's after several growths."""
    B, H, D = 2, 3, 64
    dev = K.KVLayerCache(K.LayerQuantConfig(0, kb, vb, r, r, 32), B, H, D, capacity_tokens=40,
                         tail_dtype=torch.float16)
    ora = O.CacheOracle(kb, vb, r, r, 32, B, H, D)
    for i, t in enumerate([30, 1, 25, 70, 1, 1, 200, 3]):
        k, v = O.random_h16(700 + 2 * i, (B, H, t, D)), O.random_h16(701 + 2 * i, (B, H, t, D))
        dev.append(torch.from_numpy(k).cuda().half(), torch.from_numpy(v).cuda().half())
        ora.append(k, v)
    assert dev.capacity_tokens() >= dev.total_tokens() == 331
    assert dev.dump() == ora.dump()


@pytest.mark.parametrize("D", [4, 8, 16, 32, 48, 96, 200])
@pytest.mark.parametrize("kb,vb", [(2, 2), (3, 4), (4, 3)])
def test_any_head_dim(cuda, D, kb, vb):
    """head_dim outside {64, 128} (the reference's own tests use 4..32; harness.hpp:50 and
    toymodel.hpp:40 default to 32 / 16): the tile layout rounds D up to a multiple of 64 with
    zero codes in the extra channels. Appends (prefill, decode, Key-group age-outs), KVCD
    dump, snapshot and the generic attention path match the oracle; dump/load round trips."""
    B, H = 2, 3
    r = 0.15
    dev = K.KVLayerCache(K.LayerQuantConfig(0, kb, vb, r, r, 32), B, H, D, capacity_tokens=256)
    ora = O.CacheOracle(kb, vb, r, r, 32, B, H, D)
    for i, t in enumerate([90, 1, 1, 40, 1, 33]):
        k, v = O.random_h16(900 + 2 * i, (B, H, t, D)), O.random_h16(901 + 2 * i, (B, H, t, D))
        dev.append(k, v)
        ora.append(k, v)
    assert dev.dump() == ora.dump()
    ks, vs = ora.snapshot()
    dks, dvs = dev.snapshot_dequantized()
    assert np.array_equal(dks.cpu().numpy().view(np.uint32), ks.view(np.uint32))
    assert np.array_equal(dvs.cpu().numpy().view(np.uint32), vs.view(np.uint32))
    q = O.random_h16(77, (B, H, 2, D))
    out = K.attend(torch.from_numpy(q).cuda(), dev).output.cpu().numpy()
    o64, _ = O.attend_f64(q, ks, vs)
    assert float(np.abs(out - o64).max()) / float(np.abs(vs).max()) <= 2e-6
    back = K.KVLayerCache.load(dev.dump(), capacity_tokens=256)
    assert back.dump() == dev.dump()
