"""GPU parity: quantize/pack, dequantize, bitpack through the C ABI vs the CPU oracle.

Bar: bit-exact words and meta (integer/byte work). Mirrors test_quant.cpp / test_bitpack.cpp.
"""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2506_08018_b200 as K

pytestmark = pytest.mark.gpu


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


def _u16(t):
    return t.cpu().numpy().view(np.uint16).reshape(-1, 2)


@pytest.mark.parametrize("bits", [1, 2, 3, 4])
@pytest.mark.parametrize("gs", [8, 16, 32, 64, 128])
@pytest.mark.parametrize("key", [True, False])
def test_quantize_sweep_bit_exact(cuda, bits, gs, key):
    for shape, seed in [((1, 2, 128, 64), 1), ((2, 3, 256, 48), 2), ((1, 1, 128, 5), 3), ((1, 4, 384, 128), 4)]:
        x = O.random_h16(seed * 100 + bits * 10 + gs, shape, sigma=1.7, mu=0.3)
        w, m = O.quantize(x, bits, gs, key)
        spec = K.QuantSpec(bits, K.Grouping.kPerChannelKey if key else K.Grouping.kPerTokenValue, gs)
        f = K.quantize_key_tensor if key else K.quantize_value_tensor
        qg = f(torch.from_numpy(x).cuda(), spec)
        assert np.array_equal(_u32(qg.codes.words), w), (shape, bits, gs, key)
        assert np.array_equal(_u16(qg.meta), m), (shape, bits, gs, key)
        # fp16 input of the same (binary16-grid) values gives the same words
        qh = f(torch.from_numpy(x).cuda().half(), spec)
        assert np.array_equal(_u32(qh.codes.words), w)
        # dequantize == value_at, bit-exact (mul then add, no FMA)
        ref = O.dequantize(w, m, key, shape, bits, gs)
        assert np.array_equal(qg.dequantize().cpu().numpy().view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("bits", [2, 3, 4])
def test_config1_shape_bit_exact(cuda, bits):
    """BASELINE config 1 shape [1,32,4096,128], gs 32, both groupings."""
    x = O.random_h16(77, (1, 32, 4096, 128))
    xd = torch.from_numpy(x).cuda()
    for key in (True, False):
        w, m = O.quantize(x, bits, 32, key)
        f = K.quantize_key_tensor if key else K.quantize_value_tensor
        qg = f(xd, K.QuantSpec(bits, K.Grouping(0 if key else 1), 32))
        assert np.array_equal(_u32(qg.codes.words), w)
        assert np.array_equal(_u16(qg.meta), m)


def test_quantize_edge_values(cuda):
    """Constant groups, negative ranges, ties at .5 (half away from zero), arbitrary fp32,
    huge values, infinities and NaNs all reproduce the reference's bits."""
    rng = np.random.default_rng(5)
    x = rng.standard_normal((1, 2, 64, 32)).astype(np.float32) * 3
    x[0, 0, :32, 0] = 0.75          # constant channel group
    x[0, 0, 5, :] = -1.25           # constant token
    x[0, 1, :, 3] = np.arange(64) * 0.5  # exact .5 ties
    x[0, 1, 7, 7] = 7e4             # beyond binary16 range
    x[0, 1, 9, 9] = -np.inf
    x[0, 1, 40, 1] = np.nan
    x[0, 0, 33, 2] = 1e-7           # subnormal binary16 meta
    for bits in (2, 3, 4):
        for key in (True, False):
            w, m = O.quantize(x, bits, 32, key)
            f = K.quantize_key_tensor if key else K.quantize_value_tensor
            qg = f(torch.from_numpy(x).cuda(), K.QuantSpec(bits, K.Grouping(0 if key else 1), 32))
            assert np.array_equal(_u32(qg.codes.words), w), (bits, key)
            assert np.array_equal(_u16(qg.meta), m), (bits, key)


@pytest.mark.parametrize("gs", [8, 32, 128])
def test_quantize_tie_dense(cuda, gs):
    """Inputs on a 1/8 grid: (x - min) / scale lands exactly on, or one rounding away from,
    half-integers for a large share of the codes -- the quantizers' reciprocal fast path
    must hand every such code to the exact IEEE-division path (half away from zero)."""
    rng = np.random.default_rng(11 + gs)
    x = (rng.integers(-16, 17, size=(2, 3, 256, 128)) / 8.0).astype(np.float32)
    x[0, 0, :, :7] = rng.integers(0, 4, size=(256, 7)) * 0.5 - 0.75  # 4 levels: ties for 2/3 bits
    x[1, 2, 3, :] = np.float32(1.0) + np.float32(2.0 ** -20) * rng.integers(-3, 4, size=128)  # near-constant
    # zero extremes of both signs: the reference keeps the FIRST of -0 / +0
    x[1, 0, 5, :] = np.abs(x[1, 0, 5, :]); x[1, 0, 5, 0::4] = 0.0; x[1, 0, 5, 1::4] = -0.0
    x[1, 0, 6, :] = np.abs(x[1, 0, 6, :]); x[1, 0, 6, 0::4] = -0.0; x[1, 0, 6, 2::4] = 0.0
    x[1, 0, 7, :] = -np.abs(x[1, 0, 7, :]); x[1, 0, 7, 3::8] = -0.0; x[1, 0, 7, 5::8] = 0.0
    x[1, 1, :, 4] = np.abs(x[1, 1, :, 4]); x[1, 1, 0::3, 4] = -0.0; x[1, 1, 1::3, 4] = 0.0
    for bits in (2, 3, 4):
        for key in (True, False):
            w, m = O.quantize(x, bits, gs, key)
            f = K.quantize_key_tensor if key else K.quantize_value_tensor
            qg = f(torch.from_numpy(x).cuda(), K.QuantSpec(bits, K.Grouping(0 if key else 1), gs))
            assert np.array_equal(_u32(qg.codes.words), w), (bits, key)
            assert np.array_equal(_u16(qg.meta), m), (bits, key)


def test_known_words(cuda):
    # test_bitpack.cpp:77-96 / :133-142
    assert K.pack_uniform([0] * 16, 2).words_u32().tolist() == [0]
    assert K.pack_uniform([3] * 16, 2).words_u32().tolist() == [0xFFFFFFFF]
    b = K.pack_uniform([0, 1, 2, 3], 2)
    assert b.words_u32().tolist() == [0xE4] and K.unpack_uniform(b, 3) == 3
    assert K.unpack_uniform(K.pack_uniform([1], 1), 0) == 1
    assert K.pack_mixed3([7] * 10 + [3]).words_u32().tolist() == [0xFFFFFFFF]
    assert K.pack_mixed3([0] * 11).words_u32().tolist() == [0]


def test_pack_errors_name_index(cuda):
    with pytest.raises(K.KvmixInvalidArgument, match="index 2"):
        K.pack_uniform([1, 2, 4, 0], 2)
    codes = [0] * 15
    codes[14] = 4
    K.pack_mixed3(codes)
    codes[14] = 8
    with pytest.raises(K.KvmixInvalidArgument, match="block 1.*index 3"):
        K.pack_mixed3(codes)
    with pytest.raises(K.KvmixInvalidArgument):
        K.pack_mixed3([0] * 10 + [4])
    for bad in (3, 8, 0):
        with pytest.raises(K.KvmixInvalidArgument):
            K.feat_per_word(bad)
    buf = K.pack_uniform([0, 1, 2, 3], 2)
    with pytest.raises(K.KvmixOutOfRange):
        buf.get(4)
    with pytest.raises(K.KvmixInvalidArgument):
        K.unpack_uniform(K.pack_mixed3([1, 2, 3]), 0)
    with pytest.raises(K.KvmixInvalidArgument):
        K.unpack_mixed3(buf, 0)


def test_pack_roundtrip_every_length(cuda):
    """test_bitpack.cpp:199-214 (lengths 0..1000, step 37 on the GPU)."""
    rng = np.random.default_rng(0x1009)
    for n in list(range(0, 40)) + list(range(40, 1001, 37)):
        for bits in (1, 2, 4):
            c = rng.integers(0, 1 << bits, n).astype(np.uint32)
            buf = K.pack_uniform(c, bits)
            assert buf.word_count() == (n * bits + 31) // 32
            assert np.array_equal(buf.words_u32(), O.pack(c, bits))
            assert np.array_equal(K.unpack(buf), c)
        c = np.array([rng.integers(0, 4 if i % 11 == 10 else 8) for i in range(n)], np.uint32)
        buf = K.pack_mixed3(c)
        assert buf.word_count() == (n + 10) // 11
        assert np.array_equal(buf.words_u32(), O.pack(c, 3))
        assert np.array_equal(K.unpack(buf), c)


def test_key_rejects_ragged(cuda):
    with pytest.raises(K.KvmixInvalidArgument):
        K.quantize_key_tensor(torch.zeros(1, 1, 33, 2, device="cuda"), K.QuantSpec(4, K.Grouping.kPerChannelKey, 32))
    with pytest.raises(K.KvmixInvalidArgument):
        K.quantize_key_tensor(torch.zeros(1, 1, 32, 2, device="cuda"), K.QuantSpec(4, K.Grouping.kPerTokenValue, 32))


def test_kvqg_golden_bytes(cuda):
    """test_quant.cpp:264-310."""
    v = torch.tensor([0.0, 1.0, 2.0, 3.0]).reshape(1, 1, 1, 4).cuda()
    qg = K.quantize_value_tensor(v, K.QuantSpec(2, K.Grouping.kPerTokenValue, 4))
    golden = bytes([ord("K"), ord("V"), ord("Q"), ord("G"), 1, 2, 1, 0, 4, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0,
                    4, 0, 0, 0, 1, 0, 0, 0, 0, 0, 0, 0, 4, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 0, 0, 0, 0x00, 0x3C,
                    0x00, 0x00, 0xE4, 0, 0, 0])
    assert K.serialize_quantized_groups(qg) == golden
    back = K.deserialize_quantized_groups(golden)
    assert back.spec.bits == 2 and back.spec.group_size == 4
    assert torch.equal(back.dequantize(), qg.dequantize())
    with pytest.raises(K.KvmixRuntimeError):
        K.deserialize_quantized_groups(b"X" + golden[1:])
    with pytest.raises(K.KvmixRuntimeError):
        K.deserialize_quantized_groups(golden[:-1])


@pytest.mark.parametrize("bits", [2, 3, 4])
@pytest.mark.parametrize("key", [True, False])
def test_value_at_and_get_per_element(cuda, bits, key):
    """QuantizedGroups::value_at / PackedBuffer::get (quant.cpp:97-100, bitpack.cpp:69-82) read
    one word and one meta pair each, bit-exact with the bulk dequantize / oracle decode."""
    shape = (2, 3, 64, 40)
    x = O.random_h16(bits * 7 + key, shape, sigma=1.3)
    spec = K.QuantSpec(bits, K.Grouping.kPerChannelKey if key else K.Grouping.kPerTokenValue, 32)
    qg = (K.quantize_key_tensor if key else K.quantize_value_tensor)(torch.from_numpy(x).cuda(), spec)
    full = qg.dequantize().cpu().numpy()
    w, _ = O.quantize(x, bits, 32, key)
    rng = np.random.default_rng(bits)
    for _ in range(40):
        b, h, t, d = (int(rng.integers(0, n)) for n in shape)
        assert np.float32(qg.value_at(b, h, t, d)).view(np.uint32) == full[b, h, t, d].view(np.uint32)
        si = qg.stream_index(b, h, t, d)
        assert qg.codes.get(si) == O.get(w, si, bits)
    with pytest.raises(K.KvmixOutOfRange):
        qg.codes.get(qg.codes.logical_len)
