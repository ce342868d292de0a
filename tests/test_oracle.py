"""Pins the CPU oracle (oracle/kvmix_oracle.c + CacheOracle) to the reference (CPU tier).

Three anchors: (1) the reference test-suite's own known answers (test_bitpack.cpp,
test_quant.cpp, test_cache.cpp), (2) golden fixtures generated from the UNMODIFIED
reference library (tests/golden/make_golden.py), (3) live cross-checks against
oracle/_ref when it was built in this container.
"""
import json
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLD, "golden.json")) as f:
        idx = json.load(f)
    return idx, np.load(os.path.join(GOLD, "golden.npz"))


def test_known_words():
    # test_bitpack.cpp:77-96, :133-142
    assert O.pack([0] * 16, 2).tolist() == [0]
    assert O.pack([3] * 16, 2).tolist() == [0xFFFFFFFF]
    assert O.pack([0, 1, 2, 3], 2).tolist() == [0xE4]
    assert O.get(O.pack([0, 1, 2, 3], 2), 3, 2) == 3
    assert O.pack([7] * 10 + [3], 3).tolist() == [0xFFFFFFFF]
    assert O.pack([0] * 11, 3).tolist() == [0]
    with pytest.raises(O.OracleError, match="index 2"):
        O.pack([1, 2, 4, 0], 2)
    with pytest.raises(O.OracleError):
        O.pack([0] * 10 + [4], 3)


def test_word_counts_and_density():
    # test_bitpack.cpp:162-186, acceptance criterion 2
    rng = np.random.default_rng(0x3B17)
    for n in (0, 1, 10, 11, 12, 110, 513, 1000):
        c = np.array([rng.integers(0, 4 if i % 11 == 10 else 8) for i in range(n)], np.uint32)
        w = O.pack(c, 3)
        assert len(w) == (n + 10) // 11
        assert all(O.get(w, i, 3) == c[i] for i in range(n))
    for n in (110, 1100, 11000):
        assert O.words_for(n, 3) == n // 11 and (n + 9) // 10 == n // 10


def test_quantizer_formula_cases():
    # test_quant.cpp:56-118 via the element codec
    L = O.lib()
    assert L.ko_encode(1.4, 1.0, 0.0, 2, 0) == 1
    assert L.ko_encode(1.5, 1.0, 0.0, 2, 0) == 2  # half away from zero
    assert L.ko_encode(2.5, 1.0, 0.0, 2, 0) == 3
    assert L.ko_encode(5.0, 0.0, 5.0, 2, 0) == 0  # constant group
    assert L.ko_encode(3.0, 1.0, 0.0, 3, 10) == 1  # Mixed3 narrow slot: scale*7/3, q_max 3
    x = np.array([0, 1, 2, 3], np.float32)
    s, m = O.lib().ko_compute_meta.argtypes, None
    w, meta = O.quantize(x.reshape(1, 1, 1, 4), 2, 4, key=False)
    assert w.tolist() == [0xE4] and meta.tolist() == [[0x3C00, 0x0000]]


def test_binary16_spot_values(golden):
    idx, _ = golden
    for f, h in idx["half"]:
        assert O.half_from_float(f) == h, f
    assert O.half_from_float(1.0) == 0x3C00
    assert abs(O.float_from_half(O.half_from_float(0.1)) - 0.0999755859375) < 1e-12
    assert O.round_through_half(-2.5) == -2.5


def test_rpc_target(golden):
    idx, _ = golden
    # test_cache.cpp:31-39 + fixtures from the reference
    assert O.rpc_target(10, 0.2) == 2 and O.rpc_target(25, 0.1) == 2 and O.rpc_target(201, 0.2) == 40
    for n, r, want in idx["rpc_target"]:
        assert O.rpc_target(n, r) == want


def test_quantize_matches_golden(golden):
    idx, arr = golden
    for case in idx["quant"]:
        i = case["i"]
        w, m = O.quantize(arr[f"q{i}_x"], case["bits"], case["gs"], case["key"])
        assert np.array_equal(w, arr[f"q{i}_words"]), case
        assert np.array_equal(m, arr[f"q{i}_meta"]), case


def test_cache_oracle_matches_golden(golden):
    idx, arr = golden
    for case in idx["cache"]:
        i = case["i"]
        c = O.CacheOracle(case["kbits"], case["vbits"], case["rk"], case["rv"], case["gs"], case["B"], case["H"], case["D"])
        seed = case["seed"]
        B, H, D = case["B"], case["H"], case["D"]
        for s, t in enumerate(case["chunks"]):
            c.append(O.random_h16(seed + 2 * s, (B, H, t, D)), O.random_h16(seed + 2 * s + 1, (B, H, t, D), sigma=2.0))
            tr = case["trace"][s]
            got = dict(c.counters(), **c.memory_usage())
            for k in ("total", "key_tail", "value_tail", "quant_keys", "quant_values", "key_segments",
                      "value_segments", "packed_payload_bits", "metadata_bits", "tail_bits", "total_bits"):
                assert got[k] == tr[k], (case["i"], s, k)
        assert np.array_equal(np.frombuffer(c.dump(), np.uint8), arr[f"c{i}_dump"])
        ks, vs = c.snapshot()
        assert np.array_equal(ks, arr[f"c{i}_keys"]) and np.array_equal(vs, arr[f"c{i}_values"])
        out, cs = O.attend_f32(arr[f"c{i}_q"], ks, vs)
        # reference_attend and attend are bit-identical on the CPU (same order)
        assert np.array_equal(out, arr[f"c{i}_refattend"])
        assert np.array_equal(out, arr[f"c{i}_attend"])
        assert cs == case["checksum"] == case["ref_checksum"]


def test_shrink_rule_replay_long_trace():
    """acceptance criterion 6 on the integer bookkeeping: 1000 prefill + 500 decode."""
    for r, gs in ((0.2, 32), (0.1, 32)):
        kt = C_k = 0
        import ctypes
        tail = ctypes.c_int64(0)
        vtail = ctypes.c_int64(0)
        q = qv = 0
        L = O.lib()
        q += L.ko_shrink(ctypes.byref(tail), 1000, r, gs, 1)
        qv += L.ko_shrink(ctypes.byref(vtail), 1000, r, gs, 0)
        for _ in range(500):
            q += L.ko_shrink(ctypes.byref(tail), 1, r, gs, 1)
            qv += L.ko_shrink(ctypes.byref(vtail), 1, r, gs, 0)
        assert q + tail.value == 1500 and qv + vtail.value == 1500
        assert q % gs == 0


def test_memory_accounting_known_answers():
    # test_cache.cpp:171-184: fully quantized 2-bit gs32 -> 16/3
    c = O.CacheOracle(2, 2, 0.0, 0.0, 32, 1, 1, 32)
    c.append(O.random_h16(3, (1, 1, 128, 32)), O.random_h16(4, (1, 1, 128, 32)))
    m = c.memory_usage()
    assert m["tail_bits"] == 0 and abs(m["compression_ratio"] - 16.0 / 3.0) < 1e-12
    assert O.CacheOracle(2, 2, 0.1, 0.1, 32, 1, 1, 8).memory_usage()["compression_ratio"] == 1.0


def test_criterion7_compression_ratio():
    """acceptance.cpp:352-401: 32-layer mixed config, 4096 + 1024 tokens -> 4.82969."""
    def words_for(n, bits):
        return (n + 10) // 11 if bits == 3 else (n * bits + 31) // 32
    total = base = 0
    for layer in range(32):
        hi = layer < 6
        kb, vb, r = (3, 4, 0.2) if hi else (2, 2, 0.1)
        r32 = float(np.float32(r))
        nh, d = 4, 64
        kt = vt = tot = 0
        payload = meta = 0
        for t in [4096] + [1] * 1024:
            tot += t
            kt += t
            vt += t
            aged = (kt - O.rpc_target(kt, r32)) // 32 * 32
            if aged > 0:
                payload += words_for(aged * nh * d, kb) * 32
                meta += nh * d * (aged // 32) * 32
                kt -= aged
            aged = vt - O.rpc_target(vt, r32)
            if aged > 0:
                payload += words_for(aged * nh * d, vb) * 32
                meta += aged * nh * ((d + 31) // 32) * 32
                vt -= aged
        total += payload + meta + (kt + vt) * nh * d * 16
        base += tot * nh * d * 32
    assert abs(base / total - 4.82969) < 5e-6


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built in this container")
def test_oracle_vs_live_reference():
    rng = np.random.default_rng(7)
    for trial in range(20):
        bits, gs = int(rng.integers(1, 5)), int(rng.choice([4, 8, 16, 32, 64]))
        key = bool(trial % 2)
        T = gs * int(rng.integers(1, 5)) if key else int(rng.integers(1, 40))
        x = O.random_h16(trial, (int(rng.integers(1, 3)), int(rng.integers(1, 4)), T, int(rng.integers(1, 70))),
                         sigma=float(rng.uniform(0.1, 4)), mu=float(rng.uniform(-2, 2)))
        w, m = O.quantize(x, bits, gs, key)
        w2, m2 = O.ref_quantize(x, bits, gs, key)
        assert np.array_equal(w, w2) and np.array_equal(m, m2)
    c = O.CacheOracle(3, 2, 0.37, 0.11, 32, 2, 2, 16)
    r = O.RefCache(3, 2, 0.37, 0.11, 32, 2, 2, 16)
    for s in range(30):
        t = int(rng.integers(1, 50))
        k, v = O.random_h16(500 + s, (2, 2, t, 16)), O.random_h16(900 + s, (2, 2, t, 16))
        c.append(k, v)
        r.append(k, v)
        assert c.counters() == r.counters()
    assert c.dump() == r.dump()


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built in this container")
@pytest.mark.parametrize("vb", [2, 3, 4])
def test_oracle_special_values_vs_live_reference(vb):
    """NaN / +-0 / inf in aged tokens (group first element, mid-group): the oracle's fold
    equals the reference's (quant.hpp:170-182) -- pins the oracle for the GPU special-value
    tests (tests/test_cache_gpu.py::test_decode_append_special_values)."""
    from test_cache_gpu import _special_token
    B, H, D = 1, 2, 128
    ora = O.CacheOracle(2, vb, 0.1, 0.1, 32, B, H, D)
    ref = O.RefCache(2, vb, 0.1, 0.1, 32, B, H, D)
    k, v = O.random_h16(7, (B, H, 64, D)), O.random_h16(8, (B, H, 64, D))
    ora.append(k, v)
    ref.append(k, v)
    rng = np.random.default_rng(vb)
    for step in range(40):
        kn, vn = O.random_h16(2000 + step, (B, H, 1, D)), _special_token(rng, B, H, D, step)
        ora.append(kn, vn)
        ref.append(kn, vn)
    assert ora.dump() == ref.dump()
