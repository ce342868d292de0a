"""C-ABI and host-logic checks that need no GPU (CPU tier).

* libkvmix_b200.so loads and exports every function include/kvmix_b200.h declares;
* host-only entry points (validation, rpc_target, word/group counts) follow the
  reference's semantics and error types;
* without a CUDA device the compute entry points fail loudly (no CPU fallback);
* quant_config.txt I/O mirrors profiler.cpp (format, validation, error messages).
"""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest
import torch

import paper_2506_08018_b200 as K
from paper_2506_08018_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "kvmix_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kvmix_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    names = declared()
    assert len(names) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (kvmix_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    L = C.CDLL(_lib.LIB_PATH)
    for n in names:
        getattr(L, n)


def test_abi_version_and_counts():
    L = K.lib()
    assert L.kvmix_abi_version() == 1
    assert L.kvmix_packed_word_count(16, 2) == 1 and L.kvmix_packed_word_count(17, 2) == 2
    assert L.kvmix_packed_word_count(11, 3) == 1 and L.kvmix_packed_word_count(1000, 3) == 91
    assert L.kvmix_group_count(0, 2, 3, 64, 48, 32) == 2 * 3 * 48 * 2
    assert L.kvmix_group_count(1, 1, 2, 5, 48, 32) == 1 * 2 * 5 * 2
    assert K.feat_per_word(4) == 8 and K.feat_per_word(2) == 16 and K.feat_per_word(1) == 32
    for bad in (3, 8, 0):
        with pytest.raises(K.KvmixInvalidArgument):
            K.feat_per_word(bad)


def test_rpc_target_and_validation():
    # test_cache.cpp:31-47
    assert K.rpc_target(10, 0.2) == 2 and K.rpc_target(25, 0.1) == 2 and K.rpc_target(0, 0.2) == 0
    assert K.rpc_target(201, 0.2) == 40 and K.rpc_target(7, 1.0) == 7
    with pytest.raises(K.KvmixInvalidArgument):
        K.rpc_target(-1, 0.2)
    with pytest.raises(K.KvmixInvalidArgument):
        K.rpc_target(10, 1.5)
    assert K.LayerQuantConfig.default_rpc_for_bits(4) == np.float32(0.2)
    assert K.LayerQuantConfig.default_rpc_for_bits(2) == np.float32(0.1)
    for bad in (K.LayerQuantConfig(0, 5, 2), K.LayerQuantConfig(0, 2, 2, -0.1, 0.1), K.LayerQuantConfig(0, 2, 2, group_size=0)):
        with pytest.raises(K.KvmixInvalidArgument):
            bad.validate()
        st = K.lib().kvmix_config_validate(C.byref(_lib.LayerConfigC(bad.layer_index, bad.key_bits, bad.value_bits,
                                                                      bad.key_rpc_ratio, bad.value_rpc_ratio,
                                                                      bad.group_size)))
        assert st == _lib.INVALID_ARGUMENT


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    with pytest.raises(K.KvmixCudaError):
        K.KVLayerCache(K.LayerQuantConfig(), 1, 1, 64)
    out = np.zeros(4, np.uint32)
    st = K.lib().kvmix_unpack(out.ctypes.data, 1, 2, out.ctypes.data, None)
    assert st == _lib.CUDA_ERROR


def test_config_roundtrip_and_format():
    cfg = K.tiered_config(32, 6)
    txt = K.write_config(cfg)
    lines = txt.splitlines()
    assert lines[:4] == ["kvmix-config v1", "provenance gradient-guided", "n_layers 32", "group_size 32"]
    assert lines[4] == "layer 0 key_bits 3 value_bits 4 key_rpc 0.2 value_rpc 0.2"
    assert lines[-1] == "layer 31 key_bits 2 value_bits 2 key_rpc 0.1 value_rpc 0.1"
    back = K.read_config(txt)
    assert back == cfg
    assert K.average_bits(cfg) == (2.1875, 2.375)  # acceptance criterion 1 (20% high tier)
    u = K.uniform_config(3, 4, 0.25, 64)
    assert K.read_config(K.write_config(u)) == u
    r = K.ModelQuantConfig(layers=u.layers, provenance=K.Provenance.kRandom, random_seed=99)
    assert "provenance random seed=99" in K.write_config(r)
    assert K.read_config(K.write_config(r)).random_seed == 99


def test_config_errors():
    with pytest.raises(K.KvmixRuntimeError, match="header"):
        K.read_config("nope v1\n")
    with pytest.raises(K.KvmixRuntimeError, match="missing provenance"):
        K.read_config("kvmix-config v1\nn_layers 1\n")
    with pytest.raises(K.KvmixRuntimeError, match="unknown directive"):
        K.read_config("kvmix-config v1\nprovenance uniform\nbogus 1\n")
    with pytest.raises(K.KvmixRuntimeError, match="n_layers says"):
        K.read_config("kvmix-config v1\nprovenance uniform\nn_layers 2\nlayer 0 key_bits 2 value_bits 2 key_rpc 0.1 value_rpc 0.1\n")
    with pytest.raises(K.KvmixRuntimeError, match="cache bit widths"):
        K.read_config("kvmix-config v1\nprovenance uniform\nlayer 0 key_bits 5 value_bits 2 key_rpc 0.1 value_rpc 0.1\n")
    with pytest.raises(K.KvmixRuntimeError, match="malformed"):
        K.read_config("kvmix-config v1\nprovenance uniform\nlayer 0 key_bits 2\n")
    # comments and blank lines are ignored
    ok = K.read_config("# hi\nkvmix-config v1 # c\n\nprovenance uniform\nlayer 0 key_bits 2 value_bits 3 key_rpc 0.5 value_rpc 1\n")
    assert ok.layers[0].value_bits == 3 and ok.layers[0].value_rpc_ratio == 1.0


def test_allocate_bits():
    # acceptance criterion 1 arithmetic: top floor(f*L) layers get the high tier
    rng = np.random.default_rng(11)
    km, vm = rng.uniform(0.01, 5.0, 32), rng.uniform(0.01, 5.0, 32)
    c20 = K.allocate_bits(km, vm, K.BitAllocationParams(high_fraction=0.2))
    c30 = K.allocate_bits(km, vm, K.BitAllocationParams(high_fraction=0.3))
    assert K.average_bits(c20) == (2.1875, 2.375) and K.average_bits(c30) == (2.28125, 2.5625)
    # ties break toward the lower layer index
    c = K.allocate_bits([1.0, 1.0, 1.0], [1.0, 1.0, 1.0], K.BitAllocationParams(high_fraction=0.34))
    assert [lc.key_bits for lc in c.layers] == [3, 2, 2]


def test_kvqg_host_roundtrip():
    """KVQG (de)serialisation is host logic; the golden bytes of test_quant.cpp:264-310."""
    golden = bytes([ord("K"), ord("V"), ord("Q"), ord("G"), 1, 2, 1, 0, 4, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0,
                    4, 0, 0, 0, 1, 0, 0, 0, 0, 0, 0, 0, 4, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 0, 0, 0, 0x00, 0x3C,
                    0x00, 0x00, 0xE4, 0, 0, 0])
    qg = K.deserialize_quantized_groups(golden, device="cpu")
    assert qg.spec.bits == 2 and qg.spec.group_size == 4 and qg.shape.d == 4
    assert K.serialize_quantized_groups(qg) == golden
    with pytest.raises(K.KvmixRuntimeError, match="magic"):
        K.deserialize_quantized_groups(b"X" + golden[1:], device="cpu")
    with pytest.raises(K.KvmixRuntimeError, match="truncated"):
        K.deserialize_quantized_groups(golden[:-1], device="cpu")
    with pytest.raises(K.KvmixRuntimeError, match="trailing"):
        K.deserialize_quantized_groups(golden + b"\0", device="cpu")
