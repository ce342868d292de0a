"""Toy decoder through the device caches (test_toymodel.cpp:290-324):
a full-precision cache (r = 1) decodes token-identically to the no-cache recompute oracle,
prefill == stepwise, and a KVmix cache stays close to full precision."""
import pytest
import torch

import paper_2506_08018_b200 as K
from paper_2506_08018_b200 import decoder as T

HP = T.ToyHyperparams(vocab_size=256, d_model=256, n_layers=4, n_heads=4, head_dim=64, d_ff=512, max_seq=128)


@pytest.mark.gpu
def test_full_precision_decode_matches_recompute(cuda):
    m = T.ToyTransformer.random(HP, seed=3)
    prompt = [5, 17, 99, 3, 250]
    got = T.generate(m, prompt, 40)
    ref = T.generate_recompute_reference(m, prompt, 40)
    assert got == ref


@pytest.mark.gpu
def test_prefill_equals_stepwise(cuda):
    m = T.ToyTransformer.random(HP, seed=4)
    toks = [1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11]
    a = T.CachedDecoder(m)
    la = a.prefill(toks)
    b = T.CachedDecoder(m)
    for t in toks:
        lb = b.step(t)
    assert a.position() == b.position() == len(toks)
    assert torch.allclose(la, lb, rtol=1e-4, atol=1e-4)
    # both continue identically through the cache
    assert torch.allclose(a.step(42), b.step(42), rtol=1e-4, atol=1e-4)
    assert a.layer_cache(0).total_tokens() == len(toks) + 1


@pytest.mark.gpu
def test_kvmix_cache_decode_tracks_full_precision(cuda):
    m = T.ToyTransformer.random(HP, seed=5)
    quant = K.tiered_config(HP.n_layers, 1)  # layer 0 K3/V4 r=0.2, the rest K2/V2 r=0.1
    fp, q = T.CachedDecoder(m), T.CachedDecoder(m, quant)
    toks = [7, 100, 31, 64] + list(range(40, 100))
    cos, agree = [], 0
    for t in toks:
        a, b = fp.step(t), q.step(t)
        cos.append(float(torch.nn.functional.cosine_similarity(a, b, dim=0)))
        agree += int(torch.argmax(a) == torch.argmax(b))
    assert min(cos) > 0.9
    assert agree >= 0.6 * len(toks)
    assert q.layer_cache(1).memory_usage().packed_payload_bits > 0  # the packed cache was used


def test_decoder_cpu_oracle_and_errors():
    hp = T.ToyHyperparams(vocab_size=32, d_model=64, n_layers=2, n_heads=2, head_dim=32, d_ff=64, max_seq=16)
    m = T.ToyTransformer.random(hp, seed=1, device="cpu")
    out = T.generate_recompute_reference(m, [1, 2, 3], 5)
    assert len(out) == 8 and all(0 <= t < 32 for t in out)
    logits, keys, values = T.causal_forward(m, [1, 2, 3])
    assert logits.shape == (32,) and keys[0].shape == (1, 2, 3, 32) and len(values) == 2
    with pytest.raises(ValueError):
        T.causal_forward(m, [40])
    with pytest.raises(ValueError):
        T.ToyHyperparams(d_model=64, n_heads=3, head_dim=16).validate()
    with pytest.raises(ValueError):
        T.generate(m, [], 3)
