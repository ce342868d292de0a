"""Generate golden fixtures from the UNMODIFIED reference (oracle/_ref/libkvmix_ref.so).

Run in a container that has /root/reference (the library is built from its sources by
oracle/Makefile):   python tests/golden/make_golden.py
Writes tests/golden/golden.npz (+ golden.json index). The fixtures pin the CPU oracle
restatement (tests/test_oracle.py) and the GPU path (tests/test_*_gpu.py) without needing
/root/reference at test time.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402

QUANT_CASES = [
    # (seed, B, H, T, D, bits, gs, key)
    (1, 1, 2, 64, 48, 2, 32, True), (2, 1, 2, 64, 48, 3, 32, True), (3, 1, 2, 64, 48, 4, 32, True),
    (4, 2, 1, 96, 16, 3, 16, True), (5, 1, 1, 128, 64, 1, 64, True), (6, 1, 3, 7, 48, 3, 32, False),
    (7, 1, 2, 5, 48, 2, 32, False), (8, 2, 2, 9, 128, 4, 64, False), (9, 1, 1, 11, 33, 3, 8, False),
    (10, 1, 4, 32, 128, 3, 32, True), (11, 1, 4, 32, 128, 3, 32, False), (12, 1, 1, 1, 128, 2, 128, False),
]

CACHE_CASES = [
    # (seed, kbits, vbits, rk, rv, gs, B, H, D, chunks)
    (100, 2, 2, 0.1, 0.1, 32, 1, 2, 64, [300, 1, 1, 1, 40, 1, 70, 1]),
    (200, 3, 4, 0.2, 0.2, 32, 2, 2, 64, [129, 1, 1, 33, 1, 1, 64]),
    (300, 4, 3, 0.3, 0.15, 64, 1, 3, 64, [500, 7, 1, 1, 90]),
    (400, 3, 3, 0.05, 0.5, 32, 1, 1, 128, [96, 1, 1, 1, 1, 200]),
]


def main():
    assert O.ref_available(), "build oracle/_ref first (make -C oracle ref)"
    arrays, index = {}, {"quant": [], "cache": [], "rpc_target": [], "half": []}
    for i, (seed, B, H, T, D, bits, gs, key) in enumerate(QUANT_CASES):
        x = O.ref_random_h16(seed, (B, H, T, D), sigma=1.5, mu=0.25)
        w, m = O.ref_quantize(x, bits, gs, key)
        arrays[f"q{i}_x"], arrays[f"q{i}_words"], arrays[f"q{i}_meta"] = x, w, m
        index["quant"].append(dict(i=i, seed=seed, shape=[B, H, T, D], bits=bits, gs=gs, key=key))
    for i, (seed, kb, vb, rk, rv, gs, B, H, D, chunks) in enumerate(CACHE_CASES):
        rc = O.RefCache(kb, vb, rk, rv, gs, B, H, D)
        trace = []
        for s, t in enumerate(chunks):
            k = O.ref_random_h16(seed + 2 * s, (B, H, t, D))
            v = O.ref_random_h16(seed + 2 * s + 1, (B, H, t, D), sigma=2.0)
            rc.append(k, v)
            trace.append(dict(rc.counters(), **{k2: v2 for k2, v2 in rc.memory_usage().items()}))
        q = O.ref_random_h16(seed + 999, (B, H, 2, D), sigma=2.0)
        out, cs = rc.attend(q)
        rout, rcs = rc.attend(q, reference=True)
        dump = rc.dump()
        arrays[f"c{i}_q"], arrays[f"c{i}_attend"], arrays[f"c{i}_refattend"] = q, out, rout
        arrays[f"c{i}_dump"] = np.frombuffer(dump, np.uint8)
        ks, vs = rc.snapshot()
        arrays[f"c{i}_keys"], arrays[f"c{i}_values"] = ks, vs
        index["cache"].append(dict(i=i, seed=seed, kbits=kb, vbits=vb, rk=rk, rv=rv, gs=gs, B=B, H=H, D=D,
                                   chunks=chunks, trace=trace, checksum=cs, ref_checksum=rcs,
                                   dump_sha256=hashlib.sha256(dump).hexdigest()))
    R = O.ref()
    for n, r in [(10, 0.2), (25, 0.1), (0, 0.2), (201, 0.2), (7, 1.0), (10, float(np.float32(0.7))),
                 (1000, float(np.float32(0.1))), (4096, float(np.float32(0.1))), (8192, float(np.float32(0.2)))]:
        index["rpc_target"].append([n, r, int(R.ref_rpc_target(n, r))])
    for f in [1.0, 0.0, -0.0, 0.1, 65504.0, 65520.0, 1e-7, 6e-8, 2.5e-8, -3.0, 1e30, float("inf"), float("-inf")]:
        index["half"].append([f, int(R.ref_half_from_float(f))])
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(index, fh, indent=1)
    print("wrote", len(arrays), "arrays")


if __name__ == "__main__":
    main()
