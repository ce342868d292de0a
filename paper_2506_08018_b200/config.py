"""Per-layer bit-allocation config: LayerQuantConfig / ModelQuantConfig and the
quant_config.txt format (cache.hpp:26-38, quant_config.hpp:17-53, profiler.cpp:104-123,
:162-267). Pure host logic; validation errors match the reference's messages."""
from __future__ import annotations

import dataclasses
import enum
import io
import math

import numpy as np

from ._lib import KvmixInvalidArgument, KvmixRuntimeError


class Provenance(enum.IntEnum):
    kGradientGuided = 0
    kRandom = 1
    kUniformBits = 2


def _f32(x) -> float:
    return float(np.float32(x))


@dataclasses.dataclass
class LayerQuantConfig:
    layer_index: int = 0
    key_bits: int = 2
    value_bits: int = 2
    key_rpc_ratio: float = 0.1
    value_rpc_ratio: float = 0.1
    group_size: int = 32

    def __post_init__(self):
        # the reference stores the ratios as float (cache.hpp:30-31)
        self.key_rpc_ratio = _f32(self.key_rpc_ratio)
        self.value_rpc_ratio = _f32(self.value_rpc_ratio)

    def __setattr__(self, name, value):
        if name in ("key_rpc_ratio", "value_rpc_ratio"):
            value = _f32(value)
        object.__setattr__(self, name, value)

    @staticmethod
    def default_rpc_for_bits(bits: int) -> float:
        """tier convention (cache.hpp:35): 3/4-bit layers keep 20%, 2-bit 10%."""
        return _f32(0.2) if bits >= 3 else _f32(0.1)

    def validate(self) -> None:
        """cache.cpp:14-28."""
        L = f"layer {self.layer_index}"
        if not (2 <= self.key_bits <= 4 and 2 <= self.value_bits <= 4):
            raise KvmixInvalidArgument(f"{L}: cache bit widths must be 2, 3 or 4")
        if not (0.0 <= self.key_rpc_ratio <= 1.0 and 0.0 <= self.value_rpc_ratio <= 1.0):
            raise KvmixInvalidArgument(f"{L}: rpc ratios must lie in [0, 1]")
        if self.group_size <= 0:
            raise KvmixInvalidArgument(f"{L}: group_size must be positive")


@dataclasses.dataclass
class ModelQuantConfig:
    layers: list = dataclasses.field(default_factory=list)
    provenance: Provenance = Provenance.kUniformBits
    random_seed: int = 0

    def validate(self) -> None:
        for i, lc in enumerate(self.layers):
            if lc.layer_index != i:
                raise KvmixInvalidArgument(f"ModelQuantConfig: layer {i} has index {lc.layer_index}")
            lc.validate()


def uniform_config(n_layers: int, bits: int, rpc_ratio: float, group_size: int = 32) -> ModelQuantConfig:
    cfg = ModelQuantConfig(provenance=Provenance.kUniformBits)
    cfg.layers = [LayerQuantConfig(i, bits, bits, rpc_ratio, rpc_ratio, group_size) for i in range(n_layers)]
    cfg.validate()
    return cfg


def full_precision_config(n_layers: int) -> ModelQuantConfig:
    """r = 1 keeps every token in the full-precision tail (quant_config.hpp:50-53)."""
    return uniform_config(n_layers, 4, 1.0)


@dataclasses.dataclass
class BitAllocationParams:
    high_fraction: float = 0.2
    high_key_bits: int = 3
    high_value_bits: int = 4
    low_bits: int = 2
    rpc_high: float = 0.2
    rpc_low: float = 0.1
    group_size: int = 32


def _top_set(scores, n_high):
    order = sorted(range(len(scores)), key=lambda i: -scores[i])  # stable: ties -> lower index
    high = [False] * len(scores)
    for i in order[:n_high]:
        high[i] = True
    return high


def allocate_bits(key_mean, value_mean, p: BitAllocationParams = BitAllocationParams()) -> ModelQuantConfig:
    """allocate_bits (profiler.cpp:104-112): the top floor(f*L) layers by mean importance get
    the high tier, independently for Keys and Values."""
    if p.high_fraction < 0.0 or p.high_fraction > 1.0:
        raise KvmixInvalidArgument("high_fraction must lie in [0, 1]")
    n = len(key_mean)
    n_high = int(math.floor(p.high_fraction * n))
    kh, vh = _top_set(list(key_mean), n_high), _top_set(list(value_mean), n_high)
    cfg = ModelQuantConfig(provenance=Provenance.kGradientGuided)
    for i in range(n):
        cfg.layers.append(LayerQuantConfig(i, p.high_key_bits if kh[i] else p.low_bits,
                                           p.high_value_bits if vh[i] else p.low_bits,
                                           p.rpc_high if kh[i] else p.rpc_low, p.rpc_high if vh[i] else p.rpc_low,
                                           p.group_size))
    return cfg


def average_bits(config: ModelQuantConfig) -> tuple[float, float]:
    """profiler.cpp:114-123."""
    if not config.layers:
        return 0.0, 0.0
    n = float(len(config.layers))
    return sum(lc.key_bits for lc in config.layers) / n, sum(lc.value_bits for lc in config.layers) / n


def tiered_config(n_layers: int, high_layers: int, group_size: int = 32) -> ModelQuantConfig:
    """The KVmix tiering the benchmarks use (acceptance.cpp:356-366): layers < high_layers at
    K3/V4 with r = 0.2, the rest K2/V2 with r = 0.1."""
    cfg = ModelQuantConfig(provenance=Provenance.kGradientGuided)
    for i in range(n_layers):
        hi = i < high_layers
        r = 0.2 if hi else 0.1
        cfg.layers.append(LayerQuantConfig(i, 3 if hi else 2, 4 if hi else 2, r, r, group_size))
    cfg.validate()
    return cfg


def _float_str(v: float) -> str:
    """std::to_chars(float): shortest round-trip, fixed vs scientific by length (fixed on ties)."""
    x = np.float32(v)
    fixed = np.format_float_positional(x, unique=True, trim="-")
    sci = np.format_float_scientific(x, unique=True, trim="-", exp_digits=2)
    return sci if len(sci) < len(fixed) else fixed


def write_config(config: ModelQuantConfig, os_=None) -> str:
    """write_config (profiler.cpp:162-184)."""
    out = io.StringIO()
    out.write("kvmix-config v1\nprovenance ")
    if config.provenance == Provenance.kGradientGuided:
        out.write("gradient-guided")
    elif config.provenance == Provenance.kRandom:
        out.write(f"random seed={config.random_seed}")
    else:
        out.write("uniform")
    out.write(f"\nn_layers {len(config.layers)}\n")
    out.write(f"group_size {config.layers[0].group_size if config.layers else 32}\n")
    for lc in config.layers:
        out.write(f"layer {lc.layer_index} key_bits {lc.key_bits} value_bits {lc.value_bits} key_rpc "
                  f"{_float_str(lc.key_rpc_ratio)} value_rpc {_float_str(lc.value_rpc_ratio)}\n")
    s = out.getvalue()
    if os_ is not None:
        os_.write(s)
    return s


def read_config(text) -> ModelQuantConfig:
    """read_config (profiler.cpp:194-267): same directives, same runtime_error messages."""
    if hasattr(text, "read"):
        text = text.read()
    cfg = ModelQuantConfig()
    declared_layers, declared_group = -1, -1
    saw_header = saw_prov = False

    def err(n, why):
        raise KvmixRuntimeError(f"config line {n}: {why}")

    def as_int(tok):
        try:
            return int(tok)
        except (TypeError, ValueError):
            return None

    def as_float(tok):
        try:
            return float(tok)
        except (TypeError, ValueError):
            return None

    for n, line in enumerate(text.split("\n"), 1):
        line = line.split("#", 1)[0]
        words = line.split()
        if not words:
            continue
        w = words[0]
        if not saw_header:
            if w != "kvmix-config" or len(words) < 2 or words[1] != "v1":
                err(n, "expected 'kvmix-config v1' header")
            saw_header = True
        elif w == "provenance":
            if len(words) < 2:
                err(n, "missing provenance kind")
            kind = words[1]
            if kind == "gradient-guided":
                cfg.provenance = Provenance.kGradientGuided
            elif kind == "uniform":
                cfg.provenance = Provenance.kUniformBits
            elif kind.startswith("random"):
                cfg.provenance = Provenance.kRandom
                if len(words) < 3 or not words[2].startswith("seed="):
                    err(n, "random provenance needs seed=<u64>")
                cfg.random_seed = int(words[2][5:])
            else:
                err(n, f"unknown provenance '{kind}'")
            saw_prov = True
        elif w == "n_layers":
            v = as_int(words[1]) if len(words) > 1 else None
            if v is None or v < 1:
                err(n, "bad n_layers")
            declared_layers = v
        elif w == "group_size":
            v = as_int(words[1]) if len(words) > 1 else None
            if v is None or v < 1:
                err(n, "bad group_size")
            declared_group = v
        elif w == "layer":
            f = words[1:]
            ok = len(f) >= 9 and f[1] == "key_bits" and f[3] == "value_bits" and f[5] == "key_rpc" and f[7] == "value_rpc"
            vals = (as_int(f[0]), as_int(f[2]), as_int(f[4]), as_float(f[6]), as_float(f[8])) if ok else None
            if not ok or any(v is None for v in vals):
                err(n, "malformed layer record")
            cfg.layers.append(LayerQuantConfig(vals[0], vals[1], vals[2], vals[3], vals[4],
                                               declared_group if declared_group > 0 else 32))
        else:
            err(n, f"unknown directive '{w}'")
    if not saw_header:
        raise KvmixRuntimeError("config: empty file or missing header")
    if not saw_prov:
        raise KvmixRuntimeError("config: missing provenance")
    if declared_layers >= 0 and declared_layers != len(cfg.layers):
        raise KvmixRuntimeError(f"config: n_layers says {declared_layers} but found {len(cfg.layers)} records")
    try:
        cfg.validate()
    except KvmixInvalidArgument as e:
        raise KvmixRuntimeError(f"config: {e}") from None
    return cfg
