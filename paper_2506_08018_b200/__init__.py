"""paper_2506_08018_b200 -- B200-native KVmix mixed-precision KV-cache hot path.

The product is libkvmix_b200.so (hand-written sm_100a kernels behind the C ABI in
include/kvmix_b200.h). This package is the host-side mirror of the reference's C++ API
(/root/reference/proj/include/kvmix/{bitpack,quant,cache,quant_config,attention}.hpp):
same names, same argument meaning, same error behaviour, over torch CUDA tensors.
There is no CPU fallback: importing without the built library fails loudly.
"""
from ._lib import (KvmixCudaError, KvmixError, KvmixInvalidArgument, KvmixOutOfMemory, KvmixOutOfRange,
                   KvmixRuntimeError, launch_count, launch_count_of, lib, scratch_allocated, scratch_reset,
                   set_knob, tensor_core_launches)
from .quant import (GroupMeta, Grouping, PackedBuffer, PackLayout, QuantizedGroups, QuantSpec, TensorShape,
                    deserialize_quantized_groups, feat_per_word, kMixed3Block, mixed3_q_max, mixed3_wide_scale,
                    pack_mixed3, pack_uniform, packed_word_count, q_max_for_bits, quantize_key_tensor,
                    quantize_value_tensor, serialize_quantized_groups, unpack, unpack_mixed3, unpack_uniform)
from .config import (BitAllocationParams, LayerQuantConfig, ModelQuantConfig, Provenance, allocate_bits,
                     average_bits, full_precision_config, read_config, tiered_config, uniform_config, write_config)
from .cache import KVLayerCache, MemoryReport, rpc_target
from .attention import (AttentionOutput, DecodeStep, append_attend, append_attend_layers, attend, attend_layers, attention_inv_scale, dump_scores_csv, fused_pv,
                        fused_qk_scores, reference_attend, softmax_rows)

lib()  # fail at import time if the native library is missing

__all__ = [n for n in dir() if not n.startswith("_")]
