"""B200-native Stream Generation Service hot path (StreamRL, arXiv 2504.15930).

The product is libsgs.so (C-ABI, include/sgs.h): hand-written sm_100a kernels
plus the host scheduler / dispatcher.  This package is its thin binding; it
raises ImportError-style errors when the library is missing instead of
falling back to anything else.
"""
from .sgs import (Instance, SgsError, comm_unique_id, dispatch_plan, elastic_plan, fit_profile, kv_pack, kv_unpack, lib,
                  op_argmax, op_decode_attention, op_decode_attention_timed, op_gemm, op_prefill_attention, op_rmsnorm, op_rope_append,
                  op_sample_top_p, op_silu_mul, rope_table, make_weights, tp_tail_plan, weight_tensors)

__all__ = ["Instance", "SgsError", "comm_unique_id", "dispatch_plan", "elastic_plan", "fit_profile", "kv_pack", "kv_unpack", "lib",
           "op_argmax", "op_decode_attention", "op_decode_attention_timed", "op_gemm", "op_prefill_attention", "op_rmsnorm", "op_rope_append",
           "op_sample_top_p", "op_silu_mul", "rope_table", "make_weights", "tp_tail_plan", "weight_tensors"]
