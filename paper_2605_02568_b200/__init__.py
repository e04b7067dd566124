"""B200-native CSA lightning indexer (arXiv 2605.02568, StreamIndex).

Hot path: score I(t,s) = sum_h w[t,h] * relu(q[t,h] . K[s]) -> causal mask ->
per-query top-k, on sm_100a through the C-ABI in include/csaidx_cuda.h.
"""
