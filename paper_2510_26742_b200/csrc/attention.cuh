// Parameter block of the tcgen05 flash-attention kernel (fattn.cu).
//
// Semantics follow the reference `Evaluator::attention` (proj/src/evaluate.cpp:225-252):
// per head h, P = softmax(Q_h K_{h % kv_heads}^T / sqrt(d)) with no mask, O_h = P V.
// Keys/values are the row-concatenation of two segments, which is how `ae.kcat` /
// `ae.vcat` (proj/src/builder.cpp:321-329) are consumed without materialising the concat.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace pi0b {

struct AttnParams {
    const __nv_bfloat16* q;   // [q_rows, heads*d] (row stride ldq)
    long long ldq;
    int q_rows, heads, kv_heads;
    const __nv_bfloat16* k0;  // segment 0: [rows0, kv_heads*d] keys, values
    const __nv_bfloat16* v0;
    long long ld0;
    int rows0;
    int rows0_valid;          // keys [rows0_valid, rows0) of segment 0 are padding and masked (<= 0: none):
                              // a prefix padded to a 32-row multiple ahead of a second segment
    const __nv_bfloat16* k1;  // segment 1 (rows1 may be 0)
    const __nv_bfloat16* v1;
    long long ld1;
    int rows1;
    float scale_log2;         // log2(e) / sqrt(d)
    __nv_bfloat16* out;       // [q_rows, heads*d]
    long long ldo;
    int kv_splits;            // grid.y = key splits (1, 2, 4, 8): a (1, S, 1) cluster per q tile,
                              // partials exchanged through `ws` (attention_ws_bytes) + a cluster barrier
    void* ws;                 // key-split workspace (kv_splits > 1)
    int kv_per_split;         // informational: keys per split
};

// Tensor maps of one attention launch (fattn.cu make_fattn_maps): Q [q_rows, heads*d] and the two
// key / value segments [rows, kv_heads*d], bf16, boxes of 64 columns x 32 (Q; K/V of two segments)
// or 64 rows (K/V of one segment), 128-byte swizzle.
// Bytes of the key-split workspace of one launch (0 when kv_splits <= 1).
inline long long attention_ws_bytes(const AttnParams& p, int head_dim) {
    const int S = p.kv_splits > 1 ? p.kv_splits : 1;
    if (S == 1) return 0;
    const int dv = head_dim == 72 ? 128 : head_dim;  // fattn.cu DV (PV width)
    const long long grows = (long long)(p.heads / p.kv_heads) * p.q_rows;
    const long long tiles = (grows + 127) / 128 * p.kv_heads;
    const long long blk = (128 / S) * (2LL * dv + 8);
    return tiles * S * S * blk;
}

struct FaMaps {
    CUtensorMap q, k0, v0, k1, v1;
    int kv_box;  // key rows per K/V box: 64 (one key segment) or 32 (a tile may straddle two)
};

}  // namespace pi0b
