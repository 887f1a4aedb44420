// Parameter block of the tcgen05 GEMM + fused-epilogue kernel (gemm.cu).
//
// One launch computes, for every valid row r < M and column n < N,
//     z[r, n] = sum_k A[r, k] * W[n, k]          (bf16 x bf16 -> fp32 in TMEM)
// and then applies the epilogue of one reference graph node
// (proj/src/evaluate.cpp:160-223, EpilogueOp order RmsScale -> Bias -> Rope /
// Gelu / GeluGate / SiluBias -> Residual).  The weight W is stored [N, K]
// K-major (the reference's W[k, m] transposed once at pack time).
#pragma once

#include <stdint.h>

namespace pi0b {

enum GemmMode : int {
    kModeBf16 = 0,      // out(bf16) = act(rowscale*z + bias), optional RoPE / GELU
    kModeGate = 1,      // out(bf16)[:, j] = (s*z_up) * gelu(s*z_gate), tile-interleaved weights
    kModeF32Store = 2,  // out(fp32) = rowscale*z + bias; outb(bf16) copy; stats += out^2
    kModeResid = 3,     // out(fp32) += scale*(rowscale*z + bias) in place; outb; stats
    kModeSiluTable = 4, // out(bf16) = silu(z + table_row)
};

// Split-K factor limit: the splits of a tile form one (portable-size) thread-block cluster.
constexpr int kGemmMaxSplits = 8;

enum GemmFlags : int {
    kFlagRowScale = 1,  // multiply row r by 1/sqrt(row_stats[r]*inv_width + eps)
    kFlagBias = 2,
    kFlagGelu = 4,
    kFlagRope = 8,      // rotate pairs (j, j+128) of every 256-wide head in cols < rope_cols
    kFlagRopePacked = 16,  // bn = 128 over kPermRope-packed weights: a tile = 64 columns of one head
                           // followed by their 64 RoPE partners (written back to j and j + 128)
    kFlagWarmEpi = 32,     // set by launch_gemm: run the epilogue once "dry" during the mainloop
    kFlagStageBf16 = 64,   // set by launch_gemm: bf16 tiles staged in smem, written as whole rows
};

struct GemmParams {
    int M, N, K;
    int splits;               // split-K factor (grid.z = cluster size, 1..kGemmMaxSplits)
    int kb_per_split;         // 64-wide k-blocks per split
    int mode, flags;
    const float* row_stats;   // [M] sum of squares of the A rows (RmsStats node)
    float inv_width, eps;
    const float* bias;        // [N]
    const float* table_row;   // [N] SiluBias row for this flow step
    const float* rope_cs;     // [positions][128] x {cos, sin}
    int rope_pos0, rope_cols;
    float resid_scale;
    void* out;                // bf16 or fp32, leading dimension ldo (elements)
    long long ldo;
    void* outb;               // bf16 shadow of an fp32 output
    long long ldob;
    float* out_stats;         // [M] += sum over written columns of out^2
    const float* row0_src;    // kModeF32Store: also write row -1 from this fp32 row
    int persist;              // 1: one CTA per SM walks the tiles (splits == 1), TMEM double buffer
    int mt;                   // 128-row m-tiles per CTA (1, or 2 with bn = 256 and splits == 1)
    int cg;                   // 2: CTA-pair tcgen05 (cta_group::2) 256 x 256 tiles (bn = 256, splits == 1,
                              //    weight tensor map box = 128 rows)
};

}  // namespace pi0b
