// Host/device restatements of the reference's deterministic parameter streams
// (proj/src/tensor.cpp:7-47): SplitMix64, FNV-1a seed hashing, and the uniform
// draw lo + (hi - lo) * u with u = (x >> 11) * 2^-53, all evaluated in IEEE fp64
// without contraction so the device reproduces the host stream bit for bit.
// Plus the single-RNE fp64 -> bf16 rule used for every WEIGHT (gen_weights on the device and
// set_weight from a host WeightStore).  Activation inputs go through fp32 instead, because
// that is the engine's activation format: the prompt rows enter the fp32 residual stream
// (kernels_misc.cu rows_to_f32_kernel) and the image patches are converted as
// bf16(float(x)) (host: pi0b_f64_to_bf16_host / engine.cu host_bf16; device:
// f64_to_bf16_rows_kernel; bit-identical to each other).  bf16(float(x)) differs from the
// single-RNE rule only when x lies within 2^-29 relative of a bf16 rounding tie.
#pragma once

#include <math.h>
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define PI0B_HD __host__ __device__ __forceinline__
#else
#define PI0B_HD inline
#endif

namespace pi0b {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;

// Output n (0-based) of the SplitMix64 stream seeded with `seed`
// (Rng::next_u64 advances the state before mixing, proj/src/tensor.cpp:7-14).
PI0B_HD uint64_t splitmix_at(uint64_t seed, uint64_t n) {
    uint64_t z = seed + (n + 1) * kGolden;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// Element n of random_tensor(rows, cols, lo, hi, seed), row-major.
PI0B_HD double uniform_at(uint64_t seed, uint64_t n, double lo, double hi) {
    const double u = double(splitmix_at(seed, n) >> 11) * 0x1.0p-53;
#if defined(__CUDA_ARCH__)
    return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u));
#else
    volatile double span = hi - lo;  // keep the three roundings separate
    volatile double prod = span * u;
    return lo + prod;
#endif
}

// fp64 -> bf16 with a single round-to-nearest-even (no double rounding): truncate to
// fp32, OR in a sticky bit when inexact (round-to-odd), then RNE to bf16.
PI0B_HD uint16_t f64_to_bf16_bits(double x) {
    float f = float(x);
    if (fabs(double(f)) > fabs(x)) f = nextafterf(f, 0.0f);
    uint32_t u;
    memcpy(&u, &f, 4);
    if (double(f) != x) u |= 1u;
    u += 0x7fffu + ((u >> 16) & 1u);
    return uint16_t(u >> 16);
}

}  // namespace pi0b
