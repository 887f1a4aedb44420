// Non-GEMM kernels of the engine:
//   * gen_weight_kernel   - device-side `gen_weights` (proj/src/evaluate.cpp:38-75): every
//                           W[k, m] element of a weight instance is drawn from its own
//                           SplitMix64 counter and written, rounded to bf16, straight into
//                           the packed [N, K] K-major layout the GEMM consumes;
//   * pack_weight_kernel  - the same packing for host-supplied fp64 weights (WeightStore);
//   * gen_vector_kernel   - biases / bias-table rows as fp32;
//   * rows_to_f32_kernel  - fp64 input rows -> fp32 residual rows + bf16 shadow + row
//                           sum-of-squares (noise -> Euler state, prompt -> LLM rows);
//   * f64_to_bf16_kernel  - fp64 rows -> bf16 rows with a padded pitch (patches, state);
//   * f32_to_f64_kernel   - the [63, 32] action chunk back to fp64.
#include "numerics.cuh"
#include "ptx.cuh"
#include "veshard.cuh"

#include <algorithm>

namespace pi0b {

// Packed row of logical weight column j (0 <= j < m) — the weight layout the GEMMs consume.
//   kPermNone   identity;
//   kPermGate*  gated FFN weights [up | gate] (proj/src/passes.cpp:448) interleaved per tile:
//               tile t holds up columns [G t, G t + G) then the matching gate columns
//               (G = 128 for the 256-wide prefill tiles, 64 for the 128-row skinny tiles);
//   kPermRope   skinny qkv: inside every 256-wide head the RoPE partners (j, j + 128) land
//               64 rows apart in the same 128-row tile; columns >= rope_cols (V) stay put.
enum PackPerm { kPermNone = 0, kPermGate128 = 1, kPermGate64 = 2, kPermRope = 3 };

__host__ __device__ inline int packed_row(int j, int m, int perm, int rope_cols) {
    if (perm == kPermGate128 || perm == kPermGate64) {
        const int G = perm == kPermGate128 ? 128 : 64;
        const int half = m / 2;
        const bool gate = j >= half;
        const int c = gate ? j - half : j;
        return (c / G) * (2 * G) + (gate ? G : 0) + (c % G);
    }
    if (perm == kPermRope && j < rope_cols) {
        const int h = j >> 8, w = j & 255;
        const int part = w >> 7, i = w & 127;
        return (h << 8) + (i >> 6) * 128 + part * 64 + (i & 63);
    }
    return j;
}

// grid: (ceil(k/8 / 32), m) ; block 32 -> each thread emits 8 consecutive k of column j.
__global__ void gen_weight_kernel(__nv_bfloat16* dst, long long ldk, int k, int m, int perm, int rope_cols,
                                  uint64_t seed, double lo, double hi) {
    const int j = blockIdx.y;
    const int p0 = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
    if (p0 >= k) return;
    uint16_t v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int pp = p0 + i;
        v[i] = pp < k ? f64_to_bf16_bits(uniform_at(seed, uint64_t(pp) * m + j, lo, hi)) : 0;
    }
    uint16_t* out = reinterpret_cast<uint16_t*>(dst) + (long long)packed_row(j, m, perm, rope_cols) * ldk + p0;
    if (p0 + 8 <= k && (ldk % 8) == 0) {
        uint4 u;
        u.x = v[0] | (uint32_t(v[1]) << 16);
        u.y = v[2] | (uint32_t(v[3]) << 16);
        u.z = v[4] | (uint32_t(v[5]) << 16);
        u.w = v[6] | (uint32_t(v[7]) << 16);
        *reinterpret_cast<uint4*>(out) = u;
    } else {
        for (int i = 0; i < 8 && p0 + i < k; ++i) out[i] = v[i];
    }
}

// Host fp64 W[k, m] (already on device) -> packed bf16 [N, K].
__global__ void pack_weight_kernel(__nv_bfloat16* dst, long long ldk, const double* w, int k, int m,
                                   int perm, int rope_cols) {
    const int j = blockIdx.y;
    const int p0 = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
    if (p0 >= k) return;
    uint16_t* out = reinterpret_cast<uint16_t*>(dst) + (long long)packed_row(j, m, perm, rope_cols) * ldk + p0;
    for (int i = 0; i < 8 && p0 + i < k; ++i) out[i] = f64_to_bf16_bits(w[(long long)(p0 + i) * m + j]);
}

__global__ void gen_vector_kernel(float* dst, int n, uint64_t seed, double lo, double hi) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = float(uniform_at(seed, uint64_t(i), lo, hi));
}

__global__ void f64_to_f32_kernel(float* dst, const double* src, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = float(src[i]);
}

// One warp per row.
__global__ void rows_to_f32_kernel(const double* src, int rows, int cols, float* dst, long long ldd,
                                   __nv_bfloat16* dstb, long long lddb, float* stats) {
    const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    float ss = 0.f;
    for (int c = lane; c < cols; c += 32) {
        const float x = float(src[(long long)row * cols + c]);
        if (dst) dst[(long long)row * ldd + c] = x;
        if (dstb) dstb[(long long)row * lddb + c] = __float2bfloat16_rn(x);
        ss += x * x;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffff, ss, o);
    if (stats && lane == 0) stats[row] = ss;
}

// `host_bf16` (nullable): a device flag set when the host delivered the rows already converted,
// packed in `srcb` (Engine::stage_patches_bf16: a quarter of the bytes cross PCIe); then this is
// only the copy into the padded operand.
__global__ void f64_to_bf16_rows_kernel(const double* src, int rows, int cols, __nv_bfloat16* dst,
                                        long long ldd, const int* host_bf16, const __nv_bfloat16* srcb) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)rows * cols) return;
    const int r = int(i / cols), c = int(i % cols);
    dst[(long long)r * ldd + c] = (host_bf16 && *host_bf16) ? srcb[i] : __float2bfloat16_rn(float(src[i]));
}

__global__ void f32_to_f64_kernel(const float* src, long long lds, int rows, int cols, double* dst) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows * cols) return;
    dst[i] = double(src[(long long)(i / cols) * lds + (i % cols)]);
}

// Packed [rows, K] (pitch ldk) -> tile-contiguous [rows/128][K/64] blocks of 16 KB, each the exact
// Tile-contiguous copy of a packed [rows, k] weight for the action-expert megakernel: block
// (n_tile, kb) is the shared-memory image of a 64 x 64 operand tile in the 128-byte swizzle
// (16-byte chunk c of row r at (c ^ (r & 7))), zero-padded past `rows` / `k`.  The megakernel
// streams these with contiguous copies (a [64 x 64] box of the row-major weight is 64 pieces
// of 128 B at a K-element stride: poor DRAM locality).  order 1 ("paired", aemk.cuh
// AeTileOrder): tile 2T + s takes rows 128T + 32s + [0, 32) and their partners 64 rows later;
// order 2: plain 128-row tiles (16 KB blocks).
__global__ void tile_weight_kernel(const __nv_bfloat16* src, int rows, int k, long long ldk, __nv_bfloat16* dst,
                                   int kblocks, int order) {
    const long long tile = blockIdx.x;  // (n_tile * kblocks + kb)
    const int nt = int(tile / kblocks), kb = int(tile % kblocks);
    const int R = order == 2 ? 128 : 64;
    for (int q = threadIdx.x; q < R * 8; q += blockDim.x) {
        const int r = q >> 3, c = q & 7;
        const int row = order == 1 ? (nt >> 1) * 128 + (r >> 5) * 64 + (nt & 1) * 32 + (r & 31) : nt * R + r;
        const int col = kb * 64 + c * 8;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (row < rows && col < k) v = *reinterpret_cast<const uint4*>(src + (long long)row * ldk + col);
        *reinterpret_cast<uint4*>(dst + tile * (R * 64) + r * 64 + ((c ^ (r & 7)) << 3)) = v;
    }
}


// Image front-end: camera frames [views][H][W*C] (fp64, channels interleaved)
// -> half-pixel-centre bilinear resize to side x side (the reference's rtvla::bilinear_resize,
// proj/src/tensor.cpp:180-212, same fp64 operation order with FMA contraction disabled, so the
// resized values are bit-identical) -> img2col into the ve.embed input patches [views*g*g][P*P*C]
// (the reference draws `patches` at random and leaves the flattening unspecified; this engine's
// order: patch row t = view*g*g + (y / P)*g + (x / P), feature ((y % P)*P + (x % P))*C + c).
__global__ void image_patches_kernel(const double* img, int views, int H, int W, int C, int side, int P,
                                     double* patches) {
    const long long n = (long long)views * side * side * C;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int c = int(i % C);
    const int ox = int((i / C) % side);
    const int oy = int((i / ((long long)C * side)) % side);
    const int v = int(i / ((long long)C * side * side));
    auto clampd = [](double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); };
    const double sy = clampd(__dsub_rn(__ddiv_rn(__dmul_rn(oy + 0.5, double(H)), double(side)), 0.5), 0.0, double(H - 1));
    const double sx = clampd(__dsub_rn(__ddiv_rn(__dmul_rn(ox + 0.5, double(W)), double(side)), 0.5), 0.0, double(W - 1));
    const int y0 = int(sy), x0 = int(sx);
    const int y1 = min(y0 + 1, H - 1), x1 = min(x0 + 1, W - 1);
    const double ty = __dsub_rn(sy, double(y0)), tx = __dsub_rn(sx, double(x0));
    const double* im = img + (long long)v * H * W * C;
    const double v00 = im[((long long)y0 * W + x0) * C + c], v01 = im[((long long)y0 * W + x1) * C + c];
    const double v10 = im[((long long)y1 * W + x0) * C + c], v11 = im[((long long)y1 * W + x1) * C + c];
    const double top = __dadd_rn(v00, __dmul_rn(__dsub_rn(v01, v00), tx));
    const double bot = __dadd_rn(v10, __dmul_rn(__dsub_rn(v11, v10), tx));
    const double out = __dadd_rn(top, __dmul_rn(__dsub_rn(bot, top), ty));
    const int g = side / P;
    const long long t = (long long)v * g * g + (oy / P) * g + (ox / P);
    const int f = ((oy % P) * P + (ox % P)) * C + c;
    patches[t * (P * P * C) + f] = out;
}

// --------------------------------------------------------------------- launchers

cudaError_t launch_tile_weight(const __nv_bfloat16* src, int rows, int k, long long ldk, __nv_bfloat16* dst,
                               int order, cudaStream_t st) {
    const int R = order == 2 ? 128 : 64;
    const int kblocks = (k + 63) / 64, ntiles = (rows + R - 1) / R;
    tile_weight_kernel<<<ntiles * kblocks, 256, 0, st>>>(src, rows, k, ldk, dst, kblocks, order);
    return cudaGetLastError();
}

cudaError_t launch_gen_weight(__nv_bfloat16* dst, long long ldk, int k, int m, int perm, int rope_cols,
                              uint64_t seed, double lo, double hi, cudaStream_t st) {
    dim3 grid((k / 8 + 1 + 31) / 32, m);
    gen_weight_kernel<<<grid, 32, 0, st>>>(dst, ldk, k, m, perm, rope_cols, seed, lo, hi);
    return cudaGetLastError();
}
cudaError_t launch_pack_weight(__nv_bfloat16* dst, long long ldk, const double* w, int k, int m,
                               int perm, int rope_cols, cudaStream_t st) {
    dim3 grid((k / 8 + 1 + 31) / 32, m);
    pack_weight_kernel<<<grid, 32, 0, st>>>(dst, ldk, w, k, m, perm, rope_cols);
    return cudaGetLastError();
}
cudaError_t launch_gen_vector(float* dst, int n, uint64_t seed, double lo, double hi, cudaStream_t st) {
    gen_vector_kernel<<<(n + 255) / 256, 256, 0, st>>>(dst, n, seed, lo, hi);
    return cudaGetLastError();
}
cudaError_t launch_f64_to_f32(float* dst, const double* src, int n, cudaStream_t st) {
    f64_to_f32_kernel<<<(n + 255) / 256, 256, 0, st>>>(dst, src, n);
    return cudaGetLastError();
}
cudaError_t launch_rows_to_f32(const double* src, int rows, int cols, float* dst, long long ldd,
                               __nv_bfloat16* dstb, long long lddb, float* stats, cudaStream_t st) {
    rows_to_f32_kernel<<<(rows + 3) / 4, 128, 0, st>>>(src, rows, cols, dst, ldd, dstb, lddb, stats);
    return cudaGetLastError();
}
cudaError_t launch_f64_to_bf16_rows(const double* src, int rows, int cols, __nv_bfloat16* dst,
                                    long long ldd, cudaStream_t st, const int* host_bf16,
                                    const __nv_bfloat16* srcb) {
    const long long n = (long long)rows * cols;
    f64_to_bf16_rows_kernel<<<int((n + 255) / 256), 256, 0, st>>>(src, rows, cols, dst, ldd, host_bf16, srcb);
    return cudaGetLastError();
}
cudaError_t launch_f32_to_f64(const float* src, long long lds, int rows, int cols, double* dst,
                              cudaStream_t st) {
    f32_to_f64_kernel<<<(rows * cols + 255) / 256, 256, 0, st>>>(src, lds, rows, cols, dst);
    return cudaGetLastError();
}

cudaError_t launch_image_patches(const double* img, int views, int H, int W, int C, int side, int P, double* patches,
                                 cudaStream_t st) {
    if (views < 1 || H < 2 || W < 2 || C < 1 || side < P || side % P) return cudaErrorInvalidValue;
    const long long n = (long long)views * side * side * C;
    image_patches_kernel<<<int((n + 255) / 256), 256, 0, st>>>(img, views, H, W, C, side, P, patches);
    return cudaGetLastError();
}

}  // namespace pi0b

// ------------------------------------------------------------------ view-sharded vision encoder
// the VE attention is joint over every view's tokens (proj/src/builder.cpp:
// 219-222), so a view-sharded VE must all-gather each layer's q|k|v rows before the attention.
// One engine per shard (one per GPU); each pushes its own rows straight into every peer's
// gathered buffer (P2P stores over NVLink; peers' buffers mapped by CUDA IPC), then publishes a
// sequence number into each peer's flag slot with a system-scope release.  The receiving side's
// wait kernel polls its own flags with system-scope acquire loads.  Sequence number of step s of
// inference e: 64 e + s + 1 (monotone, so nothing is ever reset).
namespace pi0b {

__global__ void ve_push_kernel(const VePushArgs a) {
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
    for (int s = 0; s < a.nseg; ++s)
        for (long long i = tid; i < a.n16[s]; i += nth) {
            const uint4 v = __ldcg(a.src[s] + i);
            for (int p = 0; p < a.npeer; ++p) a.dst[p][s][i] = v;
        }
    __threadfence_system();  // this CTA's peer stores are visible system-wide
    __syncthreads();
    __shared__ unsigned last;
    if (threadIdx.x == 0) last = atomicAdd(a.done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last && threadIdx.x < a.npeer) {
        __threadfence_system();
        const unsigned v = 64u * *a.epoch + a.step + 1u;
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.flag[threadIdx.x]), "r"(v) : "memory");
        if (threadIdx.x == 0) *a.done = 0u;  // every CTA has arrived: ready for the next launch
    }
}

// Lane p waits until flags[p] (written by peer p) reaches this inference's sequence number for
// `step`; traps after ~10 s (a peer that never arrives) instead of hanging the GPU.
__global__ void ve_wait_kernel(const unsigned* flags, unsigned mask, const unsigned* epoch, unsigned step) {
    const int p = threadIdx.x;
    if (p >= 32 || !((mask >> p) & 1u)) return;
    const unsigned target = 64u * *epoch + step + 1u;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        unsigned v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + p) : "memory");
        if (int(v - target) >= 0) break;
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 10000000000ull) __trap();
        __nanosleep(200);
    }
}

__global__ void ve_epoch_kernel(unsigned* epoch) { *epoch += 1u; }

cudaError_t launch_ve_push(const VePushArgs& a, cudaStream_t st) {
    long long n = 0;
    for (int s = 0; s < a.nseg; ++s) n = n > a.n16[s] ? n : a.n16[s];
    const int blocks = int(std::min<long long>(64, (n + 255) / 256 + 1));
    ve_push_kernel<<<blocks, 256, 0, st>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_ve_wait(const unsigned* flags, unsigned mask, const unsigned* epoch, unsigned step, cudaStream_t st) {
    ve_wait_kernel<<<1, 32, 0, st>>>(flags, mask, epoch, step);
    return cudaGetLastError();
}
cudaError_t launch_ve_epoch(unsigned* epoch, cudaStream_t st) {
    ve_epoch_kernel<<<1, 1, 0, st>>>(epoch);
    return cudaGetLastError();
}

}  // namespace pi0b
