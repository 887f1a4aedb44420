// View-sharded vision encoder: the fused push + signal and the wait kernels
// (kernels_misc.cu), shared between the engine (engine.cu) and the kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pi0b {

struct VePushArgs {
    const uint4* src[3];       // own rows, 16-byte pieces
    uint4* dst[8][3];          // the same rows in each peer's buffers
    long long n16[3];
    int nseg, npeer;
    unsigned* flag[8];         // my flag slot in each peer's sync block
    const unsigned* epoch;     // own inference counter
    unsigned* done;            // own CTA arrival counter (the last CTA publishes)
    unsigned step;
};

// sync block of one shard: flags [8] (by source shard), inference counter, arrival counter
constexpr int kVeSyncWords = 16, kVeEpoch = 8, kVeDone = 9, kVeMaxShards = 8;

cudaError_t launch_ve_push(const VePushArgs& a, cudaStream_t st);
cudaError_t launch_ve_wait(const unsigned* flags, unsigned mask, const unsigned* epoch, unsigned step, cudaStream_t st);
cudaError_t launch_ve_epoch(unsigned* epoch, cudaStream_t st);

}  // namespace pi0b
