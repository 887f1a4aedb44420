// Whole-graph timeline instrumentation (variant builds only, -DPI0B_KTRACE;
// scripts/graph_timeline.py).  Every CTA of an instrumented kernel appends one record
// {tag, t_start, t_dep, t_end} (globaltimer ns) to the buffer set by pi0b_ktrace_buffer():
// t_dep = when its producer thread returned from griddepcontrol.wait (0 if it never waited).
// buffer[0] is the record counter shared by every translation unit.
#pragma once

#ifdef PI0B_KTRACE
namespace pi0b {
namespace {
__device__ unsigned long long* g_kt;  // one copy per translation unit; all point at one buffer
}
}  // namespace pi0b
// t_dep goes through a per-CTA-index slot past the records (written after griddepcontrol.wait,
// read and cleared at exit: the next kernel of the chain writes it only after this one completed).
constexpr unsigned long long kKtDepBase = 8 + 4 * 262144ull;
#define KT_BLOCK_ (blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z))
#define KT_SMEM unsigned long long kt_t0_ = 0
#define KT_START()                                                                             \
    do {                                                                                       \
        if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(kt_t0_));       \
    } while (0)
#define KT_DEP()                                                                               \
    do {                                                                                       \
        if (g_kt) {                                                                            \
            unsigned long long t_;                                                             \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                             \
            g_kt[kKtDepBase + KT_BLOCK_] = t_;                                                 \
        }                                                                                      \
    } while (0)
#define KT_END(tag)                                                                            \
    do {                                                                                       \
        if (threadIdx.x == 0 && g_kt) {                                                        \
            unsigned long long t_;                                                             \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                             \
            const unsigned long long i_ = atomicAdd(g_kt, 1ull);                               \
            unsigned long long* r_ = g_kt + 8 + 4 * i_;                                        \
            r_[0] = (tag);                                                                     \
            r_[1] = kt_t0_;                                                                    \
            r_[2] = g_kt[kKtDepBase + KT_BLOCK_];                                              \
            r_[3] = t_;                                                                        \
            g_kt[kKtDepBase + KT_BLOCK_] = 0;                                                  \
        }                                                                                      \
    } while (0)
#define KT_SETTER(name)                                                                        \
    int name(unsigned long long* p) { return int(cudaMemcpyToSymbol(g_kt, &p, sizeof(p))); }
#else
#define KT_SMEM \
    do {        \
    } while (0)
#define KT_START() \
    do {           \
    } while (0)
#define KT_DEP() \
    do {         \
    } while (0)
#define KT_END(tag) \
    do {            \
    } while (0)
#define KT_SETTER(name) \
    int name(unsigned long long*) { return 0; }
#endif
