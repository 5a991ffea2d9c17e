// Device helpers shared by the rsort kernels (sm_100a): PTX wrappers for
// relaxed GPU-scope status words, mbarrier + 1-D bulk (TMA engine) copies, lane masks.
#pragma once

// programmatic dependent launch along the radix-256 sort's kernel chain K1 -> K2 ->
// K3 x P -> K4 (0 = plain launches).  Each kernel of the chain waits (pdl_wait) before
// its first global access, so a launch may be scheduled while its predecessor drains;
// the wait returns once the predecessor grid has completed and its writes are visible.
#ifndef RS_PDL
#define RS_PDL 1
#endif
#include <cstdint>
#include <cuda_runtime.h>
#include <utility>

namespace rs {
__device__ __forceinline__ void pdl_wait() {
#if RS_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
// lets the next kernel of the chain launch; issued only by grids whose CTAs are all
// resident at once (persistent or one wave), so a waiting dependent never holds a
// slot one of this grid's CTAs still needs
__device__ __forceinline__ void pdl_trigger() {
#if RS_PDL
    asm volatile("griddepcontrol.launch_dependents;" :::);
#endif
}
// launch with the programmatic-serialisation attribute when pdl (and RS_PDL) is set
template <typename... KP, typename... A>
inline cudaError_t launch_chain(bool pdl, void (*kern)(KP...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                A&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (RS_PDL && pdl) ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...);
}
}  // namespace rs

// Checked builds (-DRS_CHECKED, tests only): bounds asserts on computed store
// indices (compute-sanitizer is not available on the GPU pool).
#ifdef RS_CHECKED
#include <cassert>
#define RS_DCHECK(cond) assert(cond)
#else
#define RS_DCHECK(cond) ((void)0)
#endif

namespace rs {

constexpr int kMaxPasses = 16;

// ----------------------------------------------------------------- lanes --
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
__device__ __forceinline__ uint32_t lanemask_gt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_gt;" : "=r"(m));
    return m;
}

// named barrier over `count` threads (a multiple of 32) of the CTA
__device__ __forceinline__ void named_barrier_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// ------------------------------------------------ GPU-scope status words --
// Look-back status words pack flag and value in one 32-bit word, so a single
// relaxed access is atomic; no ordering with other data is needed.
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_gpu(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_gpu(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_gpu(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ------------------------------------------------ mbarrier + bulk copies --
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
// 1-D bulk copy global -> shared through the TMA engine; completion counted on `bar`.
// dst, src 16-byte aligned; bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// 1-D bulk copy shared -> global through the TMA engine (bulk async-group of the
// issuing thread).  dst, src 16-byte aligned; bytes a multiple of 16.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// this thread's bulk stores have finished reading shared memory
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// this thread's bulk stores are complete
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// prefetch `bytes` (multiple of 16) at 16-byte aligned `src` into L2 through the TMA engine
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// lanes of this warp whose 8-bit digit d equals mine, from 8 ballots
__device__ __forceinline__ uint32_t peers8(uint32_t d) {
    // Lanes that disagree with me on bit b are the set bits of ballot(bit b) ^ s_b,
    // s_b = my bit b as 0 / 0xffffffff; peers = ~OR_b(...).  s_b in one PRMT: a
    // multiply by 0x10204080 moves nibble bit i to the MSB of byte i, and PRMT's
    // sign-replicate selector broadcasts that MSB to all four bytes.
    uint32_t dis;
    asm("{\n"
        ".reg .pred p;\n"
        ".reg .b32 t, s, m, ylo, yhi;\n"
        "and.b32 t, %1, 15;\n"
        "mul.lo.u32 ylo, t, 0x10204080;\n"
        "shr.u32 t, %1, 4;\n"
        "mul.lo.u32 yhi, t, 0x10204080;\n"
        "mov.b32 %0, 0;\n"
#define RS_PEER_BIT(B, Y, SEL)                     \
    "and.b32 t, %1, " #B ";\n"                    \
    "setp.ne.u32 p, t, 0;\n"                      \
    "vote.sync.ballot.b32 m, p, 0xffffffff;\n"    \
    "prmt.b32 s, " #Y ", 0, " #SEL ";\n"          \
    "xor.b32 m, m, s;\n"                          \
    "or.b32 %0, %0, m;\n"
        RS_PEER_BIT(1, ylo, 0x8888) RS_PEER_BIT(2, ylo, 0x9999)
        RS_PEER_BIT(4, ylo, 0xAAAA) RS_PEER_BIT(8, ylo, 0xBBBB)
        RS_PEER_BIT(16, yhi, 0x8888) RS_PEER_BIT(32, yhi, 0x9999)
        RS_PEER_BIT(64, yhi, 0xAAAA) RS_PEER_BIT(128, yhi, 0xBBBB)
#undef RS_PEER_BIT
        "}\n"
        : "=r"(dis)
        : "r"(d));
    return ~dis;
}

// ------------------------------------------------------------ key traits --
template <typename K>
__device__ __forceinline__ uint32_t digit_of(K k, int shift, uint32_t mask) {
    return static_cast<uint32_t>(k >> shift) & mask;
}
template <>
__device__ __forceinline__ uint32_t digit_of<uint32_t>(uint32_t k, int shift, uint32_t mask) {
    return (k >> shift) & mask;
}

}  // namespace rs
