// Microbenchmark: the radix pass's [store] phase with element-granular TMA tensor
// stores vs warp-contiguous STG.  A tile of 256 bucket runs (lengths around L,
// varying) sits in shared memory, each run starting on a 16-byte boundary; run d
// goes to bucket region d at a destination with arbitrary 4-byte alignment.
//   mode 0: STG — each warp stores 32 consecutive tile slots per instruction
//           (the current kernel's store, with its per-slot bucket lookup)
//   mode 1: TMA — thread d stores its run with 1-D tensor stores of 64/32/16/8/4
//           keys (binary decomposition, coordinates in elements) + STG for the
//           last len % 4 keys
// The tile is loaded once per tile from global memory (coalesced), as in the pass.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmarun tmarun.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

constexpr int R = 256;
constexpr int T = 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

struct Maps {
    CUtensorMap m[5];  // box 64, 32, 16, 8, 4 keys
};

template <int MODE, int ALIGN, int MINBOX>
__global__ void __launch_bounds__(T) k_store(const __grid_constant__ Maps maps, const unsigned* __restrict__ src,
                                             unsigned* __restrict__ dst, const unsigned* __restrict__ runlen,
                                             size_t ntiles, size_t region, int tile_cap) {
    extern __shared__ __align__(128) unsigned sm[];
    __shared__ unsigned s_start[R + 1], s_len[R];
    __shared__ unsigned long long s_g[R];
    unsigned char* s_bkt = reinterpret_cast<unsigned char*>(sm + tile_cap);  // slot -> bucket (mode 0)
    const int tid = threadIdx.x;
    for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        // run lengths of this tile (a fixed pseudo-random pattern per tile), 4-aligned starts
        {
            const unsigned len = runlen[(t * R + tid) % (R * 64)];
            unsigned a = (len + ALIGN - 1) & ~(unsigned)(ALIGN - 1), incl = a;
            for (int d = 1; d < 32; d <<= 1) {
                unsigned y = __shfl_up_sync(0xffffffffu, incl, d);
                if ((tid & 31) >= d) incl += y;
            }
            __shared__ unsigned s_w[8];
            if ((tid & 31) == 31) s_w[tid >> 5] = incl;
            __syncthreads();
            unsigned wb = 0;
            for (int w = 0; w < (tid >> 5); ++w) wb += s_w[w];
            s_start[tid] = wb + incl - a;
            s_len[tid] = len;
            // destination: region d, position t*avg + misalignment (arbitrary 4-byte alignment)
            s_g[tid] = (unsigned long long)tid * region + t * 96 + ((tid * 7 + t * 3) & 31);
            if (tid == R - 1) s_start[R] = wb + incl;
            __syncthreads();
            if (MODE == 0)
                for (unsigned i = 0; i < a; ++i) s_bkt[wb + incl - a + i] = (unsigned char)tid;
        }
        const int total = (int)s_start[R];
        // load the tile (coalesced, 8 in flight)
        const unsigned* s = src + t * (size_t)tile_cap;
        for (int b = tid; b < total; b += T * 8) {
            unsigned v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = b + j * T < total ? __ldcs(s + b + j * T) : 0u;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (b + j * T < total) sm[b + j * T] = v[j];
        }
        if (MODE == 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (MODE == 0) {
            // warp-contiguous store as in the pass: slot i's bucket from a per-slot table
            // (the pass reads it from the key's digit), its offset from shared memory
            for (int i = tid; i < total; i += T) {
                const unsigned d = s_bkt[i];
                const unsigned off = i - s_start[d];
                if (off < s_len[d]) __stcs(dst + s_g[d] + off, sm[i]);
            }
        } else {
            const unsigned len = s_len[tid], st = s_start[tid];
            const unsigned long long g = s_g[tid];
            unsigned done = 0;
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                const unsigned box = 64u >> k;
                if ((int)box < MINBOX) break;
                while (len - done >= box) {
                    const int x = (int)(g + done);
                    asm volatile("cp.async.bulk.tensor.1d.global.shared::cta.bulk_group [%0, {%1}], [%2];"
                                 ::"l"(&maps.m[k]), "r"(x), "r"(smem_u32(sm + st + done))
                                 : "memory");
                    done += box;
                    if (k > 0) break;  // after the 64-key chunks each smaller box is used at most once
                }
            }
            for (; done < len; ++done) __stcs(dst + g + done, sm[st + done]);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        __syncthreads();
    }
    if (MODE == 1) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const size_t n = 1ull << 30;
    unsigned *a, *b, *rl;
    cudaMalloc(&a, n * 4);
    cudaMalloc(&b, n * 4 + (1 << 20));
    cudaMemset(a, 1, n * 4);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    if (!enc) {
        printf("no cuTensorMapEncodeTiled\n");
        return 1;
    }
    Maps maps;
    for (int k = 0; k < 5; ++k) {
        cuuint64_t dim[1] = {n + (1 << 18)}, stride[1] = {4};
        cuuint32_t box[1] = {64u >> k}, es[1] = {1};
        CUresult r = enc(&maps.m[k], CU_TENSOR_MAP_DATA_TYPE_UINT32, 1, b, dim, stride, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            printf("encode failed %d\n", (int)r);
            return 1;
        }
    }
    for (int L : {88, 40, 160}) {
        std::vector<unsigned> h(R * 64);
        unsigned x = 12345;
        for (auto& v : h) {  // lengths L/2 .. 3L/2
            x = x * 1664525u + 1013904223u;
            v = L / 2 + (x >> 8) % (L + 1);
        }
        cudaMalloc(&rl, h.size() * 4);
        cudaMemcpy(rl, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
        const int tile_cap = R * (3 * L / 2 + 32);
        const size_t ntiles = n / (size_t)tile_cap;
        const size_t region = n / R;
        // bytes actually moved: sum of run lengths over tiles
        double keys = 0;
        for (size_t t = 0; t < ntiles; ++t)
            for (int d = 0; d < R; ++d) keys += h[(t * R + d) % (R * 64)];
        const size_t smem = (size_t)tile_cap * 5;
        struct V { int mode, align, minbox; const char* name; void (*k)(Maps, const unsigned*, unsigned*, const unsigned*, size_t, size_t, int); };
        V vs[] = {{0, 4, 4, "STG a4", k_store<0, 4, 4>}, {1, 32, 32, "TMA a32 box>=32", k_store<1, 32, 32>},
                  {1, 4, 64, "TMA a4 box64", k_store<1, 4, 64>}, {1, 4, 4, "TMA a4 box>=4", k_store<1, 4, 4>}};
        for (auto& v : vs) {
            auto kern = v.k;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            for (int grid : {296}) {
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                kern<<<grid, T, smem>>>(maps, a, b, rl, ntiles, region, tile_cap);
                cudaEventRecord(e0);
                for (int r = 0; r < 5; ++r) kern<<<grid, T, smem>>>(maps, a, b, rl, ntiles, region, tile_cap);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                ms /= 5;
                cudaError_t err = cudaGetLastError();
                printf("L=%3d %-16s grid %3d: %.3f ms  %.0f GB/s (read+write)  %s\n", L, v.name, grid, ms,
                       keys * 8 / ms / 1e6, cudaGetErrorString(err));
                if (err != cudaSuccess) return 1;
            }
        }
        cudaFree(rl);
    }
    return 0;
}
