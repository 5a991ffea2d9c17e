// Minimal 1-D TMA tensor store check: 64 u32 from shared memory to global
// coordinate X (element-granular), tensor map as a __grid_constant__ parameter.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__global__ void k(const __grid_constant__ CUtensorMap m, int x, int box) {
    __shared__ __align__(128) unsigned s[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s[i] = 1000 + i;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(s + (box == 4 ? 4 : 0)));
        asm volatile("cp.async.bulk.tensor.1d.global.shared::cta.bulk_group [%0, {%1}], [%2];" ::"l"(&m), "r"(x),
                     "r"(sa)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const size_t n = 1 << 20;
    unsigned* b;
    cudaMalloc(&b, n * 4);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    for (int box : {64, 4}) {
        for (int x : {0, 5, 1001}) {
            cudaMemset(b, 0, n * 4);
            CUtensorMap m;
            cuuint64_t dim[1] = {n}, stride[1] = {4};
            cuuint32_t bx[1] = {(cuuint32_t)box}, es[1] = {1};
            CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 1, b, dim, stride, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            k<<<1, 128>>>(m, x, box);
            cudaError_t e = cudaDeviceSynchronize();
            unsigned h[80];
            cudaMemcpy(h, b + (x > 8 ? x - 8 : 0), sizeof(h), cudaMemcpyDeviceToHost);
            printf("box %d x %d: encode %d, %s; around x:", box, x, (int)r, cudaGetErrorString(e));
            for (int i = 0; i < 12; ++i) printf(" %u", h[(x > 8 ? 8 : x) - 2 + i + 2]);
            printf("\n");
            if (e != cudaSuccess) return 1;
        }
    }
    return 0;
}
