// Microbenchmark: DRAM efficiency of the radix pass's write pattern.  A tile of
// 256*L keys is read coalesced and written as 256 runs of L keys, run d of tile t
// at bucket region d (regions n/256 keys apart), position t*L — the output pattern
// of a radix-256 pass on uniform digits with tiles of 256*L keys.  "inplace"
// writes the tile back contiguously instead (the aligned-store ablation).  Each
// thread keeps 16 loads in flight.
#include <cstdio>
#include <cuda_runtime.h>

template <int LG>
__global__ void __launch_bounds__(256) k_runs(const unsigned* __restrict__ src, unsigned* __restrict__ dst, size_t n,
                                              int inplace, int misalign) {
    constexpr int L = 1 << LG;
    const size_t tile_keys = 256ull * L;
    const size_t ntiles = n / tile_keys;
    const size_t region = n / 256;
    for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const unsigned* s = src + t * tile_keys;
        for (int b0 = 0; b0 < (int)tile_keys; b0 += 256 * 16) {
            unsigned v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = (b0 + j * 256 < (int)tile_keys) ? __ldcs(s + b0 + j * 256 + threadIdx.x) : 0u;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int b = b0 + j * 256 + threadIdx.x;
                if (b >= (int)tile_keys) break;
                size_t g;
                if (inplace) g = t * tile_keys + b;
                else g = (size_t)(b >> LG) * region + t * L + (b & (L - 1)) + (misalign ? ((b >> LG) * 3) & 31 : 0);
                __stcs(dst + g, v[j]);
            }
        }
    }
}

template <int LG>
void run(const unsigned* a, unsigned* b, size_t n, int inplace, int mis, int grid) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_runs<LG><<<grid, 256>>>(a, b, n, inplace, mis);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_runs<LG><<<grid, 256>>>(a, b, n, inplace, mis);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    printf("%s%s L=%4d (run %5d B) grid %4d: %.3f ms  %.0f GB/s\n", inplace ? "inplace" : "runs   ", mis ? "+mis" : "    ",
           1 << LG, 4 << LG, grid, ms, (double)n * 8 / ms / 1e6);
}

int main() {
    const size_t n = 1ull << 30;
    unsigned *a, *b;
    cudaMalloc(&a, n * 4);
    cudaMalloc(&b, n * 4 + 4096);
    cudaMemset(a, 1, n * 4);
    for (int grid : {296, 592, 1184}) {
        run<7>(a, b, n, 1, 0, grid);
        run<4>(a, b, n, 0, 0, grid);
        run<5>(a, b, n, 0, 0, grid);
        run<6>(a, b, n, 0, 0, grid);
        run<7>(a, b, n, 0, 0, grid);
        run<8>(a, b, n, 0, 0, grid);
        run<9>(a, b, n, 0, 0, grid);
        run<10>(a, b, n, 0, 0, grid);
        run<6>(a, b, n, 0, 1, grid);
        run<7>(a, b, n, 0, 1, grid);
        run<8>(a, b, n, 0, 1, grid);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
