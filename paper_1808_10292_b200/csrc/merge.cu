// GSD step 5 ("Subsequences X_{k,j} ... are merged into Y_j
// using p-way merging"): the p received runs (source-rank order, each sorted)
// are merged by a tree of stable 2-way merge-path merges, ⌈log2 p⌉ levels, each
// level one read + one write of the data.  Ties go to the lower source rank
// (the left input of every merge), which keeps pair sorts globally stable
// (R16).
//
//   k_merge_split  one thread per output tile boundary: merge-path co-rank by
//                  binary search on the diagonal
//   k_merge_tile   one CTA per output tile: both input segments staged in
//                  shared memory, per-thread co-rank search + sequential merge of
//                  ITEMS outputs, coalesced store through shared memory
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "merge.h"

namespace rs {

#ifndef RS_MERGE_ITEMS
#define RS_MERGE_ITEMS 32  // measured at 2^31, p = 8: 8 -> 2.62, 16 -> 2.10, 24 -> 2.12, 32 -> 1.85, 48 -> 2.28, 64 -> 2.10 ms per rank
#endif
constexpr int kMT = 256;                 // threads per merge CTA
constexpr int kMItems = RS_MERGE_ITEMS;  // outputs per thread
constexpr int kMTile = kMT * kMItems;

// first i in [lo, hi] such that taking i elements of A and diag-i of B is a valid
// stable merge prefix (A wins ties)
template <typename K>
__device__ __forceinline__ size_t corank(const K* A, size_t na, const K* B, size_t nb, size_t diag) {
    size_t lo = diag > nb ? diag - nb : 0, hi = diag < na ? diag : na;
    while (lo < hi) {
        const size_t mid = (lo + hi) >> 1;
        if (A[mid] <= B[diag - 1 - mid]) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

template <typename K>
__global__ void k_merge_split(const K* __restrict__ A, size_t na, const K* __restrict__ B, size_t nb, size_t ntiles,
                              size_t d_base, size_t d_end, size_t* __restrict__ split) {
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t > ntiles) return;
    const size_t diag = min(d_base + t * (size_t)kMTile, d_end);
    split[t] = corank<K>(A, na, B, nb, diag);
}

// shared-memory index with one pad word per 32 (spreads the data-dependent
// merge reads over the banks)
__device__ __forceinline__ int mpad(int i) { return i + (i >> 5); }
constexpr int kMTilePad = kMTile + kMTile / 32 + 1;

template <typename K, bool V>
__global__ void __launch_bounds__(kMT) k_merge_tile(const K* __restrict__ A, const uint32_t* __restrict__ VA, size_t na,
                                                    const K* __restrict__ B, const uint32_t* __restrict__ VB, size_t nb,
                                                    const size_t* __restrict__ split, size_t d_base, size_t d_end,
                                                    K* __restrict__ out, uint32_t* __restrict__ vout) {
    // s_k: A segment then B segment (padded index); reused for the merged tile
    extern __shared__ __align__(16) unsigned char merge_smem[];
    K* s_k = reinterpret_cast<K*>(merge_smem);
    uint32_t* s_v = reinterpret_cast<uint32_t*>(merge_smem + (size_t)kMTilePad * sizeof(K));
    const size_t t = blockIdx.x;
    // merged positions [d0, d1) of the diagonal range [d_base, d_end) -> out[d - d_base]
    const size_t d0 = d_base + t * (size_t)kMTile, d1 = min(d0 + kMTile, d_end);
    const size_t a0 = split[t], a1 = split[t + 1];
    const size_t b0 = d0 - a0, b1 = d1 - a1;
    out += d0 - d_base;
    if (V) vout += d0 - d_base;
    const int la = (int)(a1 - a0), lb = (int)(b1 - b0), len = la + lb;
    // stage a segment: scalar head up to 16-byte alignment, 16-byte vector body, scalar tail
    auto stage = [&](const K* src, size_t s0, int l, int at) {
        constexpr int VE = 16 / sizeof(K);
        const int head = min(l, (int)((VE - (reinterpret_cast<uintptr_t>(src + s0) / sizeof(K)) % VE) % VE));
        const int nvec = (l - head) / VE;
        for (int i = threadIdx.x; i < head; i += kMT) s_k[mpad(at + i)] = src[s0 + i];
        const uint4* vb = reinterpret_cast<const uint4*>(src + s0 + head);
        for (int v = threadIdx.x; v < nvec; v += kMT) {
            const uint4 x = __ldcs(vb + v);
            const K* xs = reinterpret_cast<const K*>(&x);
#pragma unroll
            for (int e = 0; e < VE; ++e) s_k[mpad(at + head + v * VE + e)] = xs[e];
        }
        for (int i = head + nvec * VE + threadIdx.x; i < l; i += kMT) s_k[mpad(at + i)] = src[s0 + i];
    };
    stage(A, a0, la, 0);
    stage(B, b0, lb, la);
    if (V) {
        for (int i = threadIdx.x; i < la; i += kMT) s_v[mpad(i)] = VA[a0 + i];
        for (int i = threadIdx.x; i < lb; i += kMT) s_v[mpad(la + i)] = VB[b0 + i];
    }
    __syncthreads();
    auto KA = [&](int i) { return s_k[mpad(i)]; };
    auto KB = [&](int i) { return s_k[mpad(la + i)]; };
    const int diag = min((int)threadIdx.x * kMItems, len);
    int lo = diag > lb ? diag - lb : 0, hi = diag < la ? diag : la;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (KA(mid) <= KB(diag - 1 - mid)) lo = mid + 1;
        else hi = mid;
    }
    int ia = lo, ib = diag - lo;
    const int cnt = min(kMItems, len - diag);
    K ha = ia < la ? KA(ia) : K(0), hb = ib < lb ? KB(ib) : K(0);
    K ok[kMItems];
    uint32_t ov[V ? kMItems : 1];
#pragma unroll
    for (int o = 0; o < kMItems; ++o) {
        if (o < cnt) {
            const bool takeA = ib >= lb || (ia < la && ha <= hb);
            if (takeA) {
                ok[o] = ha;
                if (V) ov[o] = s_v[mpad(ia)];
                ++ia;
                ha = ia < la ? KA(ia) : K(0);
            } else {
                ok[o] = hb;
                if (V) ov[o] = s_v[mpad(la + ib)];
                ++ib;
                hb = ib < lb ? KB(ib) : K(0);
            }
        }
    }
    __syncthreads();  // segments consumed: reuse s_k / s_v for the merged tile
#pragma unroll
    for (int o = 0; o < kMItems; ++o)
        if (o < cnt) {
            s_k[mpad(diag + o)] = ok[o];
            if (V) s_v[mpad(diag + o)] = ov[o];
        }
    __syncthreads();
    // store: scalar head up to 16-byte alignment of the destination, vector body, scalar tail
    constexpr int VE = 16 / sizeof(K);
    const int mis = (int)((reinterpret_cast<uintptr_t>(out) / sizeof(K)) % VE);
    const int head = min(len, (VE - mis) % VE);
    const int nvec = (len - head) / VE;
    for (int i = threadIdx.x; i < head; i += kMT) out[i] = s_k[mpad(i)];
    uint4* vo = reinterpret_cast<uint4*>(out + head);
    for (int v = threadIdx.x; v < nvec; v += kMT) {
        uint4 x;
        K* xs = reinterpret_cast<K*>(&x);
#pragma unroll
        for (int e = 0; e < VE; ++e) xs[e] = s_k[mpad(head + v * VE + e)];
        RS_DCHECK(d0 + head + (size_t)v * VE + VE <= d_end);
        vo[v] = x;
    }
    for (int i = head + nvec * VE + threadIdx.x; i < len; i += kMT) out[i] = s_k[mpad(i)];
    if (V)
        for (int i = threadIdx.x; i < len; i += kMT) {
            RS_DCHECK(d0 + i < d_end);
            vout[i] = s_v[mpad(i)];
        }
}

// merged positions [lo, hi) of the stable merge of A and B (ties to A) -> out[0, hi - lo)
template <typename K, bool V>
static rs_status_t merge2_range(const K* A, const uint32_t* VA, size_t na, const K* B, const uint32_t* VB, size_t nb,
                                size_t lo, size_t hi, K* out, uint32_t* vout, size_t* split, cudaStream_t st) {
    if (hi <= lo) return RS_OK;
    const size_t ntiles = (hi - lo + kMTile - 1) / kMTile;
    {
        LaunchScope ls("merge_split", st);
        k_merge_split<K><<<(unsigned)((ntiles + 1 + 255) / 256), 256, 0, st>>>(A, na, B, nb, ntiles, lo, hi, split);
    }
    {
        const size_t smem = (size_t)kMTilePad * (sizeof(K) + (V ? 4 : 0));
        rs_status_t s = kernel_setup(reinterpret_cast<const void*>(k_merge_tile<K, V>), kMT, smem, nullptr);
        if (s != RS_OK) return s;
        LaunchScope ls("merge_tile", st);
        k_merge_tile<K, V><<<(unsigned)ntiles, kMT, smem, st>>>(A, VA, na, B, VB, nb, split, lo, hi, out, vout);
    }
    RS_CUDA_TRY(cudaGetLastError());
    return RS_OK;
}

template <typename K, bool V>
static rs_status_t merge2(const K* A, const uint32_t* VA, size_t na, const K* B, const uint32_t* VB, size_t nb, K* out,
                          uint32_t* vout, size_t* split, cudaStream_t st) {
    return merge2_range<K, V>(A, VA, na, B, VB, nb, 0, na + nb, out, vout, split, st);
}

size_t merge_scratch_bytes(size_t total) { return ((total + kMTile - 1) / kMTile + 2) * sizeof(size_t); }

// Tree of 2-way merges over runs [roff[k], roff[k+1]) of `runs` (k < p).  Level
// buffers alternate between `runs` and `tmp`; levels are arranged so that the
// last one writes `out`.  The runs buffer is clobbered.
template <typename K, bool V>
static rs_status_t merge_tree(K* runs, uint32_t* vruns, const std::vector<uint64_t>& roff, K* tmp, uint32_t* vtmp,
                              K* out, uint32_t* vout, size_t* split, cudaStream_t st) {
    const int p = (int)roff.size() - 1;
    const size_t total = roff[p];
    if (total == 0) return RS_OK;
    std::vector<uint64_t> off(roff.begin(), roff.end());
    int levels = 0;
    for (int q = p; q > 1; q = (q + 1) / 2) ++levels;
    if (levels == 0) {  // one run: it is Y_j
        RS_CUDA_TRY(cudaMemcpyAsync(out, runs, total * sizeof(K), cudaMemcpyDeviceToDevice, st));
        if (V) RS_CUDA_TRY(cudaMemcpyAsync(vout, vruns, total * 4, cudaMemcpyDeviceToDevice, st));
        return RS_OK;
    }
    K* src = runs;
    uint32_t* vsrc = vruns;
    K* other = tmp;
    uint32_t* vother = vtmp;
    for (int l = 0; l < levels; ++l) {
        const bool last = l == levels - 1;
        K* dst = last ? out : other;
        uint32_t* vdst = V ? (last ? vout : vother) : nullptr;
        const int q = (int)off.size() - 1;
        std::vector<uint64_t> noff;
        noff.push_back(0);
        for (int k = 0; k < q; k += 2) {
            const uint64_t a0 = off[k], a1 = off[k + 1];
            if (k + 1 < q) {
                const uint64_t b1 = off[k + 2];
                rs_status_t s = merge2<K, V>(src + a0, V ? vsrc + a0 : nullptr, a1 - a0, src + a1, V ? vsrc + a1 : nullptr,
                                             b1 - a1, dst + a0, V ? vdst + a0 : nullptr, split, st);
                if (s != RS_OK) return s;
                noff.push_back(b1);
            } else {  // odd run out: carried to the next level
                if (a1 > a0) {
                    RS_CUDA_TRY(cudaMemcpyAsync(dst + a0, src + a0, (a1 - a0) * sizeof(K), cudaMemcpyDeviceToDevice, st));
                    if (V)
                        RS_CUDA_TRY(cudaMemcpyAsync(vdst + a0, vsrc + a0, (a1 - a0) * 4, cudaMemcpyDeviceToDevice, st));
                }
                noff.push_back(a1);
            }
        }
        off.swap(noff);
        other = src;
        vother = vsrc;
        src = dst;
        vsrc = vdst;
    }
    return RS_OK;
}

// Tree whose level 0 reads p runs at arbitrary addresses (e.g. peers' sorted
// blocks over NVLink, mapped by CUDA IPC): level 0 merges run pairs into a level
// buffer, later levels alternate between `out` and `tmp` so the last writes `out`.
template <typename K, bool V>
static rs_status_t merge_tree_ptrs(const std::vector<const void*>& rk, const std::vector<const uint32_t*>& rv,
                                   const std::vector<uint64_t>& len, K* tmp, uint32_t* vtmp, K* out, uint32_t* vout,
                                   size_t* split, cudaStream_t st) {
    const int p = (int)len.size();
    std::vector<uint64_t> off(p + 1, 0);
    for (int k = 0; k < p; ++k) off[k + 1] = off[k] + len[k];
    const size_t total = off[p];
    if (total == 0) return RS_OK;
    int levels = 0;
    for (int q = p; q > 1; q = (q + 1) / 2) ++levels;
    auto buf = [&](int level) { return ((levels - 1 - level) % 2 == 0) ? out : tmp; };
    auto vbuf = [&](int level) { return ((levels - 1 - level) % 2 == 0) ? vout : vtmp; };
    K* dst = levels == 0 ? out : buf(0);
    uint32_t* vdst = V ? (levels == 0 ? vout : vbuf(0)) : nullptr;
    std::vector<uint64_t> noff(1, 0);
    for (int k = 0; k < p; k += 2) {  // level 0 (or the single run)
        const K* A = static_cast<const K*>(rk[k]);
        if (k + 1 < p) {
            const K* B = static_cast<const K*>(rk[k + 1]);
            rs_status_t s = merge2<K, V>(A, V ? rv[k] : nullptr, len[k], B, V ? rv[k + 1] : nullptr, len[k + 1],
                                         dst + off[k], V ? vdst + off[k] : nullptr, split, st);
            if (s != RS_OK) return s;
            noff.push_back(off[k + 2]);
        } else {
            if (len[k]) {
                RS_CUDA_TRY(cudaMemcpyAsync(dst + off[k], A, len[k] * sizeof(K), cudaMemcpyDefault, st));
                if (V) RS_CUDA_TRY(cudaMemcpyAsync(vdst + off[k], rv[k], len[k] * 4, cudaMemcpyDefault, st));
            }
            noff.push_back(off[k + 1]);
        }
    }
    if (levels <= 1) return RS_OK;
    // levels 1..: contiguous runs in buf(l-1) -> buf(l); the generic tree clobbers its input
    // buffer, which here is free scratch (tmp or out)
    for (int l = 1; l < levels; ++l) {
        K* src = buf(l - 1);
        uint32_t* vsrc = V ? vbuf(l - 1) : nullptr;
        K* d = buf(l);
        uint32_t* vd = V ? vbuf(l) : nullptr;
        const int q = (int)noff.size() - 1;
        std::vector<uint64_t> nn(1, 0);
        for (int k = 0; k < q; k += 2) {
            const uint64_t a0 = noff[k], a1 = noff[k + 1];
            if (k + 1 < q) {
                const uint64_t b1 = noff[k + 2];
                rs_status_t s = merge2<K, V>(src + a0, V ? vsrc + a0 : nullptr, a1 - a0, src + a1,
                                             V ? vsrc + a1 : nullptr, b1 - a1, d + a0, V ? vd + a0 : nullptr, split, st);
                if (s != RS_OK) return s;
                nn.push_back(b1);
            } else {
                if (a1 > a0) {
                    RS_CUDA_TRY(cudaMemcpyAsync(d + a0, src + a0, (a1 - a0) * sizeof(K), cudaMemcpyDeviceToDevice, st));
                    if (V) RS_CUDA_TRY(cudaMemcpyAsync(vd + a0, vsrc + a0, (a1 - a0) * 4, cudaMemcpyDeviceToDevice, st));
                }
                nn.push_back(a1);
            }
        }
        noff.swap(nn);
    }
    return RS_OK;
}

rs_status_t merge_runs_ptrs(int key_bytes, const std::vector<const void*>& rk, const std::vector<const uint32_t*>& rv,
                            const std::vector<uint64_t>& len, void* tmp, uint32_t* vtmp, void* out, uint32_t* vout,
                            size_t* split, cudaStream_t st) {
    const bool V = !rv.empty() && rv[0] != nullptr;
    if (key_bytes == 4) {
        if (V)
            return merge_tree_ptrs<uint32_t, true>(rk, rv, len, static_cast<uint32_t*>(tmp), vtmp,
                                                   static_cast<uint32_t*>(out), vout, split, st);
        return merge_tree_ptrs<uint32_t, false>(rk, rv, len, static_cast<uint32_t*>(tmp), nullptr,
                                                static_cast<uint32_t*>(out), nullptr, split, st);
    }
    if (V)
        return merge_tree_ptrs<uint64_t, true>(rk, rv, len, static_cast<uint64_t*>(tmp), vtmp,
                                               static_cast<uint64_t*>(out), vout, split, st);
    return merge_tree_ptrs<uint64_t, false>(rk, rv, len, static_cast<uint64_t*>(tmp), nullptr,
                                            static_cast<uint64_t*>(out), nullptr, split, st);
}

rs_status_t merge_range(int key_bytes, const void* A, const uint32_t* VA, size_t na, const void* B, const uint32_t* VB,
                        size_t nb, size_t lo, size_t hi, void* out, uint32_t* vout, size_t* split, cudaStream_t st) {
    const bool V = VA != nullptr;
    if (key_bytes == 4) {
        if (V)
            return merge2_range<uint32_t, true>(static_cast<const uint32_t*>(A), VA, na, static_cast<const uint32_t*>(B),
                                                VB, nb, lo, hi, static_cast<uint32_t*>(out), vout, split, st);
        return merge2_range<uint32_t, false>(static_cast<const uint32_t*>(A), nullptr, na,
                                             static_cast<const uint32_t*>(B), nullptr, nb, lo, hi,
                                             static_cast<uint32_t*>(out), nullptr, split, st);
    }
    if (V)
        return merge2_range<uint64_t, true>(static_cast<const uint64_t*>(A), VA, na, static_cast<const uint64_t*>(B), VB,
                                            nb, lo, hi, static_cast<uint64_t*>(out), vout, split, st);
    return merge2_range<uint64_t, false>(static_cast<const uint64_t*>(A), nullptr, na, static_cast<const uint64_t*>(B),
                                         nullptr, nb, lo, hi, static_cast<uint64_t*>(out), nullptr, split, st);
}

rs_status_t merge_runs_tree(int key_bytes, void* runs, uint32_t* vruns, const std::vector<uint64_t>& roff, void* tmp,
                            uint32_t* vtmp, void* out, uint32_t* vout, size_t* split, cudaStream_t st) {
    const bool V = vruns != nullptr;
    if (key_bytes == 4) {
        if (V)
            return merge_tree<uint32_t, true>(static_cast<uint32_t*>(runs), vruns, roff, static_cast<uint32_t*>(tmp),
                                              vtmp, static_cast<uint32_t*>(out), vout, split, st);
        return merge_tree<uint32_t, false>(static_cast<uint32_t*>(runs), nullptr, roff, static_cast<uint32_t*>(tmp),
                                           nullptr, static_cast<uint32_t*>(out), nullptr, split, st);
    }
    if (V)
        return merge_tree<uint64_t, true>(static_cast<uint64_t*>(runs), vruns, roff, static_cast<uint64_t*>(tmp), vtmp,
                                          static_cast<uint64_t*>(out), vout, split, st);
    return merge_tree<uint64_t, false>(static_cast<uint64_t*>(runs), nullptr, roff, static_cast<uint64_t*>(tmp), nullptr,
                                       static_cast<uint64_t*>(out), nullptr, split, st);
}

}  // namespace rs
