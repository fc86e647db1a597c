// mclx_dev.cuh -- device primitives shared by the libmclx kernels (sm_100a).
//
// Team = one CTA of NT threads working on one matrix column.  Everything here is
// plain CUDA C++ (warp shuffles/ballots, shared-memory atomics, block scans); the
// path is sparse gather/hash/select work, not a dense contraction, so there are
// no tensor-core instructions anywhere in this library (north star).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mclx {

constexpr int kEmptyKey = -1;          // unoccupied hash slot
constexpr int kPadKey = 0x7fffffff;    // bitonic padding, sorts after every row id
constexpr int kMaxWarps = 32;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

// Fibonacci hashing of a row id onto [0, cap): the top bits of row * 2^32/phi,
// range-reduced by a multiply-high so that cap need not be a power of two.
__device__ __forceinline__ uint32_t hash_slot(int row, uint32_t cap) {
    return __umulhi((uint32_t)row * 0x9E3779B1u, cap);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        T w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}
template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        T w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}

// Block-wide sum / max.  `sh` holds >= NT/32 elements of T.  Every thread gets the result.
template <int NT, typename T>
__device__ __forceinline__ T block_sum(T v, T *sh) {
    v = warp_sum(v);
    if (NT == 32) return v;
    __syncthreads();
    if (lane_id() == 0) sh[warp_id()] = v;
    __syncthreads();
    T r = T(0);
#pragma unroll
    for (int i = 0; i < NT / 32; i++) r += sh[i];
    return r;
}
template <int NT, typename T>
__device__ __forceinline__ T block_max(T v, T *sh) {
    v = warp_max(v);
    if (NT == 32) return v;
    __syncthreads();
    if (lane_id() == 0) sh[warp_id()] = v;
    __syncthreads();
    T r = sh[0];
#pragma unroll
    for (int i = 1; i < NT / 32; i++) r = sh[i] > r ? sh[i] : r;
    return r;
}

// Block-wide exclusive scan of small ints; `total` receives the block sum.
template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int *sh, int &total) {
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane_id() >= o) x += y;
    }
    if (NT == 32) {
        total = __shfl_sync(0xffffffffu, x, 31);
        return x - v;
    }
    __syncthreads();
    if (lane_id() == 31) sh[warp_id()] = x;
    __syncthreads();
    int off = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < NT / 32; i++) {
        int s = sh[i];
        off += (i < warp_id()) ? s : 0;
        tot += s;
    }
    total = tot;
    return off + x - v;
}

template <typename V>
__device__ __forceinline__ uint32_t val_bits(V v) {
    return __float_as_uint((float)v);  // positive floats order like their bit patterns
}

// Order-preserving in-place compaction of (keys, vals)[0, len) by predicate keep(key, val).
// Safe in place: chunk c is fully read before the scan's barrier, and its writes land at
// indices <= the chunk's own indices, below every unread element.  Returns the kept count.
template <int NT, typename V, class Pred>
__device__ int compact_inplace(int *keys, V *vals, int len, Pred keep, int *sh) {
    int base = 0;
    for (int c = 0; c < len; c += NT) {
        int i = c + (int)threadIdx.x;
        int k = 0;
        V v = V(0);
        int f = 0;
        if (i < len) {
            k = keys[i];
            v = vals[i];
            f = keep(k, v) ? 1 : 0;
        }
        int tot;
        int pos = block_excl_scan<NT>(f, sh, tot);
        if (f) {
            keys[base + pos] = k;
            vals[base + pos] = v;
        }
        base += tot;
    }
    __syncthreads();
    return base;
}

// Bitonic sort of (keys, vals)[0, P) ascending by key; P a power of two, padded by caller.
template <int NT, typename V>
__device__ void bitonic_sort(int *keys, V *vals, int P) {
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P; i += NT) {
                int ixj = i ^ j;
                if (ixj > i) {
                    int a = keys[i], b = keys[ixj];
                    bool up = ((i & k) == 0);
                    if ((a > b) == up) {
                        keys[i] = b;
                        keys[ixj] = a;
                        V t = vals[i];
                        vals[i] = vals[ixj];
                        vals[ixj] = t;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// Sort the K entries (keys, vals)[0, K) by key and write them, values mapped by
// xf(v) -> float, to out_row / out_val[0, K) in global memory.
// Interpolation bucket sort: rows are spread over [min, max] (vertex ids carry no
// order), so nbk ~ K/2 buckets by (row - min) * nbk / (max - min + 1) hold ~2 entries
// each.  Counters live in the table's free slots keys[K, cap).  Entries are scattered
// to their bucket's slice of the output, then each bucket (tiny) is insertion-sorted in
// place.  If some bucket is large (clustered rows), fall back to a shared-memory
// bitonic sort.  Requires K <= cap (cap a power of two) and K < cap for the counters.
template <int NT, typename V, class XF>
__device__ void sort_write(int *keys, V *vals, int K, int cap, int32_t *out_row, float *out_val,
                           XF xf, int *sh) {
    if (K <= 0) return;
    int lo = 0x7fffffff, hi = 0;
    for (int i = threadIdx.x; i < K; i += NT) {
        const int r = keys[i];
        lo = r < lo ? r : lo;
        hi = r > hi ? r : hi;
    }
    lo = -block_max<NT, int>(-lo, sh);
    hi = block_max<NT, int>(hi, sh);
    {
        // Fast path: build the sorted column in the table's free space -- keys[K, 2K) and
        // vals[K, 2K) (as float) for the output, counters at keys[2K, 2K + nbk) -- with
        // insertion sorts inside the (tiny) buckets, then one coalesced copy out.
        int nbk = 1;
        while (nbk * 4 <= K) nbk *= 2;
        if (2 * K + nbk <= cap) {
            int *okey = keys + K;
            float *oval = reinterpret_cast<float *>(vals + K);
            int *cnt = keys + 2 * K;
            for (int i = threadIdx.x; i < nbk; i += NT) cnt[i] = 0;
            __syncthreads();
            const uint64_t range = (uint64_t)(hi - lo) + 1;
            for (int i = threadIdx.x; i < K; i += NT)
                atomicAdd(&cnt[(int)(((uint64_t)(keys[i] - lo) * nbk) / range)], 1);
            __syncthreads();
            const int per = (nbk + NT - 1) / NT;
            const int b0 = threadIdx.x * per;
            int loc = 0, mx = 0;
            for (int b = b0; b < b0 + per && b < nbk; b++) {
                loc += cnt[b];
                mx = cnt[b] > mx ? cnt[b] : mx;
            }
            int tot;
            int off = block_excl_scan<NT>(loc, sh, tot);
            mx = block_max<NT, int>(mx, sh);
            if (mx <= 48) {
                for (int b = b0; b < b0 + per && b < nbk; b++) {
                    const int c = cnt[b];
                    cnt[b] = off;
                    off += c;
                }
                __syncthreads();
                for (int i = threadIdx.x; i < K; i += NT) {
                    const int r = keys[i];
                    const int pos = atomicAdd(&cnt[(int)(((uint64_t)(r - lo) * nbk) / range)], 1);
                    okey[pos] = r;
                    oval[pos] = xf(vals[i]);
                }
                __syncthreads();
                for (int b = threadIdx.x; b < nbk; b += NT) {
                    const int start = b ? cnt[b - 1] : 0, end = cnt[b];
                    for (int i = start + 1; i < end; i++) {
                        const int r = okey[i];
                        const float v = oval[i];
                        int j = i - 1;
                        while (j >= start && okey[j] > r) {
                            okey[j + 1] = okey[j];
                            oval[j + 1] = oval[j];
                            j--;
                        }
                        okey[j + 1] = r;
                        oval[j + 1] = v;
                    }
                }
                __syncthreads();
                for (int i = threadIdx.x; i < K; i += NT) {
                    out_row[i] = okey[i];
                    out_val[i] = oval[i];
                }
                __syncthreads();
                return;
            }
            __syncthreads();
        }
    }
    int free_slots = cap - K;
    int nbk = 1;
    while (nbk * 2 <= free_slots && nbk * 4 <= K) nbk *= 2;
    int *cnt = keys + K;
    if (free_slots >= 1) {
        for (int i = threadIdx.x; i < nbk; i += NT) cnt[i] = 0;
        __syncthreads();
        const uint64_t range = (uint64_t)(hi - lo) + 1;
        for (int i = threadIdx.x; i < K; i += NT)
            atomicAdd(&cnt[(int)(((uint64_t)(keys[i] - lo) * nbk) / range)], 1);
        __syncthreads();
        // exclusive scan of the counters (contiguous chunks per thread) + largest bucket
        const int per = (nbk + NT - 1) / NT;
        const int b0 = threadIdx.x * per;
        int loc = 0, mx = 0;
        for (int b = b0; b < b0 + per && b < nbk; b++) {
            loc += cnt[b];
            mx = cnt[b] > mx ? cnt[b] : mx;
        }
        int tot;
        int off = block_excl_scan<NT>(loc, sh, tot);
        mx = block_max<NT, int>(mx, sh);
        if (mx <= 48) {
            for (int b = b0; b < b0 + per && b < nbk; b++) {
                const int c = cnt[b];
                cnt[b] = off;
                off += c;
            }
            __syncthreads();
            for (int i = threadIdx.x; i < K; i += NT) {
                const int r = keys[i];
                const int pos = atomicAdd(&cnt[(int)(((uint64_t)(r - lo) * nbk) / range)], 1);
                out_row[pos] = r;
                out_val[pos] = xf(vals[i]);
            }
            __syncthreads();
            for (int b = threadIdx.x; b < nbk; b += NT) {
                const int start = b ? cnt[b - 1] : 0, end = cnt[b];
                for (int i = start + 1; i < end; i++) {
                    const int r = __ldcg(out_row + i);
                    const float v = __ldcg(out_val + i);
                    int j = i - 1;
                    while (j >= start && __ldcg(out_row + j) > r) {
                        out_row[j + 1] = __ldcg(out_row + j);
                        out_val[j + 1] = __ldcg(out_val + j);
                        j--;
                    }
                    out_row[j + 1] = r;
                    out_val[j + 1] = v;
                }
            }
            __syncthreads();
            return;
        }
        __syncthreads();
    }
    // fallback: bitonic sort in place (K <= cap, cap a power of two)
    int P = 1;
    while (P < K) P <<= 1;
    for (int i = K + threadIdx.x; i < P; i += NT) keys[i] = kPadKey;
    __syncthreads();
    bitonic_sort<NT, V>(keys, vals, P);
    for (int i = threadIdx.x; i < K; i += NT) {
        out_row[i] = keys[i];
        out_val[i] = xf(vals[i]);
    }
    __syncthreads();
}

// ------------------------------------------------------------------ warp-scoped helpers
// (the private-slice kernel family: each warp owns a slice of the table and an ordered
// row range, so the epilogue works slice by slice with warp ballots instead of CTA scans)

// In-place, order-preserving compaction of (keys, vals)[0, len) by keep(key, val) within
// one warp (chunks of 32 read before written; writes land at or below the chunk).
template <typename V, class Pred>
__device__ __forceinline__ int warp_compact(int *keys, V *vals, int len, Pred keep) {
    const int lane = lane_id();
    const unsigned lt = (1u << lane) - 1u;
    int base = 0;
    for (int c = 0; c < len; c += 32) {
        const int i = c + lane;
        int k = 0;
        V v = V(0);
        bool f = false;
        if (i < len) {
            k = keys[i];
            v = vals[i];
            f = keep(k, v);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        __syncwarp();
        if (f) {
            keys[base + __popc(bal & lt)] = k;
            vals[base + __popc(bal & lt)] = v;
        }
        base += __popc(bal);
        __syncwarp();
    }
    return base;
}

// Warp-level bitonic sort of (keys, vals)[0, P), P a power of two, padded by the caller.
template <typename V>
__device__ void warp_bitonic_sort(int *keys, V *vals, int P) {
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane_id(); i < P; i += 32) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const int a = keys[i], b = keys[ixj];
                    if ((a > b) == ((i & k) == 0)) {
                        keys[i] = b;
                        keys[ixj] = a;
                        const V t = vals[i];
                        vals[i] = vals[ixj];
                        vals[ixj] = t;
                    }
                }
            }
            __syncwarp();
        }
    }
}

// Sort the K entries of one warp's slice (keys, vals)[0, K) by row and write them, mapped
// by xf, to out_row / out_val[0, K): interpolation bucket sort in the slice's free space
// (keys/vals[K, 2K) for the output, counters at keys[2K, 2K + nbk)), else an in-place
// bitonic sort (slice length scap a power of two >= K).
template <typename V, class XF>
__device__ void warp_sort_write(int *keys, V *vals, int K, int scap, int32_t *out_row,
                                float *out_val, XF xf) {
    if (K <= 0) return;
    const int lane = lane_id();
    int lo = 0x7fffffff, hi = 0;
    for (int i = lane; i < K; i += 32) {
        const int r = keys[i];
        lo = r < lo ? r : lo;
        hi = r > hi ? r : hi;
    }
    lo = warp_min(lo);
    hi = warp_max(hi);
    int nbk = 1;
    while (nbk * 4 <= K) nbk *= 2;
    if (2 * K + nbk <= scap) {
        int *okey = keys + K;
        float *oval = reinterpret_cast<float *>(vals + K);
        int *cnt = keys + 2 * K;
        for (int i = lane; i < nbk; i += 32) cnt[i] = 0;
        __syncwarp();
        const uint64_t range = (uint64_t)(hi - lo) + 1;
        for (int i = lane; i < K; i += 32)
            atomicAdd(&cnt[(int)(((uint64_t)(keys[i] - lo) * nbk) / range)], 1);
        __syncwarp();
        // exclusive scan of the counters, 32 contiguous chunks
        const int per = (nbk + 31) / 32;
        const int b0 = lane * per;
        int loc = 0, mx = 0;
        for (int b = b0; b < b0 + per && b < nbk; b++) {
            loc += cnt[b];
            mx = cnt[b] > mx ? cnt[b] : mx;
        }
        int inc = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        mx = warp_max(mx);
        if (mx <= 48) {
            int off = inc - loc;
            for (int b = b0; b < b0 + per && b < nbk; b++) {
                const int c = cnt[b];
                cnt[b] = off;
                off += c;
            }
            __syncwarp();
            for (int i = lane; i < K; i += 32) {
                const int r = keys[i];
                const int pos = atomicAdd(&cnt[(int)(((uint64_t)(r - lo) * nbk) / range)], 1);
                okey[pos] = r;
                oval[pos] = xf(vals[i]);
            }
            __syncwarp();
            for (int b = lane; b < nbk; b += 32) {
                const int start = b ? cnt[b - 1] : 0, end = cnt[b];
                for (int i = start + 1; i < end; i++) {
                    const int r = okey[i];
                    const float v = oval[i];
                    int j = i - 1;
                    while (j >= start && okey[j] > r) {
                        okey[j + 1] = okey[j];
                        oval[j + 1] = oval[j];
                        j--;
                    }
                    okey[j + 1] = r;
                    oval[j + 1] = v;
                }
            }
            __syncwarp();
            for (int i = lane; i < K; i += 32) {
                out_row[i] = okey[i];
                out_val[i] = oval[i];
            }
            __syncwarp();
            return;
        }
        __syncwarp();
    }
    int P = 1;
    while (P < K) P <<= 1;
    for (int i = K + lane; i < P; i += 32) keys[i] = kPadKey;
    __syncwarp();
    warp_bitonic_sort<V>(keys, vals, P);
    for (int i = lane; i < K; i += 32) {
        out_row[i] = keys[i];
        out_val[i] = xf(vals[i]);
    }
    __syncwarp();
}

// Warp 0 only: find the digit d of a 256-bin histogram at which the running count
// (from the top digit when DESC, from digit 0 otherwise) first reaches `rem`.
// out[0] = d, out[1] = count strictly before d in that order, out[2] = hist[d].
template <bool DESC>
__device__ __forceinline__ void find_digit(const unsigned *hist, int rem, int *out) {
    const int lane = lane_id();
    unsigned c[8];
    unsigned sum = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        int d = DESC ? 255 - (lane * 8 + i) : lane * 8 + i;
        c[i] = hist[d];
        sum += c[i];
    }
    unsigned inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    unsigned excl = inc - sum;
    if (excl < (unsigned)rem && inc >= (unsigned)rem) {
        unsigned run = excl;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (run + c[i] >= (unsigned)rem) {
                out[0] = DESC ? 255 - (lane * 8 + i) : lane * 8 + i;
                out[1] = (int)run;
                out[2] = (int)c[i];
                break;
            }
            run += c[i];
        }
    }
}

// Exact top-K of (vals desc, keys asc) over entries [0, n) (every entry valid):
// radix select on the fp32 bit pattern (8-bit digits), then on the row id among the
// entries equal to the K-th value.  Entry e is kept iff
//   bits(e) > t  or  (bits(e) == t and key(e) <= rowcut).
template <int NT, typename V>
__device__ void radix_select_topk(const int *keys, const V *vals, int n, int K, uint32_t &t,
                                  int &rowcut, unsigned *hist, int *sint) {
    uint32_t prefix = 0, mask = 0;
    int rem = K, eq = 0;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += NT) hist[i] = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += NT) {
            uint32_t b = val_bits(vals[i]);
            if ((b & mask) == prefix) atomicAdd(&hist[(b >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (threadIdx.x < 32) find_digit<true>(hist, rem, sint);
        __syncthreads();
        uint32_t d = (uint32_t)sint[0];
        rem -= sint[1];
        eq = sint[2];
        prefix |= d << shift;
        mask |= 0xFFu << shift;
        __syncthreads();
    }
    t = prefix;
    if (rem == eq) {
        rowcut = 0x7fffffff;
        return;
    }
    uint32_t rp = 0, rm = 0;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += NT) hist[i] = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += NT) {
            uint32_t b = val_bits(vals[i]);
            uint32_t k = (uint32_t)keys[i];
            if (b == t && (k & rm) == rp) atomicAdd(&hist[(k >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (threadIdx.x < 32) find_digit<false>(hist, rem, sint);
        __syncthreads();
        rp |= (uint32_t)sint[0] << shift;
        rm |= 0xFFu << shift;
        rem -= sint[1];
        __syncthreads();
    }
    rowcut = (int)rp;
}

// radix_select_topk over W per-warp segments: warp w's entries are (keys, vals)[0, n) of
// its own slice (pointers and n differ per warp); the histograms are CTA-wide.
template <int NT, typename V>
__device__ void radix_select_topk_seg(const int *keys, const V *vals, int n, int K, uint32_t &t,
                                      int &rowcut, unsigned *hist, int *sint) {
    const int lane = lane_id();
    uint32_t prefix = 0, mask = 0;
    int rem = K, eq = 0;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += NT) hist[i] = 0;
        __syncthreads();
        for (int i = lane; i < n; i += 32) {
            const uint32_t b = val_bits(vals[i]);
            if ((b & mask) == prefix) atomicAdd(&hist[(b >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (threadIdx.x < 32) find_digit<true>(hist, rem, sint);
        __syncthreads();
        const uint32_t d = (uint32_t)sint[0];
        rem -= sint[1];
        eq = sint[2];
        prefix |= d << shift;
        mask |= 0xFFu << shift;
        __syncthreads();
    }
    t = prefix;
    if (rem == eq) {
        rowcut = 0x7fffffff;
        return;
    }
    uint32_t rp = 0, rm = 0;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += NT) hist[i] = 0;
        __syncthreads();
        for (int i = lane; i < n; i += 32) {
            const uint32_t b = val_bits(vals[i]);
            const uint32_t k = (uint32_t)keys[i];
            if (b == t && (k & rm) == rp) atomicAdd(&hist[(k >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (threadIdx.x < 32) find_digit<false>(hist, rem, sint);
        __syncthreads();
        rp |= (uint32_t)sint[0] << shift;
        rm |= 0xFFu << shift;
        rem -= sint[1];
        __syncthreads();
    }
    rowcut = (int)rp;
}

// Parameters of the prune / select / recover / inflate step (readings Q3-Q9).
struct PruneParams {
    double theta;   // keep v >= theta
    int S;          // select_k
    int R;          // recover_k (0 = off)
    double pct;     // recover when kept mass < pct
    double r;       // inflation exponent
    int r_is_2;
    int kmax;       // max(S, R, 1): staging capacity per column
};

// Branch of a column (same numbering as the oracle): 0 thresh, 1 select, 2 recover,
// 3 argmax, 4 empty.  K = number of entries kept.
__device__ __forceinline__ int prune_branch(const PruneParams &pp, int64_t nnz, int64_t m,
                                            double s, int64_t &K) {
    if (m > pp.S) {
        K = pp.S;
        return 1;
    }
    if (pp.R > 0 && m < pp.R && s < pp.pct && nnz > m) {
        K = pp.R < nnz ? pp.R : nnz;
        return 2;
    }
    if (m > 0) {
        K = m;
        return 0;
    }
    if (nnz > 0) {
        K = 1;
        return 3;
    }
    K = 0;
    return 4;
}

__device__ __forceinline__ double pow_r(double w, const PruneParams &pp) {
    return pp.r_is_2 ? w * w : pow(w, pp.r);
}

__device__ __forceinline__ void atomic_max_nonneg_float(float *addr, float v) {
    // non-negative floats order like their int bit patterns
    atomicMax(reinterpret_cast<int *>(addr), __float_as_int(v));
}

// Alg. 1 lines 4-5 on one unpruned column (rows ascending, in global memory, read by the
// whole CTA): threshold stats, branch (Q5, Q7, Q8), exact top-K by radix select,
// renormalise + chaos (Q9), Hadamard power r and renormalise (Q1).  The kept
// entries are extracted in row order with a block scan, so the output stays sorted.
// Writes srow/sval at soff[col], scnt[col], chaos_out[col] (if given) and folds the
// chaos into *chaos_max and the kept count into *out_count (if given).  All NT threads call.
// With fnnz >= 0 the entries given are only CANDIDATES of the column (the top max(S, R) of
// every row-range part, run_split) and (fnnz, fm, fs) are the statistics of the whole
// unpruned column: the branch is decided on those, the selection runs on the candidates.
template <int NT>
__device__ void prune_column(const int32_t *rows, const float *vals, int nnz, int64_t col,
                             const int64_t *soff, int32_t *srow, float *sval, int64_t *scnt,
                             float *chaos_out, float *chaos_max, unsigned long long *out_count,
                             const PruneParams &pp, unsigned *hist, int *sint, double *sred,
                             int *sscan, int64_t fnnz = -1, int64_t fm = 0, double fs = 0.0) {
    const int tid = threadIdx.x;
    int64_t nnz_b = nnz, m;
    double s;
    if (fnnz >= 0) {
        nnz_b = fnnz;
        m = fm;
        s = fs;
    } else {
        int mloc = 0;
        double sloc = 0.0;
        for (int i = tid; i < nnz; i += NT) {
            double v = (double)vals[i];
            if (v >= pp.theta) {
                mloc++;
                sloc += v;
            }
        }
        m = block_sum<NT, int>(mloc, sscan);
        s = block_sum<NT, double>(sloc, sred);
    }
    int64_t K;
    const int br = prune_branch(pp, nnz_b, m, s, K);
    uint32_t t = 0;
    int rowcut = 0, sel;
    if (br == 0) {
        sel = 0;
    } else if (K >= nnz) {
        sel = 2;
    } else {
        radix_select_topk<NT, float>(rows, vals, nnz, (int)K, t, rowcut, hist, sint);
        sel = 1;
    }
    auto keep = [&](int k, float v) {
        if (sel == 0) return (double)v >= pp.theta;
        if (sel == 2) return true;
        uint32_t b = val_bits(v);
        return b > t || (b == t && k <= rowcut);
    };
    double sv = 0.0, mx = 0.0, sq = 0.0, sr = 0.0;
    for (int i = tid; i < nnz; i += NT) {
        float v = vals[i];
        if (keep(rows[i], v)) {
            double d = (double)v;
            sv += d;
            mx = d > mx ? d : mx;
            sq += d * d;
            sr += pow_r(d, pp);
        }
    }
    sv = block_sum<NT, double>(sv, sred);
    mx = block_max<NT, double>(mx, sred);
    sq = block_sum<NT, double>(sq, sred);
    sr = block_sum<NT, double>(sr, sred);
    const int64_t dst = soff[col];
    int kept = 0;
    for (int c = 0; c < nnz; c += NT) {
        const int i = c + tid;
        int f = 0;
        int r = 0;
        float v = 0.f;
        if (i < nnz) {
            r = rows[i];
            v = vals[i];
            f = keep(r, v) ? 1 : 0;
        }
        int tot;
        const int pos = block_excl_scan<NT>(f, sscan, tot);
        if (f) {
            srow[dst + kept + pos] = r;
            sval[dst + kept + pos] = (float)(pow_r((double)v, pp) / sr);
        }
        kept += tot;
    }
    const float chaos = kept > 0 ? (float)((double)kept * (mx / sv - sq / (sv * sv))) : 0.0f;
    if (tid == 0) {
        scnt[col] = kept;
        if (chaos_out) chaos_out[col] = chaos;
        atomic_max_nonneg_float(chaos_max, chaos);
        if (out_count) atomicAdd(out_count, (unsigned long long)kept);
    }
    __syncthreads();
}

}  // namespace mclx
