// kernels_dense.cu -- the dense bin of the expansion step (SURVEY §8(a) a4 "dense": the
// R-MAT hub columns of C4, whose product covers a sizable share of the row space).
//
// Such a column runs as kDenseParts row-range parts (part p = rowparts [p 32/D, (p+1) 32/D)
// of A's 32-way row index), each a work item of one CTA that SWEEPS its row range tile by
// tile: a tile of kSweepTileBytes (40960 fp32 / 20480 fp64 rows) is a dense accumulator in
// shared memory -- no hashing, the slot is the row -- and every segment A_*k of the column
// keeps a cursor (its next position, in shared memory beside the tile) that advances as the
// tiles pass, so each product is gathered exactly once and each segment descriptor is read
// once per part ("per-k cursors kept ... when one CTA sweeps the tiles in
// order").  Columns with more than kSweepSeg segments take them in chunks whose cursors are
// re-found by binary search at every tile.  A touched row is one with a value > 0 -- fp64
// products of positive fp32 values never underflow; an fp32 product that underflows to 0
// marks its row with -0.0 instead (Q13: the entry stays in the structure) -- so compacting
// a tile emits its rows in ascending order, no sort.  Values are added with shared-memory
// atomics (lanes of a group walk one segment; other groups may hit the same row).  fp64
// tiles for columns with more than kFp64Terms segments (T), fp32 otherwise.  Entries go to
// the item's staging slot, which the split path stitches and prunes (k_prune); more entries
// than the slot holds flag the column for the next round.  With candidates (cand_k =
// max(S, R) > 0) a part stages only its top-cand_k entries, kept by a streaming selection in
// a shared-memory buffer (append what beats the buffer's cut, radix-select back to cand_k
// when it fills), plus the count / mass statistics of all its entries (see run_split).
//
// History: the first dense kernel gave every (column, 1/32 row range) part several passes
// over a 192 KB tile, re-reading each sub-segment's prefix and all segment descriptors at
// every pass: 112 s of C4's (R-MAT scale 22) 130 s iteration.  An L2-resident variant (one
// fp64 array of m rows per column, RED.ADD.F64) was 10x slower than tiles at scale 20.
#include <climits>

#include "kernels.h"

namespace mclx {

constexpr int kLongPerTile = 16;  // expected rows per tile above which a warp walks a segment

__device__ __forceinline__ int dense_touched(double v) { return v > 0.0 ? 1 : 0; }
// fp32 tiles start at +0 and every add is >= 0, so a touched entry is > 0 -- unless its
// products underflowed to 0.  Those are flagged by storing -0.0 (sign bit) at the first
// add of an exact zero (atomic_mark_zero); a later positive add turns it into a value.
__device__ __forceinline__ int dense_touched(float v) {
    return (v > 0.f || __float_as_uint(v) == 0x80000000u) ? 1 : 0;
}

__device__ __forceinline__ void atomic_mark_zero(float *p) {
    atomicCAS(reinterpret_cast<unsigned *>(p), 0u, 0x80000000u);
}
__device__ __forceinline__ void atomic_mark_zero(double *) {}  // fp64 products never underflow


// first position q in [lo, hi) of A with row >= r (rows of a segment ascend)
__device__ __forceinline__ uint32_t lower_row(const int2 *__restrict__ ap, uint32_t lo, uint32_t hi,
                                              int64_t r) {
    while (lo < hi) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        if ((int64_t)__ldg(&ap[mid].x) < r) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// One group of G lanes walks segment e (its cursor .. end) while the rows stay below t_end,
// adding b_kj * a_ik into the tile (4 gathers in flight per lane), then stores the segment's
// new cursor: the first position the group did not take (rows ascend in a segment).
template <int G, typename V>
__device__ __forceinline__ void sweep_walk(const int2 *__restrict__ ap, V *acc, int64_t t0,
                                           int64_t t_end, uint32_t *cur, const uint32_t *end,
                                           const float *bkj, int e, bool has, bool save) {
    const int lane_g = (int)(threadIdx.x & 31) & (G - 1);
    const uint32_t pos = has ? cur[e] : 0u, fin = has ? end[e] : 0u;
    const V b = has ? (V)bkj[e] : V(0);
    uint32_t stop = fin;
    for (uint32_t i = pos + (uint32_t)lane_g;; i += 4u * G) {
        int2 pv[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const uint32_t q = i + (uint32_t)(u * G);
            pv[u] = q < fin ? __ldg(ap + q) : make_int2(INT_MAX, 0);
        }
        bool done = false;
#pragma unroll
        for (int u = 0; u < 4; u++) {
            if (done) continue;
            if ((int64_t)pv[u].x >= t_end) {
                const uint32_t q = i + (uint32_t)(u * G);
                stop = q < fin ? q : fin;
                done = true;
            } else {
                const V prod = (V)__int_as_float(pv[u].y) * b;
                V *slot = &acc[pv[u].x - t0];
                if (prod > V(0)) atomicAdd(slot, prod);
                else atomic_mark_zero(slot);  // fp32 underflow: keep the entry
            }
        }
        if (done) break;
    }
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
        const uint32_t t = __shfl_xor_sync(0xffffffffu, stop, o);
        stop = t < stop ? t : stop;
    }
    if (has && lane_g == 0 && save) cur[e] = stop;
}

template <typename V>
__global__ void __launch_bounds__(kDenseThreads, 1) k_dense_sweep(BinArgs a) {
    constexpr int NT = kDenseThreads;
    constexpr int TILE = kSweepTileBytes / (int)sizeof(V);
    extern __shared__ __align__(16) unsigned char dsm[];
    V *acc = reinterpret_cast<V *>(dsm);
    uint32_t *cur = reinterpret_cast<uint32_t *>(dsm + kSweepTileBytes);  // segment cursors
    uint32_t *end = cur + kSweepSeg;                                        // segment ends
    float *bkj = reinterpret_cast<float *>(end + kSweepSeg);               // b_kj
    int *crow = reinterpret_cast<int *>(bkj + kSweepSeg);                   // candidates (rows)
    float *cval = reinterpret_cast<float *>(crow + kCandBuf);              // candidates (values)
    __shared__ int sscan[NT / 32];
    __shared__ int s_wcnt[32];
    __shared__ double sred[NT / 32];
    __shared__ unsigned hist[256];
    __shared__ int sint[4];
    __shared__ int s_col, s_idx, s_pr, s_nextL, s_nextS, s_nL, s_nS, s_ncand, s_reduced;
    __shared__ uint32_t s_thr;
    const bool cand = a.cand_k > 0;
    const double theta = a.pp.theta;
    const int tid = threadIdx.x, lane = tid & 31;
    const int count = *a.count;
    for (;;) {
        if (tid == 0) {
            const int idx = atomicAdd(a.counter, 1);
            s_idx = idx;
            s_col = idx < count ? a.list[idx] : -1;
            s_pr = idx < count ? a.item_pr[idx] : 0;
            s_ncand = 0;
            s_reduced = 0;
            s_thr = 0u;
        }
        __syncthreads();
        const int col = s_col, idx = s_idx, pr = s_pr;
        if (col < 0) return;
        const int p0 = pr & 0xff, p1 = pr >> 8;
        const int64_t r_lo = ((int64_t)p0 * a.m + kParts - 1) / kParts;
        const int64_t r_hi = ((int64_t)p1 * a.m + kParts - 1) / kParts;
        const int64_t bj = a.cb + col;
        const int64_t q0 = a.bcp[bj], q1 = a.bcp[bj + 1];
        const int64_t nb = q1 - q0;
        const int64_t dst0 = a.stg_off[idx], cap = a.stg_off[idx + 1] - dst0;
        const int64_t ntiles = (r_hi - r_lo + TILE - 1) / TILE;
        const bool chunked = nb > kSweepSeg;
        // a sub-segment expecting >= kLongPerTile rows per tile is walked by a whole warp,
        // shorter ones by one lane each (R-MAT columns mix hub segments with 1-3 row ones)
        const uint32_t long_len = (uint32_t)(kLongPerTile * ntiles);
        int64_t written = 0;
        int nloc = 0, mloc = 0;  // candidates: statistics of all the part's entries
        double sloc = 0.0;
        // keep the top cand_k of the candidate buffer (value desc, row asc; order-preserving,
        // so the buffer stays sorted by row); later entries must beat its cut strictly
        auto reduce_cands = [&]() {
            uint32_t t = 0;
            int rowcut = 0;
            const int nc = s_ncand;
            radix_select_topk<NT, float>(crow, cval, nc, a.cand_k, t, rowcut, hist, sint);
            const int kept = compact_inplace<NT, float>(
                crow, cval, nc,
                [=](int k, float v) {
                    const uint32_t b = val_bits(v);
                    return b > t || (b == t && k <= rowcut);
                },
                sscan);
            if (tid == 0) {
                s_ncand = kept;
                s_thr = t;
                s_reduced = 1;
            }
            __syncthreads();
        };
        for (int64_t t0 = r_lo; t0 < r_hi; t0 += TILE) {
            const int tw = (int)((r_hi - t0) < TILE ? (r_hi - t0) : TILE);
            const int64_t t_end = t0 + tw;
            for (int i = tid; i < tw; i += NT) acc[i] = V(0);
            for (int64_t c0 = q0; c0 < q1; c0 += kSweepSeg) {
                const int cnt = (int)((q1 - c0) < kSweepSeg ? (q1 - c0) : kSweepSeg);
                if (t0 == r_lo || chunked) {
                    // the part's sub-segment of every A_*k (rowpart index), and for later
                    // tiles of a chunked column the cursor re-found at the tile's first row;
                    // empty ones are dropped, long ones listed from the front, short ones
                    // from the back
                    if (tid == 0) {
                        s_nL = 0;
                        s_nS = 0;
                    }
                    __syncthreads();
                    for (int i = tid; i < cnt; i += NT) {
                        const int k = __ldg(a.brow + c0 + i);
                        const int *pk = a.rowpart + (int64_t)k * (kParts + 1);
                        const uint32_t base = (uint32_t)__ldg(a.acp + k);
                        uint32_t s = base + (uint32_t)__ldg(pk + p0);
                        const uint32_t e = base + (uint32_t)__ldg(pk + p1);
                        if (t0 > r_lo) s = lower_row(a.apair, s, e, t0);
                        if (e > s) {
                            const int slot = (e - s >= long_len) ? atomicAdd(&s_nL, 1)
                                                                  : kSweepSeg - 1 - atomicAdd(&s_nS, 1);
                            cur[slot] = s;
                            end[slot] = e;
                            bkj[slot] = __ldg(a.bval + c0 + i);
                        }
                    }
                }
                if (tid == 0) {
                    s_nextL = 0;
                    s_nextS = 0;
                }
                __syncthreads();
                // warps take long segments one at a time, then short ones 32 at a time
                const int nL = s_nL, nS = s_nS;
                for (;;) {
                    int e0 = 0;
                    if (lane == 0) e0 = atomicAdd(&s_nextL, 1);
                    e0 = __shfl_sync(0xffffffffu, e0, 0);
                    if (e0 >= nL) break;
                    sweep_walk<32, V>(a.apair, acc, t0, t_end, cur, end, bkj, e0, true, !chunked);
                }
                for (;;) {
                    int e0 = 0;
                    if (lane == 0) e0 = atomicAdd(&s_nextS, 32);
                    e0 = __shfl_sync(0xffffffffu, e0, 0);
                    if (e0 >= nS) break;
                    const int e = e0 + lane;
                    sweep_walk<1, V>(a.apair, acc, t0, t_end, cur, end, bkj, kSweepSeg - 1 - e,
                                     e < nS, !chunked);
                }
                __syncthreads();
            }
            // the tile's touched rows.  Warp w owns the contiguous rows [w RW, (w+1) RW) of the
            // tile, so the compaction needs warp ballots, not CTA-wide scans (which cost ~5 warp
            // instructions per row of the whole row space swept by every dense column).
            constexpr int RW = TILE / 32;
            const int w = tid >> 5;
            const unsigned lt = (1u << lane) - 1u;
            if (cand) {
                // candidates: rounds of 32 rows per warp (<= NT appends per round, in any
                // order -- the final set is sorted by row below); the buffer is reduced
                // (CTA-uniform decision) before a round that could overflow it
                for (int r0 = 0; r0 < RW; r0 += 32) {
                    if (s_ncand > kCandBuf - NT) reduce_cands();
                    const int i = w * RW + r0 + lane;
                    const V v = i < tw ? acc[i] : V(0);
                    const int f = dense_touched(v);
                    const float vf = fabsf((float)v);
                    if (f) {
                        nloc++;
                        if ((double)vf >= theta) {
                            mloc++;
                            sloc += (double)vf;
                        }
                    }
                    const bool acc_c = f && (!s_reduced || val_bits(vf) > s_thr);
                    const unsigned bal = __ballot_sync(0xffffffffu, acc_c);
                    if (bal) {
                        int base = 0;
                        if (lane == 0) base = atomicAdd(&s_ncand, __popc(bal));
                        base = __shfl_sync(0xffffffffu, base, 0);
                        if (acc_c) {
                            crow[base + __popc(bal & lt)] = (int32_t)(t0 + i);
                            cval[base + __popc(bal & lt)] = vf;
                        }
                    }
                    __syncthreads();
                }
            } else {
                // every entry, in row order: per-warp counts, their scan, then the writes
                int cntw = 0;
                for (int r0 = 0; r0 < RW; r0 += 32) {
                    const int i = w * RW + r0 + lane;
                    cntw += __popc(__ballot_sync(0xffffffffu, i < tw && dense_touched(acc[i])));
                }
                if (lane == 0) s_wcnt[w] = cntw;
                __syncthreads();
                const int wc = s_wcnt[lane];
                int inc = wc;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += y;
                }
                int64_t off = written + __shfl_sync(0xffffffffu, inc - wc, w);
                const int total = __shfl_sync(0xffffffffu, inc, 31);
                for (int r0 = 0; r0 < RW; r0 += 32) {
                    const int i = w * RW + r0 + lane;
                    const V v = i < tw ? acc[i] : V(0);
                    const int f = dense_touched(v);
                    const unsigned bal = __ballot_sync(0xffffffffu, f);
                    const int64_t at = off + __popc(bal & lt);
                    if (f && at < cap) {
                        a.stg_row[dst0 + at] = (int32_t)(t0 + i);
                        a.stg_val[dst0 + at] = fabsf((float)v);
                    }
                    off += __popc(bal);
                }
                written += total;
            }
            __syncthreads();
        }
        if (cand) {
            if (s_ncand > a.cand_k) reduce_cands();
            // the part's candidates, sorted by row for the stitch (parts are row ranges)
            const int nc = s_ncand;
            int P = 1;
            while (P < nc) P <<= 1;
            for (int i = nc + tid; i < P; i += NT) crow[i] = kPadKey;
            __syncthreads();
            bitonic_sort<NT, float>(crow, cval, P);
            for (int i = tid; i < nc; i += NT) {
                a.stg_row[dst0 + i] = crow[i];
                a.stg_val[dst0 + i] = cval[i];
            }
            written = nc;
            const int n_all = block_sum<NT, int>(nloc, sscan);
            const int m_all = block_sum<NT, int>(mloc, sscan);
            const double s_all = block_sum<NT, double>(sloc, sred);
            if (tid == 0) {
                a.stg_nnz[idx] = n_all;
                a.stg_m[idx] = m_all;
                a.stg_s[idx] = s_all;
            }
        }
        if (tid == 0) {
            if (written > cap) {
                a.stg_cnt[idx] = 0;
                if (atomicExch(&a.col_flag[col], 1) == 0) a.retry_list[atomicAdd(a.retry_count, 1)] = col;
            } else {
                a.stg_cnt[idx] = written;
            }
        }
        __syncthreads();
    }
}

constexpr size_t kSweepSmem = kSweepTileBytes + (size_t)kSweepSeg * 12 + (size_t)kCandBuf * 8;

cudaError_t launch_dense_part(bool fp64, const BinArgs &a, int grid, cudaStream_t s) {
    ++g_launches;
    if (fp64) k_dense_sweep<double><<<grid, kDenseThreads, kSweepSmem, s>>>(a);
    else k_dense_sweep<float><<<grid, kDenseThreads, kSweepSmem, s>>>(a);
    return cudaGetLastError();
}

int dense_part_occupancy(bool fp64) {
    auto fn = fp64 ? k_dense_sweep<double> : k_dense_sweep<float>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepSmem);
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kDenseThreads, kSweepSmem);
    return nb;
}

}  // namespace mclx
