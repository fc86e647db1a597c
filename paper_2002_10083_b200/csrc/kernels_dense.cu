// kernels_dense.cu -- the dense bin of the expansion step (SURVEY §8(a) a4 "dense": the
// R-MAT hub columns of C4, whose product covers a sizable share of the row space).
//
// Such a column is run as 32 row-range parts (rowparts of A, as the split path), each a
// (column, row tile) work item of one CTA: rows [ceil(p0 m/32), ceil(p1 m/32)) accumulate
// into a dense tile in shared memory (kDenseTileBytes: 24576 fp64 or 49152 fp32 rows per
// pass; wider parts sweep several passes, re-reading their sub-segments and skipping
// rows outside the pass).  No hashing: the slot is the row.  A touched row is one with a
// value > 0 -- fp64 products of positive fp32 values never underflow; an fp32 product
// that underflows to 0 marks its row with -0.0 instead (Q13: the entry stays in the
// structure) -- so compacting a tile emits its rows in ascending order, no sort.  Values
// are added with shared-memory atomics (groups of lanes share a segment; a CAS loop on
// sm_100).  fp64 tiles for columns with more than kFp64Terms segments (T), fp32 otherwise
// (as the hashed bins).  Entries go to the item's
// staging slot, which the split path stitches and prunes (k_prune); more entries than
// the slot holds flag the column for the next round.
//
// Tried and dropped (kept here as a note): one L2-resident fp64 array of m rows per
// column, products added by RED.ADD.F64 from CTAs splitting the column by segments
// (~210 G atomics/s into L2-resident arrays, tools/ubench_red.cu).  The L2 budget admits
// only a few columns in flight, and each column's compaction + prune then runs in one
// CTA on the critical path: 10x slower than the tiles on R-MAT scale 20.
#include "kernels.h"

namespace mclx {

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

__device__ __forceinline__ int dense_group_size(int64_t avg) {
    return avg >= 24 ? 32 : avg >= 12 ? 16 : avg >= 6 ? 8 : avg >= 3 ? 4 : avg >= 2 ? 2 : 1;
}

template <typename V>
__global__ void __launch_bounds__(kDenseThreads, 1) k_dense_part(BinArgs a) {
    constexpr int NT = kDenseThreads;
    constexpr int TILE = kDenseTileBytes / (int)sizeof(V);
    extern __shared__ __align__(16) unsigned char dsm[];
    V *acc = reinterpret_cast<V *>(dsm);
    __shared__ int64_t st_start[NT];
    __shared__ int st_k[NT];
    __shared__ float st_b[NT];
    __shared__ int sscan[NT / 32];
    __shared__ int s_col, s_idx, s_pr, s_next;
    const int tid = threadIdx.x;
    const int count = *a.count;
    for (;;) {
        if (tid == 0) {
            const int idx = atomicAdd(a.counter, 1);
            s_idx = idx;
            s_col = idx < count ? a.list[idx] : -1;
            s_pr = idx < count ? a.item_pr[idx] : 0;
            s_next = 0;
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
        const int64_t fpart = a.flops[col] * (p1 - p0) / kParts;
        const int g = dense_group_size(nb > 0 ? fpart / nb : 0);
        const int lane_g = tid & (g - 1);
        int64_t written = 0;
        for (int64_t t0 = r_lo; t0 < r_hi; t0 += TILE) {
            const int tw = (int)((r_hi - t0) < TILE ? (r_hi - t0) : TILE);
            for (int i = tid; i < tw; i += NT) acc[i] = V(0);
            __syncthreads();
            for (int64_t c0 = q0; c0 < q1; c0 += NT) {
                const int cnt = (int)((q1 - c0) < NT ? (q1 - c0) : NT);
                if (tid < cnt) {
                    const int k = __ldg(a.brow + c0 + tid);
                    const int *pk = a.rowpart + (int64_t)k * (kParts + 1);
                    const int e0 = __ldg(pk + p0), e1 = __ldg(pk + p1);
                    st_start[tid] = __ldg(a.acp + k) + e0;
                    st_k[tid] = e1 - e0;
                    st_b[tid] = __ldg(a.bval + c0 + tid);
                }
                __syncthreads();
                // segments handed to warps dynamically (32/g at a time), so warps that drew
                // short segments take more instead of idling at the batch barrier; the row
                // and value of an entry are loaded together (one round trip, not two)
                for (;;) {
                    int e0 = 0;
                    if ((tid & 31) == 0) e0 = atomicAdd(&s_next, 32 / g);
                    e0 = __shfl_sync(0xffffffffu, e0, 0);
                    if (e0 >= cnt) break;
                    const int e = e0 + (tid & 31) / g;
                    if (e >= cnt) continue;
                    const int64_t s0 = st_start[e];
                    const int len = st_k[e];
                    const V b = (V)st_b[e];
                    for (int i = lane_g; i < len; i += g) {
                        const int r = __ldg(a.arow + s0 + i);
                        const float av = __ldg(a.aval + s0 + i);
                        if (r >= t0 + tw) break;  // rows ascend: the rest is past this pass
                        if (r < t0) continue;
                        const V prod = (V)av * b;
                        if (prod > V(0)) atomicAdd(&acc[r - t0], prod);
                        else atomic_mark_zero(&acc[r - t0]);  // fp32 underflow: keep the entry
                    }
                }
                __syncthreads();
                if (tid == 0) s_next = 0;
            }
            // the pass's touched rows, in row order
            for (int i0 = 0; i0 < tw; i0 += NT) {
                const int i = i0 + tid;
                const V v = i < tw ? acc[i] : V(0);
                // fp64: value > 0 is the structure; fp32 products can underflow to 0, so
                // a touched-but-zero entry is marked by the sign bit (see the add below)
                const int f = dense_touched(v);
                int tot;
                const int pos = block_excl_scan<NT>(f, sscan, tot);
                if (f && written + pos < cap) {
                    a.stg_row[dst0 + written + pos] = (int32_t)(t0 + i);
                    a.stg_val[dst0 + written + pos] = fabsf((float)v);
                }
                written += tot;
            }
            __syncthreads();
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

cudaError_t launch_dense_part(bool fp64, const BinArgs &a, int grid, cudaStream_t s) {
    ++g_launches;
    if (fp64) k_dense_part<double><<<grid, kDenseThreads, kDenseTileBytes, s>>>(a);
    else k_dense_part<float><<<grid, kDenseThreads, kDenseTileBytes, s>>>(a);
    return cudaGetLastError();
}

int dense_part_occupancy(bool fp64) {
    auto fn = fp64 ? k_dense_part<double> : k_dense_part<float>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kDenseTileBytes);
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kDenseThreads, kDenseTileBytes);
    return nb;
}

}  // namespace mclx
