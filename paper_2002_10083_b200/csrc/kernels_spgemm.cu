// kernels_spgemm.cu -- the binned hash SpGEMM of the expansion step (PAPER.md P:159,
// Alg. 1 line 3) with its three epilogues:
//   kSym   exact symbolic pass (§V): distinct rows per output column;
//   kNum   unpruned numeric product, rows sorted ("obtained by sorting
//          the hash table");
//   kFused numeric product whose epilogue runs threshold / top-k select / recovery /
//          inflation / renormalisation on the column while it is still in the
//          shared-memory table (readings Q1-Q9), so the
//          unpruned product never reaches HBM.
//
// C_*j = sum_{k in inds(B_*j)} b_kj A_*k (Gustavson in CSC).  One CTA owns
// one output column at a time (persistent CTAs pull columns from the bin's work list).
//
// ATOMIC-FREE ACCUMULATION.  On sm_100 a shared-memory float atomicAdd is a CAS spin
// loop (ATOMS.CAST.SPIN) and shared atomics issue at ~2 cycles/lane, which caps an
// atomic-per-product hash at ~0.3 products/cycle/SM.  Instead, the row space [0, m)
// is cut into 32 ranges (rowpart index P[k][0..32] of A, computed once per call:
// P[k][i] = first position in A_*k whose row is >= ceil(i*m/32)).  The CTA's W = NT/32
// warps each own W-th of the ranges and a private W-th slice of the hash table, and
// gather only their sub-segment of every A_*k.  A warp therefore never shares a slot
// with another warp; inside the warp, the claim of an empty slot is resolved
// warp-synchronously (__match_any_sync on the slot) and the value update is a plain
// LDS/FADD/STS.  Lanes holding the same row in one instruction (possible when a warp
// gathers several short sub-segments at once) are serialised by their match rank.
// Because ranges are ordered, the compacted table is grouped by row range.
#include <type_traits>

#include "kernels.h"

namespace mclx {

constexpr int kParts = 32;  // row ranges of the rowpart index
constexpr int kUnroll = 4;  // independent (row, val) gathers per lane in flight

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Warp-synchronous insert of one (row, v) per valid lane into this warp's private
// slice (keys, vals)[0, scap).  All 32 lanes must call it (uniform control flow).
// Returns false (warp-uniform) when the slice's fill would pass `limit`.
template <int MODE, typename V>
__device__ __forceinline__ bool warp_insert(int *keys, V *vals, uint32_t scap, bool valid, int row,
                                            V v, bool may_dup, int &fill, int limit) {
    const unsigned FULL = 0xffffffffu;
    const int lane = lane_id();
    if (!__any_sync(FULL, valid)) return true;
    int rank = 0;
    unsigned maxrank = 0;
    if (may_dup) {
        const unsigned m = __match_any_sync(FULL, valid ? row : -1 - lane);
        rank = __popc(m & lanemask_lt());
        maxrank = __reduce_max_sync(FULL, valid ? (unsigned)rank : 0u);
    }
    uint32_t s = hash_slot(row, scap);
    for (unsigned r = 0; r <= maxrank; r++) {
        bool me = valid && rank == (int)r;
        while (__any_sync(FULL, me)) {
            const int k = me ? keys[s] : 0;
            const bool hit = me && k == row;
            const bool emp = me && k == kEmptyKey;
            bool claimed = false;
            const unsigned em = __ballot_sync(FULL, emp);
            if (em) {
                const unsigned grp = __match_any_sync(FULL, emp ? (int)s : -1 - lane);
                claimed = emp && (__ffs(grp) - 1) == lane;
                if (claimed) keys[s] = row;
                fill += __popc(__ballot_sync(FULL, claimed));
                if (fill > limit) return false;
            }
            if (MODE != kSym && (hit || claimed)) vals[s] += v;
            if (me && !hit && !emp) s = (s + 1 == scap) ? 0u : s + 1;
            __syncwarp();
            if (hit || claimed) me = false;
        }
    }
    return true;
}

__device__ __forceinline__ int group_size_for(int64_t avg) {
    return avg >= 24 ? 32 : avg >= 12 ? 16 : avg >= 6 ? 8 : 4;
}

template <int CAP, int NT, int MODE, bool GLOBAL>
__global__ void __launch_bounds__(NT, 1024 / NT) k_bin(BinArgs a) {
    using V = typename std::conditional<GLOBAL, double, float>::type;
    constexpr int W = NT / 32;            // warps = row-range owners
    constexpr int PSTEP = kParts / W;     // rowpart boundaries per warp
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ unsigned hist[256];
    __shared__ int sint[4];
    __shared__ double sred[NT / 32];
    __shared__ int sscan[NT / 32];
    __shared__ int s_col, s_idx, s_ovf;
    __shared__ int64_t st_start[NT];
    __shared__ int st_k[NT];
    __shared__ float st_b[NT];

    const int tid = threadIdx.x;
    const int lane = lane_id();
    const int warp = warp_id();
    const int count = *a.count;
    for (;;) {
        if (tid == 0) {
            int idx = atomicAdd(a.counter, 1);
            s_idx = idx;
            s_col = idx < count ? a.list[idx] : -1;
            s_ovf = 0;
        }
        __syncthreads();
        const int col = s_col;
        const int idx = s_idx;
        if (col < 0) return;

        int *keys;
        V *vals;
        uint32_t cap;
        if (GLOBAL) {
            keys = a.gkeys + a.goff[idx];
            vals = reinterpret_cast<V *>(a.gvals + a.goff[idx]);
            cap = (uint32_t)a.gcap[idx];
        } else {
            keys = reinterpret_cast<int *>(dsm);
            vals = reinterpret_cast<V *>(dsm + (size_t)CAP * sizeof(int));
            cap = CAP;
        }
        for (uint32_t i = tid; i < cap; i += NT) {
            keys[i] = kEmptyKey;
            if (MODE != kSym) vals[i] = V(0);
        }
        __syncthreads();

        // ---- accumulate: warp `warp` gathers rows in its ranges [warp*PSTEP, +PSTEP)
        const uint32_t scap = cap / W;
        int *wkeys = keys + (size_t)warp * scap;
        V *wvals = vals + (size_t)warp * scap;
        const int limit = (int)(scap - (scap >> 3));
        const int64_t bj = a.cb + col;
        const int64_t q0 = a.bcp[bj], q1 = a.bcp[bj + 1];
        const int64_t nb = q1 - q0;
        const int g = group_size_for(nb > 0 ? a.flops[col] / (nb * W) : 0);
        const int lane_g = lane & (g - 1);
        const int grp = lane / g;
        const int G = 32 / g;  // segments a warp gathers side by side
        const bool may_dup = G > 1;
        int fill = 0;
        bool ok = true;
        for (int64_t c0 = q0; c0 < q1; c0 += NT) {
            const int cnt = (int)((q1 - c0) < NT ? (q1 - c0) : NT);
            if (tid < cnt) {
                const int k = __ldg(a.brow + c0 + tid);
                st_k[tid] = k;
                st_start[tid] = __ldg(a.acp + k);
                st_b[tid] = __ldg(a.bval + c0 + tid);
            }
            __syncthreads();
            if (ok) {
                for (int e0 = 0; e0 < cnt; e0 += G) {
                    const int e = e0 + grp;
                    int64_t lo = 0;
                    int len = 0;
                    float bkj = 0.f;
                    if (e < cnt) {
                        const int k = st_k[e];
                        const int *pk = a.rowpart + (int64_t)k * (kParts + 1) + warp * PSTEP;
                        const int p0 = __ldg(pk), p1 = __ldg(pk + PSTEP);
                        lo = st_start[e] + p0;
                        len = p1 - p0;
                        bkj = st_b[e];
                    }
                    const unsigned nbatch = (unsigned)((len + g * kUnroll - 1) / (g * kUnroll));
                    const unsigned maxb = __reduce_max_sync(0xffffffffu, nbatch);
                    for (unsigned bi = 0; bi < maxb && ok; bi++) {
                        int rr[kUnroll];
                        V vv[kUnroll];
#pragma unroll
                        for (int u = 0; u < kUnroll; u++) {
                            const int t = (int)bi * g * kUnroll + u * g + lane_g;
                            rr[u] = t < len ? __ldg(a.arow + lo + t) : -1;
                            float av = (MODE != kSym && t < len) ? __ldg(a.aval + lo + t) : 0.f;
                            vv[u] = GLOBAL ? (V)av * (V)bkj : (V)(av * bkj);
                        }
#pragma unroll
                        for (int u = 0; u < kUnroll; u++) {
                            if (!warp_insert<MODE, V>(wkeys, wvals, scap, rr[u] >= 0, rr[u], vv[u],
                                                      may_dup, fill, limit)) {
                                ok = false;
                                break;
                            }
                        }
                    }
                    if (!ok) break;
                }
            }
            __syncthreads();
        }
        if (!ok && lane == 0) s_ovf = 1;
        __syncthreads();
        if (s_ovf) {
            if (tid == 0) a.retry_list[atomicAdd(a.retry_count, 1)] = col;
            continue;  // loop head re-syncs before s_col is rewritten
        }

        if (MODE == kSym) {
            const int nnz = block_sum<NT, int>(lane == 0 ? fill : 0, sscan);
            if (tid == 0) a.sym_nnz[col] = nnz;
            __syncthreads();
            continue;
        }

        // ---- compact occupied slots to the front of the table
        const int nnz = compact_inplace<NT, V>(
            keys, vals, (int)cap, [](int k, V) { return k != kEmptyKey; }, sscan);

        if (MODE == kNum) {
            const int64_t dst = a.c_cp[col];
            if (tid == 0 && a.c_cp[col + 1] - dst != nnz) atomicExch(a.err_flag, 1);
            sort_write<NT, V>(keys, vals, nnz, (int)cap, a.c_row + dst, a.c_val + dst,
                              [](V v) { return (float)v; }, sscan);
            continue;
        }

        // ---- kFused: threshold statistics (Q3, Q4)
        const PruneParams &pp = a.pp;
        int mloc = 0;
        double sloc = 0.0;
        for (int i = tid; i < nnz; i += NT) {
            double v = (double)vals[i];
            if (v >= pp.theta) {
                mloc++;
                sloc += v;
            }
        }
        const int m = block_sum<NT, int>(mloc, sscan);
        const double s = block_sum<NT, double>(sloc, sred);
        int64_t K;
        const int br = prune_branch(pp, nnz, m, s, K);
        uint32_t t = 0;
        int rowcut = 0;
        int sel = 0;  // 0: v >= theta, 1: top-K, 2: all
        if (br == 0) {
            sel = 0;
        } else if (K >= nnz) {
            sel = 2;
        } else {
            radix_select_topk<NT, V>(keys, vals, nnz, (int)K, t, rowcut, hist, sint);
            sel = 1;
        }
        const double theta = pp.theta;
        const int kept = compact_inplace<NT, V>(
            keys, vals, nnz,
            [=](int k, V v) {
                if (sel == 0) return (double)v >= theta;
                if (sel == 2) return true;
                uint32_t b = val_bits(v);
                return b > t || (b == t && k <= rowcut);
            },
            sscan);
        if (tid == 0 && kept != (int)K) atomicExch(a.err_flag, 2);

        // ---- renormalise, chaos (Q9), inflate, renormalise (Q1)
        double sv = 0.0, mx = 0.0, sq = 0.0, sr = 0.0;
        for (int i = tid; i < kept; i += NT) {
            double v = (double)vals[i];
            sv += v;
            mx = v > mx ? v : mx;
            sq += v * v;
            sr += pow_r(v, pp);
        }
        sv = block_sum<NT, double>(sv, sred);
        mx = block_max<NT, double>(mx, sred);
        sq = block_sum<NT, double>(sq, sred);
        sr = block_sum<NT, double>(sr, sred);
        const float chaos = kept > 0 ? (float)((double)kept * (mx / sv - sq / (sv * sv))) : 0.0f;

        const int64_t dst = a.soff[col];
        sort_write<NT, V>(keys, vals, kept, (int)cap, a.s_row + dst, a.s_val + dst,
                          [&](V v) { return (float)(pow_r((double)v, pp) / sr); }, sscan);
        if (tid == 0) {
            a.s_cnt[col] = kept;
            a.chaos[col] = chaos;
            atomicAdd(a.bin_out, (unsigned long long)kept);
            atomic_max_nonneg_float(a.chaos_max, chaos);
        }
        __syncthreads();
    }
}

template <int CAP, int NT, int MODE, bool GLOBAL>
static size_t smem_of() {
    if (GLOBAL) return 0;
    return (size_t)CAP * (MODE == kSym ? 4 : 8);
}

template <int CAP, int NT, int MODE, bool GLOBAL>
static int occ_of() {
    auto fn = k_bin<CAP, NT, MODE, GLOBAL>;
    size_t sm = smem_of<CAP, NT, MODE, GLOBAL>();
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, NT, sm);
    return nb;
}

template <int CAP, int NT, int MODE, bool GLOBAL>
static cudaError_t launch_of(const BinArgs &a, int grid, cudaStream_t s) {
    ++g_launches;
    k_bin<CAP, NT, MODE, GLOBAL><<<grid, NT, smem_of<CAP, NT, MODE, GLOBAL>(), s>>>(a);
    return cudaGetLastError();
}

#define MCLX_BIN_SWITCH(MODE, WHAT, ...)                                          \
    switch (bin) {                                                                \
        case 0: return WHAT<512, 64, MODE, false>(__VA_ARGS__);                   \
        case 1: return WHAT<1024, 64, MODE, false>(__VA_ARGS__);                  \
        case 2: return WHAT<2048, 128, MODE, false>(__VA_ARGS__);                 \
        case 3: return WHAT<4096, 256, MODE, false>(__VA_ARGS__);                 \
        case 4: return WHAT<8192, 512, MODE, false>(__VA_ARGS__);                 \
        case 5: return WHAT<16384, 1024, MODE, false>(__VA_ARGS__);               \
        default: return WHAT<0, kGlobalThreads, MODE, true>(__VA_ARGS__);         \
    }

cudaError_t launch_bin(int mode, int bin, const BinArgs &a, int grid, cudaStream_t s) {
    if (mode == kSym) { MCLX_BIN_SWITCH(kSym, launch_of, a, grid, s) }
    if (mode == kNum) { MCLX_BIN_SWITCH(kNum, launch_of, a, grid, s) }
    MCLX_BIN_SWITCH(kFused, launch_of, a, grid, s)
}

int bin_occupancy(int mode, int bin) {
    if (mode == kSym) { MCLX_BIN_SWITCH(kSym, occ_of) }
    if (mode == kNum) { MCLX_BIN_SWITCH(kNum, occ_of) }
    MCLX_BIN_SWITCH(kFused, occ_of)
}

size_t bin_smem_bytes(int mode, int bin) {
    if (mode == kSym) { MCLX_BIN_SWITCH(kSym, smem_of) }
    if (mode == kNum) { MCLX_BIN_SWITCH(kNum, smem_of) }
    MCLX_BIN_SWITCH(kFused, smem_of)
}

}  // namespace mclx
