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
// Its lanes are split into groups of g in {4,8,16,32} lanes; each group gathers one
// operand column A_*k with coalesced loads (g chosen from flops_j / nnz(B_*j), the
// average gathered segment length) and inserts a_ik * b_kj into an open-addressing
// table keyed by row (shared memory in bins 0..5, global memory + fp64 in bin 6).
#include <type_traits>

#include "kernels.h"

namespace mclx {

template <typename V>
__device__ __forceinline__ int hash_accum(int *keys, V *vals, uint32_t cap, int row, V v) {
    uint32_t s = hash_slot(row, cap);
    volatile int *vk = keys;
    for (uint32_t p = 0; p < cap; ++p) {
        int k = vk[s];
        if (k == row) {
            atomicAdd(&vals[s], v);
            return 0;
        }
        if (k == kEmptyKey) {
            int old = atomicCAS(&keys[s], kEmptyKey, row);
            if (old == kEmptyKey) {
                atomicAdd(&vals[s], v);
                return 1;
            }
            if (old == row) {
                atomicAdd(&vals[s], v);
                return 0;
            }
        }
        s = (s + 1 == cap) ? 0u : s + 1;
    }
    return -1;
}

__device__ __forceinline__ int hash_key(int *keys, uint32_t cap, int row) {
    uint32_t s = hash_slot(row, cap);
    volatile int *vk = keys;
    for (uint32_t p = 0; p < cap; ++p) {
        int k = vk[s];
        if (k == row) return 0;
        if (k == kEmptyKey) {
            int old = atomicCAS(&keys[s], kEmptyKey, row);
            if (old == kEmptyKey) return 1;
            if (old == row) return 0;
        }
        s = (s + 1 == cap) ? 0u : s + 1;
    }
    return -1;
}

__device__ __forceinline__ int group_size(int64_t f, int64_t nb, int nt) {
    int64_t avg = nb > 0 ? f / nb : 0;
    int g = avg >= 24 ? 32 : avg >= 12 ? 16 : avg >= 6 ? 8 : 4;
    return g > nt ? nt : g;
}

__device__ __forceinline__ int next_pow2(int x) { return x <= 1 ? x : 1 << (32 - __clz(x - 1)); }

template <int CAP, int NT, int MODE, bool GLOBAL>
__global__ void __launch_bounds__(NT) k_bin(BinArgs a) {
    using V = typename std::conditional<GLOBAL, double, float>::type;
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ unsigned hist[256];
    __shared__ int sint[4];
    __shared__ double sred[NT / 32];
    __shared__ int sscan[NT / 32];
    __shared__ int s_col, s_idx, s_ovf;

    const int tid = threadIdx.x;
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

        const int64_t bj = a.cb + col;
        const int64_t q0 = a.bcp[bj], q1 = a.bcp[bj + 1];
        const int64_t nb = q1 - q0;
        const int g = group_size(a.flops[col], nb, NT);
        const int lane_g = tid & (g - 1);
        const int grp = tid / g;
        const int ngrp = NT / g;
        int fresh = 0;
        bool ok = true;
        for (int64_t q = q0 + grp; q < q1; q += ngrp) {
            const int k = __ldg(a.brow + q);
            const float bkj = __ldg(a.bval + q);
            const int64_t t0 = __ldg(a.acp + k), t1 = __ldg(a.acp + k + 1);
            for (int64_t t = t0 + lane_g; t < t1; t += g) {
                const int i = __ldg(a.arow + t);
                int rc;
                if (MODE == kSym) {
                    rc = hash_key(keys, cap, i);
                } else {
                    V prod = GLOBAL ? (V)__ldg(a.aval + t) * (V)bkj : (V)(__ldg(a.aval + t) * bkj);
                    rc = hash_accum<V>(keys, vals, cap, i, prod);
                }
                if (rc < 0) ok = false;
                fresh += rc > 0;
            }
        }
        if (!ok) s_ovf = 1;
        __syncthreads();
        if (s_ovf) {
            if (tid == 0) a.retry_list[atomicAdd(a.retry_count, 1)] = col;
            continue;  // loop head re-syncs before s_col is rewritten
        }

        if (MODE == kSym) {
            int nnz = block_sum<NT, int>(fresh, sscan);
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
            const int P = next_pow2(nnz);
            for (int i = nnz + tid; i < P; i += NT) keys[i] = kPadKey;
            __syncthreads();
            bitonic_sort<NT, V>(keys, vals, P);
            for (int i = tid; i < nnz; i += NT) {
                a.c_row[dst + i] = keys[i];
                a.c_val[dst + i] = (float)vals[i];
            }
            __syncthreads();
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

        const int P = next_pow2(kept);
        for (int i = kept + tid; i < P; i += NT) keys[i] = kPadKey;
        __syncthreads();
        bitonic_sort<NT, V>(keys, vals, P);
        const int64_t dst = a.soff[col];
        for (int i = tid; i < kept; i += NT) {
            a.s_row[dst + i] = keys[i];
            a.s_val[dst + i] = (float)(pow_r((double)vals[i], pp) / sr);
        }
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
        case 4: return WHAT<8192, 256, MODE, false>(__VA_ARGS__);                 \
        case 5: return WHAT<16384, 512, MODE, false>(__VA_ARGS__);                \
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
