// kernels_esc.cu -- the low-cf expansion kernel: expand, sort, compress
// (ESC) per output column, chosen per column when the compression factor is low.
//
// PAPER.md P:368-379 §III: hash SpGEMM suits high compression factors, while at cf near 1
// (late MCL iterations: each column of A_t holds a few large entries, so almost every
// product lands on its own row) a merge-based kernel does less work; HipMCL's hybrid picks
// the library per multiplication by cf and flops (§VII-B).  Here the
// choice is per column (k_classify): f_j <= kEscCap products and cf_j = f_j / nnz_j below
// the threshold (Cohen's estimate, or the exact symbolic size) run here instead of a hash
// bin.  One CTA per column:
//   expand   warps copy the products b_kj a_ik of the column's segments A_*k into shared
//            memory (row, value) arrays, lanes over a segment's entries (coalesced);
//   sort     bitonic sort by row (f_j <= kEscCap, padded to a power of two);
//   compress a row's run of equal rows is summed (fp64) by the run's head thread (a block
//            scan of the head flags gives each distinct row its output slot).
// The compressed column is sorted by construction, so kNum writes it out directly and kFused
// hands it to prune_column (threshold / select / recover / inflate, Q1-Q9); kSym counts it.
#include "kernels.h"

namespace mclx {

template <int MODE>
__global__ void __launch_bounds__(kEscThreads) k_esc(BinArgs a) {
    constexpr int NT = kEscThreads;
    __shared__ int srow[kEscCap], orow[kEscCap];
    __shared__ float sval[kEscCap], oval[kEscCap];
    __shared__ int64_t dstart[kEscCap];
    __shared__ int doff[kEscCap + 1];
    __shared__ float db[kEscCap];
    __shared__ unsigned hist[256];
    __shared__ int sint[4];
    __shared__ double sred[NT / 32];
    __shared__ int sscan[NT / 32];
    __shared__ int s_col;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int count = *a.count;
    for (;;) {
        if (tid == 0) {
            const int idx = atomicAdd(a.counter, 1);
            s_col = idx < count ? a.list[idx] : -1;
        }
        __syncthreads();
        const int col = s_col;
        if (col < 0) return;
        const int64_t bj = a.cb + col;
        const int64_t q0 = a.bcp[bj];
        const int nb = (int)(a.bcp[bj + 1] - q0);  // <= f_j <= kEscCap
        // ---- segment descriptors and their offsets in the flat product list
        int tot = 0;
        for (int i0 = 0; i0 < nb; i0 += NT) {
            const int i = i0 + tid;
            int len = 0;
            if (i < nb) {
                const int k = __ldg(a.brow + q0 + i);
                const int64_t st = __ldg(a.acp + k);
                len = (int)(__ldg(a.acp + k + 1) - st);
                dstart[i] = st;
                db[i] = __ldg(a.bval + q0 + i);
            }
            int t2;
            const int off = block_excl_scan<NT>(len, sscan, t2);
            if (i < nb) doff[i] = tot + off;
            tot += t2;
        }
        if (tid == 0) doff[nb] = tot;
        __syncthreads();
        const int f = tot;
        // ---- expand: warp w copies segments w, w + W, ... (lanes over entries)
        for (int s = warp; s < nb; s += NT / 32) {
            const int64_t st = dstart[s];
            const int o = doff[s], len = doff[s + 1] - o;
            const float b = db[s];
            for (int e = lane; e < len; e += 32) {
                srow[o + e] = __ldg(a.arow + st + e);
                sval[o + e] = MODE == kSym ? 0.f : __ldg(a.aval + st + e) * b;
            }
        }
        int P = 1;
        while (P < f) P <<= 1;
        for (int i = f + tid; i < P; i += NT) srow[i] = kPadKey;
        __syncthreads();
        // ---- sort by row
        bitonic_sort<NT, float>(srow, sval, P);
        // ---- compress: the head of each run of equal rows sums the run
        int nnz = 0;
        for (int i0 = 0; i0 < f; i0 += NT) {
            const int i = i0 + tid;
            const int head = i < f && (i == 0 || srow[i] != srow[i - 1]);
            int t2;
            const int pos = block_excl_scan<NT>(head, sscan, t2);
            if (head) {  // fp64 run sums (a forced ESC column may have long runs)
                double v = 0.0;
                for (int q = i; q < f && srow[q] == srow[i]; q++) v += (double)sval[q];
                orow[nnz + pos] = srow[i];
                oval[nnz + pos] = (float)v;
            }
            nnz += t2;
        }
        __syncthreads();
        if (MODE == kSym) {
            if (tid == 0) a.sym_nnz[col] = nnz;
        } else if (MODE == kNum) {
            const int64_t dst = a.c_cp[col];
            if (a.c_cnt) {
                if (tid == 0) a.c_cnt[col] = nnz;
            } else if (tid == 0 && a.c_cp[col + 1] - dst != nnz) {
                atomicExch(a.err_flag, 1);
            }
            for (int i = tid; i < nnz; i += NT) {
                a.c_row[dst + i] = orow[i];
                a.c_val[dst + i] = oval[i];
            }
        } else {
            prune_column<NT>(orow, oval, nnz, col, a.soff, a.s_row, a.s_val, a.s_cnt, a.chaos,
                             a.chaos_max, a.bin_out, a.pp, hist, sint, sred, sscan);
        }
        __syncthreads();
    }
}

cudaError_t launch_esc(int mode, const BinArgs &a, int grid, cudaStream_t s) {
    ++g_launches;
    if (mode == kSym) k_esc<kSym><<<grid, kEscThreads, 0, s>>>(a);
    else if (mode == kNum) k_esc<kNum><<<grid, kEscThreads, 0, s>>>(a);
    else k_esc<kFused><<<grid, kEscThreads, 0, s>>>(a);
    return cudaGetLastError();
}

int esc_occupancy(int mode) {
    int nb = 0;
    if (mode == kSym) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_esc<kSym>, kEscThreads, 0);
    else if (mode == kNum) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_esc<kNum>, kEscThreads, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_esc<kFused>, kEscThreads, 0);
    return nb;
}

}  // namespace mclx
