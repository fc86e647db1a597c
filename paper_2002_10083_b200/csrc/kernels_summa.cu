// kernels_summa.cu -- device kernels of the 2D Sparse-SUMMA iteration (PAPER.md P:222-246
// §II "Overview of Sparse SUMMA"; "selecting top-k entries in each process and then
// exchanging").
//
//   panel extraction   A-panel = columns K_q of the local block (col_ptr rebased),
//                      B-panel = rows K_q of the local block (row ids rebased to K_q);
//   distributed prune  a column of C is split over the pr ranks of its column
//                      communicator.  Every exchange is a fixed-size NCCL all-reduce:
//                      per-column (nnz, m, s) sums decide the branch (Q5, Q7, Q8); the
//                      exact top-K cut is found by a radix select whose 256-bin digit
//                      histograms are all-reduced (4 passes on the fp32 bits of the value,
//                      then 4 on the global row id for ties); the kept set's sums are
//                      all-reduced for renormalisation, chaos and inflation.
#include <algorithm>

#include "kernels.h"

namespace mclx {

// ------------------------------------------------------------------ panels
__global__ void k_rebase_colptr(int64_t n1, const int64_t *__restrict__ cp, int64_t *__restrict__ out) {
    const int64_t base = cp[0];
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n1;
         j += (int64_t)gridDim.x * blockDim.x)
        out[j] = cp[j] - base;
}
cudaError_t launch_rebase_colptr(int64_t n1, const int64_t *cp, int64_t *out, cudaStream_t s) {
    if (n1 <= 0) return cudaSuccess;
    int64_t b = (n1 + 255) / 256;
    if (b > g_sms * 16) b = g_sms * 16;
    ++g_launches;
    k_rebase_colptr<<<(int)b, 256, 0, s>>>(n1, cp, out);
    return cudaGetLastError();
}

// Column j of the vertical stack of the s B-panels (row ranges K_q of the column stripe):
// panel 0's column j, then panel 1's (rows + k0_1), ... -- rows stay sorted because the K_q
// ascend.  Gives rank (i, j) the column stripe A[:, cols_j] as one CSC.
__global__ void k_vstack_count(int64_t nj, VStack v, int64_t *__restrict__ cnt) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nj;
         j += (int64_t)gridDim.x * blockDim.x) {
        int64_t c = 0;
        for (int q = 0; q < v.s; q++) c += v.cp[q][j + 1] - v.cp[q][j];
        cnt[j] = c;
    }
}
__global__ void k_vstack_copy(int64_t nj, VStack v, const int64_t *__restrict__ ocp,
                              int32_t *__restrict__ orow, float *__restrict__ oval) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = w0; j < nj; j += nw) {
        int64_t o = ocp[j];
        for (int q = 0; q < v.s; q++) {
            const int64_t a = v.cp[q][j], b = v.cp[q][j + 1];
            for (int64_t e = a + lane; e < b; e += 32) {
                orow[o + e - a] = (int32_t)(v.row[q][e] + v.k0[q]);
                oval[o + e - a] = v.val[q][e];
            }
            o += b - a;
        }
    }
}
cudaError_t launch_vstack(int64_t nj, const VStack &v, int64_t *cnt, const int64_t *ocp, int32_t *orow,
                          float *oval, bool count_only, cudaStream_t s) {
    if (nj <= 0) return cudaSuccess;
    ++g_launches;
    if (count_only) {
        int64_t b = (nj + 255) / 256;
        if (b > g_sms * 16) b = g_sms * 16;
        k_vstack_count<<<(int)b, 256, 0, s>>>(nj, v, cnt);
    } else {
        int64_t b = (nj * 32 + 255) / 256;
        if (b > g_sms * 32) b = g_sms * 32;
        k_vstack_copy<<<(int)b, 256, 0, s>>>(nj, v, ocp, orow, oval);
    }
    return cudaGetLastError();
}

__device__ __forceinline__ int64_t lb_rows(const int32_t *rows, int64_t lo, int64_t hi, int64_t key) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)rows[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}
// per column: first position with row >= r0 and the count of rows in [r0, r1)
__global__ void k_rowslice_count(int64_t ncols, const int64_t *__restrict__ cp,
                                 const int32_t *__restrict__ rows, int64_t r0, int64_t r1,
                                 int64_t *__restrict__ first, int64_t *__restrict__ cnt) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < ncols;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = lb_rows(rows, cp[j], cp[j + 1], r0);
        const int64_t b = lb_rows(rows, a, cp[j + 1], r1);
        first[j] = a;
        cnt[j] = b - a;
    }
}
cudaError_t launch_rowslice_count(int64_t ncols, const int64_t *cp, const int32_t *rows, int64_t r0,
                                  int64_t r1, int64_t *first, int64_t *cnt, cudaStream_t s) {
    if (ncols <= 0) return cudaSuccess;
    int64_t b = (ncols + 255) / 256;
    if (b > g_sms * 16) b = g_sms * 16;
    ++g_launches;
    k_rowslice_count<<<(int)b, 256, 0, s>>>(ncols, cp, rows, r0, r1, first, cnt);
    return cudaGetLastError();
}
__global__ void k_rowslice_copy(int64_t ncols, const int64_t *__restrict__ first,
                                const int64_t *__restrict__ ocp, const int32_t *__restrict__ rows,
                                const float *__restrict__ vals, int64_t r0,
                                int32_t *__restrict__ orow, float *__restrict__ oval) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = lane_id();
    for (int64_t j = w; j < ncols; j += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t src = first[j], dst = ocp[j], n = ocp[j + 1] - dst;
        for (int64_t i = lane; i < n; i += 32) {
            orow[dst + i] = (int32_t)(rows[src + i] - r0);
            oval[dst + i] = vals[src + i];
        }
    }
}
cudaError_t launch_rowslice_copy(int64_t ncols, const int64_t *first, const int64_t *ocp,
                                 const int32_t *rows, const float *vals, int64_t r0, int32_t *orow,
                                 float *oval, cudaStream_t s) {
    if (ncols <= 0) return cudaSuccess;
    int64_t b = (ncols * 32 + 255) / 256;
    if (b > g_sms * 32) b = g_sms * 32;
    ++g_launches;
    k_rowslice_copy<<<(int)b, 256, 0, s>>>(ncols, first, ocp, rows, vals, r0, orow, oval);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ distributed prune
constexpr int kDP = 256;

// One warp per column in every kernel below: block columns hold a few hundred entries,
// so warp shuffles / ballots replace block barriers.
__device__ __forceinline__ int64_t dp_warp0() {
    return ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
}
__device__ __forceinline__ int64_t dp_wstride() { return ((int64_t)gridDim.x * blockDim.x) >> 5; }
static int dp_grid(int64_t ncols) {
    int64_t b = (ncols * 32 + kDP - 1) / kDP;
    if (b > g_sms * 32) b = g_sms * 32;
    return b < 1 ? 1 : (int)b;
}

// local threshold statistics per column: nnz, m = #{v >= theta}, s = sum{v >= theta}
__global__ void __launch_bounds__(kDP) k_dp_stats(int64_t ncols, const int64_t *__restrict__ cp,
                                                  const float *__restrict__ vals, double theta,
                                                  int64_t *__restrict__ nnz, int64_t *__restrict__ m,
                                                  double *__restrict__ sm) {
    const int lane = lane_id();
    for (int64_t j = dp_warp0(); j < ncols; j += dp_wstride()) {
        const int64_t a = cp[j], b = cp[j + 1];
        int64_t mloc = 0;
        double sloc = 0.0;
        for (int64_t t = a + lane; t < b; t += 32) {
            const double v = (double)vals[t];
            if (v >= theta) {
                mloc++;
                sloc += v;
            }
        }
        mloc = warp_sum(mloc);
        sloc = warp_sum(sloc);
        if (lane == 0) {
            nnz[j] = b - a;
            m[j] = mloc;
            sm[j] = sloc;
        }
    }
}
cudaError_t launch_dp_stats(int64_t ncols, const int64_t *cp, const float *vals, double theta,
                            int64_t *nnz, int64_t *m, double *sm, int grid, cudaStream_t s) {
    if (ncols <= 0) return cudaSuccess;
    (void)grid;
    ++g_launches;
    k_dp_stats<<<dp_grid(ncols), kDP, 0, s>>>(ncols, cp, vals, theta, nnz, m, sm);
    return cudaGetLastError();
}

// Branch per column from the GLOBAL statistics (same on every rank of the column
// communicator).  mode: 0 thresh, 1 top-K select, 2 keep all, 3 empty.  Columns that
// need the select are appended to `sel` (order irrelevant; each rank builds the same
// set, and the histograms are indexed by column, not by list position).
__global__ void k_dp_branch(int64_t ncols, const int64_t *__restrict__ nnz,
                            const int64_t *__restrict__ m, const double *__restrict__ sm,
                            PruneParams pp, int64_t *__restrict__ K, int8_t *__restrict__ mode,
                            int32_t *__restrict__ rem, uint32_t *__restrict__ prefix,
                            int32_t *__restrict__ rowcut) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < ncols;
         j += (int64_t)gridDim.x * blockDim.x) {
        int64_t k;
        const int br = prune_branch(pp, nnz[j], m[j], sm[j], k);
        int8_t md;
        if (br == 4) md = 3;
        else if (br == 0) md = 0;
        else if (k >= nnz[j]) md = 2;
        else md = 1;
        K[j] = k;
        mode[j] = md;
        rem[j] = (int32_t)k;
        prefix[j] = 0;
        rowcut[j] = 0x7fffffff;
    }
}
cudaError_t launch_dp_branch(int64_t ncols, const int64_t *nnz, const int64_t *m, const double *sm,
                             const PruneParams &pp, int64_t *K, int8_t *mode, int32_t *rem,
                             uint32_t *prefix, int32_t *rowcut, cudaStream_t s) {
    if (ncols <= 0) return cudaSuccess;
    int64_t b = (ncols + 255) / 256;
    if (b > g_sms * 16) b = g_sms * 16;
    ++g_launches;
    k_dp_branch<<<(int)b, 256, 0, s>>>(ncols, nnz, m, sm, pp, K, mode, rem, prefix, rowcut);
    return cudaGetLastError();
}

// Local 256-bin digit histogram of pass p for every select column (hist[li][256] for list
// index li).  Passes 0-3: value bits, digit (bits >> (24-8p)) among entries whose higher
// bits match the prefix.  Passes 4-7: global row id bits among entries whose value bits
// equal the cut t = vprefix.  One warp per column with a warp-private smem histogram.
__global__ void __launch_bounds__(kDP) k_dp_hist(int64_t nsel, const int32_t *__restrict__ sel,
                                                 const int64_t *__restrict__ cp,
                                                 const int32_t *__restrict__ rows,
                                                 const float *__restrict__ vals, int64_t row0,
                                                 const int8_t *__restrict__ mode,
                                                 const uint32_t *__restrict__ vprefix,
                                                 const uint32_t *__restrict__ rprefix,
                                                 const int32_t *__restrict__ done, int pass,
                                                 unsigned *__restrict__ hist, int packed,
                                                 const int64_t *__restrict__ ccnt) {
    __shared__ unsigned hs[kDP / 32][256];
    unsigned *h = hs[threadIdx.x >> 5];
    const int lane = lane_id();
    for (int64_t li = dp_warp0(); li < nsel; li += dp_wstride()) {
        const int64_t j = sel[li];
        for (int i = lane; i < 256; i += 32) h[i] = 0;
        __syncwarp();
        if (!done[j]) {
            const int64_t a = cp[j], b = ccnt ? a + ccnt[j] : cp[j + 1];
            if (pass < 4) {
                const int shift = 24 - 8 * pass;
                const uint32_t mask = pass == 0 ? 0u : (0xFFFFFFFFu << (32 - 8 * pass));
                const uint32_t pre = vprefix[j];
                for (int64_t t = a + lane; t < b; t += 32) {
                    const uint32_t bits = __float_as_uint(vals[t]);
                    if ((bits & mask) == pre) atomicAdd(&h[(bits >> shift) & 255u], 1u);
                }
            } else {
                const int q = pass - 4;
                const int shift = 24 - 8 * q;
                const uint32_t mask = q == 0 ? 0u : (0xFFFFFFFFu << (32 - 8 * q));
                const uint32_t t0 = vprefix[j], pre = rprefix[j];
                for (int64_t t = a + lane; t < b; t += 32) {
                    const uint32_t grow = (uint32_t)(row0 + rows[t]);
                    if (__float_as_uint(vals[t]) == t0 && (grow & mask) == pre)
                        atomicAdd(&h[(grow >> shift) & 255u], 1u);
                }
            }
        }
        __syncwarp();
        if (packed)  // bins b and b + 128 as the low / high 16 bits (counts < 2^16 summed)
            for (int i = lane; i < 128; i += 32) hist[li * 128 + i] = h[i] | (h[i + 128] << 16);
        else
            for (int i = lane; i < 256; i += 32) hist[li * 256 + i] = h[i];
        __syncwarp();
    }
}
cudaError_t launch_dp_hist(int64_t nsel, const int32_t *sel, const int64_t *cp, const int32_t *rows,
                           const float *vals, int64_t row0, const int8_t *mode,
                           const uint32_t *vprefix, const uint32_t *rprefix, const int32_t *done,
                           int pass, unsigned *hist, int grid, cudaStream_t s, int packed,
                           const int64_t *ccnt) {
    if (nsel <= 0) return cudaSuccess;
    (void)grid;
    ++g_launches;
    k_dp_hist<<<dp_grid(nsel), kDP, 0, s>>>(nsel, sel, cp, rows, vals, row0, mode, vprefix, rprefix,
                                             done, pass, hist, packed, ccnt);
    return cudaGetLastError();
}

// Digit step of pass p from the GLOBAL histogram: one warp per select column.
__global__ void k_dp_digit(int64_t nsel, const int32_t *__restrict__ sel,
                           const unsigned *__restrict__ hist, int pass, uint32_t *__restrict__ vprefix,
                           uint32_t *__restrict__ rprefix, int32_t *__restrict__ rem,
                           int32_t *__restrict__ done, int32_t *__restrict__ rowcut, int packed) {
    __shared__ int sout[8][4];
    __shared__ unsigned su[8][256];  // a packed histogram, unpacked
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lw = threadIdx.x >> 5;
    const int lane = lane_id();
    for (int64_t li = w; li < nsel; li += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t j = sel[li];
        if (done[j]) continue;
        const int r = rem[j];
        const unsigned *hj = hist + li * 256;
        if (packed) {
            for (int i = lane; i < 128; i += 32) {
                const unsigned w2 = hist[li * 128 + i];
                su[lw][i] = w2 & 0xffffu;
                su[lw][i + 128] = w2 >> 16;
            }
            __syncwarp();
            hj = su[lw];
        }
        if (pass < 4) find_digit<true>(hj, r, sout[lw]);
        else find_digit<false>(hj, r, sout[lw]);
        __syncwarp();
        if (lane == 0) {
            const int d = sout[lw][0], before = sout[lw][1], eq = sout[lw][2];
            const int nrem = r - before;
            if (pass < 4) {
                const int shift = 24 - 8 * pass;
                vprefix[j] |= (uint32_t)d << shift;
                rem[j] = nrem;
                if (pass == 3 && nrem == eq) {  // every entry equal to the cut is kept
                    done[j] = 1;
                    rowcut[j] = 0x7fffffff;
                }
            } else {
                const int shift = 24 - 8 * (pass - 4);
                rprefix[j] |= (uint32_t)d << shift;
                rem[j] = nrem;
                if (pass == 7) {
                    done[j] = 1;
                    rowcut[j] = (int32_t)rprefix[j];
                }
            }
        }
        __syncwarp();
    }
}
cudaError_t launch_dp_digit(int64_t nsel, const int32_t *sel, const unsigned *hist, int pass,
                            uint32_t *vprefix, uint32_t *rprefix, int32_t *rem, int32_t *done,
                            int32_t *rowcut, cudaStream_t s, int packed) {
    if (nsel <= 0) return cudaSuccess;
    int64_t b = (nsel * 32 + 255) / 256;
    if (b > g_sms * 32) b = g_sms * 32;
    ++g_launches;
    k_dp_digit<<<(int)b, 256, 0, s>>>(nsel, sel, hist, pass, vprefix, rprefix, rem, done, rowcut,
                                      packed);
    return cudaGetLastError();
}

// flags for the select-column list: flag[j] = (mode[j] == 1)
__global__ void k_dp_selflag(int64_t ncols, const int8_t *__restrict__ mode, int64_t *__restrict__ flag) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < ncols;
         j += (int64_t)gridDim.x * blockDim.x)
        flag[j] = mode[j] == 1 ? 1 : 0;
}
__global__ void k_dp_selscatter(int64_t ncols, const int8_t *__restrict__ mode,
                                const int64_t *__restrict__ pos, int32_t *__restrict__ sel) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < ncols;
         j += (int64_t)gridDim.x * blockDim.x)
        if (mode[j] == 1) sel[pos[j]] = (int32_t)j;
}
cudaError_t launch_dp_sellist(int64_t ncols, const int8_t *mode, int64_t *flag, int64_t *pos,
                              int32_t *sel, void *tmp, cudaStream_t s) {
    if (ncols <= 0) return cudaSuccess;
    int64_t b = (ncols + 255) / 256;
    if (b > g_sms * 16) b = g_sms * 16;
    ++g_launches;
    k_dp_selflag<<<(int)b, 256, 0, s>>>(ncols, mode, flag);
    cudaError_t e = launch_scan_i64(flag, pos, ncols, tmp, s);
    if (e != cudaSuccess) return e;
    ++g_launches;
    k_dp_selscatter<<<(int)b, 256, 0, s>>>(ncols, mode, pos, sel);
    return cudaGetLastError();
}
__global__ void k_dp_undone(int64_t nsel, const int32_t *__restrict__ sel,
                            const int32_t *__restrict__ done, unsigned long long *cnt) {
    unsigned long long c = 0;
    for (int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; li < nsel;
         li += (int64_t)gridDim.x * blockDim.x)
        c += done[sel[li]] ? 0 : 1;
    c = warp_sum(c);
    if (lane_id() == 0 && c) atomicAdd(cnt, c);
}
cudaError_t launch_dp_undone(int64_t nsel, const int32_t *sel, const int32_t *done,
                             unsigned long long *cnt, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess || nsel <= 0) return e;
    ++g_launches;
    k_dp_undone<<<(int)std::min<int64_t>((nsel + 255) / 256, g_sms * 4), 256, 0, s>>>(nsel, sel, done,
                                                                                  cnt);
    return cudaGetLastError();
}

__device__ __forceinline__ bool dp_keep(int8_t md, float v, uint32_t grow, double theta, uint32_t t,
                                        int32_t rowcut) {
    if (md == 0) return (double)v >= theta;
    if (md == 2) return true;
    if (md == 1) {
        const uint32_t b = __float_as_uint(v);
        return b > t || (b == t && (int32_t)grow <= rowcut);
    }
    return false;
}

// local sums over the kept set: count, sum v, max v, sum v^2, sum v^r.  A warp per column,
// 4 x 32 entries per trip with the loads issued first (rows only for select columns, whose
// cut has a row tie-break)
constexpr int kDPU = 4;
__global__ void __launch_bounds__(kDP) k_dp_keepstats(int64_t ncols, const int64_t *__restrict__ cp,
                                                      const int32_t *__restrict__ rows,
                                                      const float *__restrict__ vals, int64_t row0,
                                                      const int8_t *__restrict__ mode,
                                                      const uint32_t *__restrict__ vprefix,
                                                      const int32_t *__restrict__ rowcut,
                                                      PruneParams pp, int64_t *__restrict__ kcnt,
                                                      double *__restrict__ sums /*[4][ncols]*/,
                                                      const int64_t *__restrict__ ccnt) {
    const int lane = lane_id();
    for (int64_t j = dp_warp0(); j < ncols; j += dp_wstride()) {
        const int64_t a = cp[j], b = ccnt ? a + ccnt[j] : cp[j + 1];
        const int8_t md = mode[j];
        const uint32_t t = vprefix[j];
        const int32_t rc = rowcut[j];
        int64_t c = 0;
        double sv = 0, mx = 0, sq = 0, sr = 0;
        for (int64_t c0 = a; c0 < b; c0 += 32 * kDPU) {
            float v[kDPU];
            int r[kDPU];
#pragma unroll
            for (int u = 0; u < kDPU; u++) {
                const int64_t i = c0 + u * 32 + lane;
                v[u] = i < b ? vals[i] : -1.f;
                r[u] = (md == 1 && i < b) ? rows[i] : 0;
            }
#pragma unroll
            for (int u = 0; u < kDPU; u++) {
                if (v[u] >= 0.f && dp_keep(md, v[u], (uint32_t)(row0 + r[u]), pp.theta, t, rc)) {
                    const double d = (double)v[u];
                    c++;
                    sv += d;
                    mx = d > mx ? d : mx;
                    sq += d * d;
                    sr += pow_r(d, pp);
                }
            }
        }
        c = warp_sum(c);
        sv = warp_sum(sv);
        mx = warp_max(mx);
        sq = warp_sum(sq);
        sr = warp_sum(sr);
        if (lane == 0) {
            kcnt[j] = c;
            sums[j] = sv;
            sums[ncols + j] = mx;
            sums[2 * ncols + j] = sq;
            sums[3 * ncols + j] = sr;
        }
    }
}
cudaError_t launch_dp_keepstats(int64_t ncols, const int64_t *cp, const int32_t *rows,
                                const float *vals, int64_t row0, const int8_t *mode,
                                const uint32_t *vprefix, const int32_t *rowcut, const PruneParams &pp,
                                int64_t *kcnt, double *sums, int grid, cudaStream_t s,
                                const int64_t *ccnt) {
    if (ncols <= 0) return cudaSuccess;
    (void)grid;
    ++g_launches;
    k_dp_keepstats<<<dp_grid(ncols), kDP, 0, s>>>(ncols, cp, rows, vals, row0, mode, vprefix, rowcut,
                                                   pp, kcnt, sums, ccnt);
    return cudaGetLastError();
}

// Write the kept entries of every local column (row order preserved, ballot compaction)
// with a' = v^r / sum_global v^r (one reciprocal per column); chaos_j = K (max w - sum w^2)
// from the global sums (sums = [sv][mx][sq][sr], all-reduced; K = global kept count).
__global__ void __launch_bounds__(kDP) k_dp_write(int64_t ncols, const int64_t *__restrict__ cp,
                                                  const int32_t *__restrict__ rows,
                                                  const float *__restrict__ vals, int64_t row0,
                                                  const int8_t *__restrict__ mode,
                                                  const uint32_t *__restrict__ vprefix,
                                                  const int32_t *__restrict__ rowcut, PruneParams pp,
                                                  const double *__restrict__ gsums,
                                                  const int64_t *__restrict__ gkcnt,
                                                  const int64_t *__restrict__ soff,
                                                  int32_t *__restrict__ srow, float *__restrict__ sval,
                                                  int64_t *__restrict__ scnt, float *__restrict__ chaos,
                                                  float *chaos_max, const int64_t *__restrict__ ccnt) {
    const int lane = lane_id();
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t j = dp_warp0(); j < ncols; j += dp_wstride()) {
        const int64_t a = cp[j], b = ccnt ? a + ccnt[j] : cp[j + 1];
        const int8_t md = mode[j];
        const uint32_t t = vprefix[j];
        const int32_t rc = rowcut[j];
        const double inv = 1.0 / gsums[3 * ncols + j];
        const int64_t dst = soff[j];
        int64_t kept = 0;
        for (int64_t c0 = a; c0 < b; c0 += 32 * kDPU) {
            float v[kDPU];
            int r[kDPU];
#pragma unroll
            for (int u = 0; u < kDPU; u++) {
                const int64_t i = c0 + u * 32 + lane;
                v[u] = i < b ? vals[i] : -1.f;
                r[u] = i < b ? rows[i] : 0;
            }
#pragma unroll
            for (int u = 0; u < kDPU; u++) {
                const bool f = v[u] >= 0.f && dp_keep(md, v[u], (uint32_t)(row0 + r[u]), pp.theta, t, rc);
                const unsigned bal = __ballot_sync(0xffffffffu, f);
                if (f) {
                    const int64_t pos = dst + kept + __popc(bal & lt);
                    srow[pos] = r[u];
                    sval[pos] = (float)(pow_r((double)v[u], pp) * inv);
                }
                kept += __popc(bal);
            }
        }
        if (lane == 0) {
            scnt[j] = kept;
            const double sv = gsums[j], mx = gsums[ncols + j], sq = gsums[2 * ncols + j];
            const int64_t K = gkcnt[j];
            const float ch = K > 0 ? (float)((double)K * (mx / sv - sq / (sv * sv))) : 0.0f;
            if (chaos) chaos[j] = ch;
            atomic_max_nonneg_float(chaos_max, ch);
        }
    }
}
cudaError_t launch_dp_write(int64_t ncols, const int64_t *cp, const int32_t *rows, const float *vals,
                            int64_t row0, const int8_t *mode, const uint32_t *vprefix,
                            const int32_t *rowcut, const PruneParams &pp, const double *gsums,
                            const int64_t *gkcnt, const int64_t *soff, int32_t *srow, float *sval,
                            int64_t *scnt, float *chaos, float *chaos_max, int grid, cudaStream_t s,
                            const int64_t *ccnt) {
    if (ncols <= 0) return cudaSuccess;
    (void)grid;
    ++g_launches;
    k_dp_write<<<dp_grid(ncols), kDP, 0, s>>>(ncols, cp, rows, vals, row0, mode, vprefix, rowcut, pp,
                                               gsums, gkcnt, soff, srow, sval, scnt, chaos, chaos_max,
                                               ccnt);
    return cudaGetLastError();
}

}  // namespace mclx
