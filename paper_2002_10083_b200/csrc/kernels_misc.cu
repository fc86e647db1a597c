// kernels_misc.cu -- the non-SpGEMM kernels of the path:
//   flop count, binning, scans / reductions, the
//   standalone prune-inflate pass (Q1-Q9), assembly of the pruned CSC,
//   Cohen's estimator, Alg. 1 line 1 preprocessing and the
//   connected components of Alg. 1 line 6.
#include "kernels.h"

namespace mclx {

int64_t g_launches = 0;
int g_sms = 148;  // SMs of the context's device (mcl_ctx_create sets it); caps grid sizes

// ------------------------------------------------------------------ flops
// f_j = sum_{k in inds(B_*j)} nnz(A_*k).  One warp per column.
__global__ void k_flops(int64_t ncols, const int64_t *__restrict__ acp,
                        const int64_t *__restrict__ bcp, const int32_t *__restrict__ brow,
                        int64_t cb, int64_t *__restrict__ f) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = lane_id();
    for (int64_t col = w; col < ncols; col += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t q0 = bcp[cb + col], q1 = bcp[cb + col + 1];
        int64_t s = 0;
        for (int64_t q = q0 + lane; q < q1; q += 32) {
            const int k = __ldg(brow + q);
            s += __ldg(acp + k + 1) - __ldg(acp + k);
        }
        s = warp_sum(s);
        if (lane == 0) f[col] = s;
    }
}

cudaError_t launch_flops(int64_t ncols, const int64_t *acp, const int64_t *bcp,
                         const int32_t *brow, int64_t cb, int64_t *f, cudaStream_t s) {
    if (ncols <= 0) return cudaSuccess;
    int64_t blocks = (ncols * 32 + 255) / 256;
    if (blocks > g_sms * 64) blocks = g_sms * 64;
    ++g_launches;
    k_flops<<<(int)blocks, 256, 0, s>>>(ncols, acp, bcp, brow, cb, f);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ (row, value) pairs of A
// 16-byte loads of 4 rows + 4 values, two 16-byte stores of 4 pairs (row / val aligned)
__global__ void k_pack_pairs4(int64_t nnz, const int4 *__restrict__ row4,
                              const float4 *__restrict__ val4, const int32_t *__restrict__ row,
                              const float *__restrict__ val, int4 *__restrict__ out) {
    const int64_t n4 = nnz >> 2;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int4 r = __ldg(row4 + i);
        const float4 v = __ldg(val4 + i);
        out[2 * i] = make_int4(r.x, __float_as_int(v.x), r.y, __float_as_int(v.y));
        out[2 * i + 1] = make_int4(r.z, __float_as_int(v.z), r.w, __float_as_int(v.w));
    }
    if (blockIdx.x == 0 && threadIdx.x < (nnz & 3)) {
        const int64_t q = (n4 << 2) + threadIdx.x;
        reinterpret_cast<int2 *>(out)[q] = make_int2(row[q], __float_as_int(val[q]));
    }
}
__global__ void k_pack_pairs1(int64_t nnz, const int32_t *__restrict__ row,
                              const float *__restrict__ val, int2 *__restrict__ out) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nnz;
         q += (int64_t)gridDim.x * blockDim.x)
        out[q] = make_int2(row[q], __float_as_int(val[q]));
}

cudaError_t launch_pack_pairs(int64_t nnz, const int32_t *row, const float *val, int2 *apair,
                              cudaStream_t s) {
    if (nnz <= 0) return cudaSuccess;
    int64_t blocks = ((nnz >> 2) + 255) / 256;
    if (blocks > g_sms * 16) blocks = g_sms * 16;
    if (blocks < 1) blocks = 1;
    ++g_launches;
    if ((((uintptr_t)row | (uintptr_t)val | (uintptr_t)apair) & 15) == 0)
        k_pack_pairs4<<<(int)blocks, 256, 0, s>>>(nnz, reinterpret_cast<const int4 *>(row),
                                                  reinterpret_cast<const float4 *>(val), row, val,
                                                  reinterpret_cast<int4 *>(apair));
    else
        k_pack_pairs1<<<(int)blocks, 256, 0, s>>>(nnz, row, val, apair);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ phase planner helpers
// bytes[j] (+)= a * x[j] + b for an int64 x (accumulate = add to bytes, else overwrite)
__global__ void k_affine_i64(int64_t n, const int64_t *x, int64_t a, int64_t b, int64_t *bytes,
                             int accumulate) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x)
        bytes[j] = (accumulate ? bytes[j] : 0) + a * x[j] + b;
}
// bytes[j] += ceil(a * est[j]) + b for a Cohen estimate est (fp32)
__global__ void k_affine_est(int64_t n, const float *est, double a, int64_t b, int64_t *bytes) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x)
        bytes[j] += (int64_t)ceil(a * (double)est[j]) + b;
}
// cut[k-1] = first j with prefix[j] >= k * total / h, k = 1 .. h-1 (prefix: exclusive scan,
// [n+1]); the batches [cut[k-1], cut[k]) then hold near-equal shares of the bytes
__global__ void k_phase_cuts(const int64_t *prefix, int64_t n, int h, int64_t *cut) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x + 1;
    if (k >= h) return;
    const int64_t total = prefix[n];
    const int64_t want = (int64_t)((__int128)total * k / h);
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (prefix[mid] < want) lo = mid + 1;
        else hi = mid;
    }
    cut[k - 1] = lo;
}

cudaError_t launch_affine_i64(int64_t n, const int64_t *x, int64_t a, int64_t b, int64_t *bytes,
                              bool accumulate, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    int64_t blocks = (n + 255) / 256;
    if (blocks > g_sms * 16) blocks = g_sms * 16;
    ++g_launches;
    k_affine_i64<<<(int)blocks, 256, 0, s>>>(n, x, a, b, bytes, accumulate ? 1 : 0);
    return cudaGetLastError();
}
cudaError_t launch_affine_est(int64_t n, const float *est, double a, int64_t b, int64_t *bytes,
                              cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    int64_t blocks = (n + 255) / 256;
    if (blocks > g_sms * 16) blocks = g_sms * 16;
    ++g_launches;
    k_affine_est<<<(int)blocks, 256, 0, s>>>(n, est, a, b, bytes);
    return cudaGetLastError();
}
cudaError_t launch_phase_cuts(const int64_t *prefix, int64_t n, int h, int64_t *cut, cudaStream_t s) {
    if (h <= 1) return cudaSuccess;
    ++g_launches;
    k_phase_cuts<<<(h + 255) / 256, 256, 0, s>>>(prefix, n, h, cut);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ gathers for host plans
// dst[i] = src[idx[i]] (the split path's part counts / the global bin's flops per listed
// column: read back instead of whole n-length arrays)
template <typename T>
__global__ void k_gather(int64_t n, const int32_t *__restrict__ idx, const T *__restrict__ src,
                         T *__restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[idx[i]];
}
cudaError_t launch_gather_i32(int64_t n, const int32_t *idx, const int32_t *src, int32_t *dst,
                              cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    int64_t b = (n + 255) / 256;
    if (b > g_sms * 16) b = g_sms * 16;
    ++g_launches;
    k_gather<int32_t><<<(int)b, 256, 0, s>>>(n, idx, src, dst);
    return cudaGetLastError();
}
cudaError_t launch_gather_i64(int64_t n, const int32_t *idx, const int64_t *src, int64_t *dst,
                              cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    int64_t b = (n + 255) / 256;
    if (b > g_sms * 16) b = g_sms * 16;
    ++g_launches;
    k_gather<int64_t><<<(int)b, 256, 0, s>>>(n, idx, src, dst);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ CSC validation
// MCLX_VALIDATE=1 (include/mclx.h MCL_ERR_FORMAT): the CSC invariants of the header --
// col_ptr[0] = 0, non-decreasing, col_ptr[n] = nnz; rows in [0, nrows) and strictly
// increasing inside each column; values finite and >= 0 (negative -> rejection,
// S:70; an unpruned product entry may underflow to 0, Q13).  One warp per
// column; violations OR bits into *flag (1 col_ptr, 2 row range, 4 row order, 8 value).
__global__ void k_validate_csc(int64_t ncols, int64_t nrows, int64_t nnz,
                               const int64_t *__restrict__ cp, const int32_t *__restrict__ row,
                               const float *__restrict__ val, int *flag) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = lane_id();
    if (w == 0 && lane == 0 && (cp[0] != 0 || cp[ncols] != nnz)) atomicOr(flag, 1);
    for (int64_t col = w; col < ncols; col += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t q0 = cp[col], q1 = cp[col + 1];
        int bad = 0;
        if (q1 < q0 || q0 < 0 || q1 > nnz) {
            bad = 1;
        } else {
            for (int64_t q = q0 + lane; q < q1; q += 32) {
                const int r = row[q];
                if (r < 0 || r >= nrows) bad |= 2;
                if (q > q0 && row[q - 1] >= r) bad |= 4;
                const float v = val[q];
                if (!(v >= 0.f) || !isfinite(v)) bad |= 8;  // NaN, inf or negative
            }
        }
        bad = __reduce_or_sync(0xffffffffu, bad);
        if (lane == 0 && bad) atomicOr(flag, bad);
    }
}

cudaError_t launch_validate_csc(int64_t ncols, int64_t nrows, int64_t nnz, const int64_t *cp,
                                const int32_t *row, const float *val, int *flag, cudaStream_t s) {
    int64_t blocks = (std::max<int64_t>(ncols, 1) * 32 + 255) / 256;
    if (blocks > g_sms * 32) blocks = g_sms * 32;
    ++g_launches;
    k_validate_csc<<<(int)blocks, 256, 0, s>>>(ncols, nrows, nnz, cp, row, val, flag);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ row-range index of A
// rowpart[k][i] = lower_bound(rows of A_*k, ceil(i*m/32)) - col_ptr[k], i = 0..32.  One
// warp per column; lane i binary-searches boundary i (independent searches).
// NP-way row-partition index (NP = 32, or kFineParts = 128 for split parts): P[k][i] =
// first position of A_*k with row >= ceil(i m / NP); boundary 4i of the 128-way index
// equals boundary i of the 32-way one.
template <int NP>
__global__ void k_rowpart(int64_t ncols, const int64_t *__restrict__ cp,
                          const int32_t *__restrict__ row, int64_t m, int *__restrict__ P) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = lane_id();
    for (int64_t k = w; k < ncols; k += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t a = cp[k], b = cp[k + 1];
    #pragma unroll
        for (int q = 0; q < NP / 32; q++) {
            const int part = lane + 32 * q;
            const int64_t bound = ((int64_t)part * m + NP - 1) / NP;
            int64_t lo = a, hi = b;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if ((int64_t)__ldg(row + mid) < bound) lo = mid + 1;
                else hi = mid;
            }
            P[k * (NP + 1) + part] = (int)(lo - a);
        }
        if (lane == 0) P[k * (NP + 1) + NP] = (int)(b - a);
    }
}
cudaError_t launch_rowpart(int64_t ncols, const int64_t *cp, const int32_t *row, int64_t m,
                           int *rowpart, cudaStream_t s, int nparts) {
    if (ncols <= 0) return cudaSuccess;
    int64_t blocks = (ncols * 32 + 255) / 256;
    if (blocks > g_sms * 32) blocks = g_sms * 32;
    ++g_launches;
    if (nparts == kFineParts) k_rowpart<kFineParts><<<(int)blocks, 256, 0, s>>>(ncols, cp, row, m, rowpart);
    else k_rowpart<32><<<(int)blocks, 256, 0, s>>>(ncols, cp, row, m, rowpart);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ reductions
__global__ void k_reduce_i64(const int64_t *__restrict__ x, int64_t n, unsigned long long *out) {
    __shared__ int64_t sh[8];
    int64_t s = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        s += x[i];
    s = block_sum<256, int64_t>(s, sh);
    if (threadIdx.x == 0) atomicAdd(out, (unsigned long long)s);
}
__global__ void k_reduce_f32(const float *__restrict__ x, int64_t n, double *out) {
    __shared__ double sh[8];
    double s = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        s += (double)x[i];
    s = block_sum<256, double>(s, sh);
    if (threadIdx.x == 0) atomicAdd(out, s);
}
static int red_grid(int64_t n) {
    int64_t b = (n + 255) / 256;
    if (b > g_sms * 4) b = g_sms * 4;
    return b < 1 ? 1 : (int)b;
}
cudaError_t launch_reduce_i64(const int64_t *x, int64_t n, unsigned long long *out, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    ++g_launches;
    k_reduce_i64<<<red_grid(n), 256, 0, s>>>(x, n, out);
    return cudaGetLastError();
}
cudaError_t launch_reduce_f32(const float *x, int64_t n, double *out, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), s);
    if (e != cudaSuccess) return e;
    ++g_launches;
    k_reduce_f32<<<red_grid(n), 256, 0, s>>>(x, n, out);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ exclusive scan (int64)
// Reduce-then-scan: tiles of 4096 elements (1024 threads x 4), tile sums scanned
// recursively, then each tile re-scanned with its offset.
constexpr int kScanNT = 1024, kScanIPT = 4, kScanTile = kScanNT * kScanIPT;

__device__ __forceinline__ int64_t block_excl_scan64(int64_t v, int64_t *sh, int64_t &total) {
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane_id() >= o) x += y;
    }
    __syncthreads();
    if (lane_id() == 31) sh[warp_id()] = x;
    __syncthreads();
    if (warp_id() == 0) {
        int64_t w = sh[lane_id()];
        int64_t z = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(0xffffffffu, z, o);
            if (lane_id() >= o) z += y;
        }
        sh[lane_id()] = z - w;
        if (lane_id() == 31) sh[32] = z;
    }
    __syncthreads();
    total = sh[32];
    return sh[warp_id()] + x - v;
}

__global__ void __launch_bounds__(kScanNT) k_scan_tiles(const int64_t *__restrict__ in, int64_t n,
                                                        int64_t *__restrict__ tile_sums) {
    __shared__ int64_t sh[33];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanIPT;
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanIPT; i++)
        if (base + i < n) s += in[base + i];
    int64_t tot;
    block_excl_scan64(s, sh, tot);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanNT) k_scan_apply(const int64_t *__restrict__ in, int64_t n,
                                                        const int64_t *__restrict__ tile_off,
                                                        int64_t *__restrict__ out) {
    __shared__ int64_t sh[33];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanIPT;
    int64_t v[kScanIPT];
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanIPT; i++) {
        v[i] = (base + i < n) ? in[base + i] : 0;
        s += v[i];
    }
    int64_t tot;
    int64_t off = block_excl_scan64(s, sh, tot) + tile_off[blockIdx.x];
#pragma unroll
    for (int i = 0; i < kScanIPT; i++) {
        if (base + i < n) out[base + i] = off;
        off += v[i];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == kScanNT - 1) out[n] = off;
}

size_t scan_tmp_bytes(int64_t n) {
    size_t b = 0;
    int64_t t = (n + kScanTile - 1) / kScanTile;
    while (t > 1) {
        b += (size_t)(t + 1) * 2 * sizeof(int64_t);
        t = (t + kScanTile - 1) / kScanTile;
    }
    return b + 64;
}

cudaError_t launch_scan_i64(const int64_t *in, int64_t *out, int64_t n, void *tmp, cudaStream_t s) {
    if (n <= 0) return cudaMemsetAsync(out, 0, sizeof(int64_t), s);
    const int64_t tiles = (n + kScanTile - 1) / kScanTile;
    if (tiles == 1) {
        int64_t *off = (int64_t *)tmp;
        cudaError_t e = cudaMemsetAsync(off, 0, sizeof(int64_t), s);
        if (e != cudaSuccess) return e;
        ++g_launches;
        k_scan_apply<<<1, kScanNT, 0, s>>>(in, n, off, out);
        return cudaGetLastError();
    }
    int64_t *sums = (int64_t *)tmp;
    int64_t *offs = sums + tiles + 1;
    ++g_launches;
    k_scan_tiles<<<(unsigned)tiles, kScanNT, 0, s>>>(in, n, sums);
    cudaError_t e = launch_scan_i64(sums, offs, tiles, (void *)(offs + tiles + 1), s);
    if (e != cudaSuccess) return e;
    ++g_launches;
    k_scan_apply<<<(unsigned)tiles, kScanNT, 0, s>>>(in, n, offs, out);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ binning
// Size bound of output column j: ub = min(f_j, m) (exact upper bound); need = the
// exact symbolic size when known, else min(ub, alpha * Cohen estimate + 16), else ub.
// Bin = smallest shared-memory table with need <= cap/2; columns whose entries sum
// more than kFp64Terms products per output entry go to the fp64 global bin (T).
__global__ void k_classify(ClassifyArgs c) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t col = c.cols ? c.cols[i] : i;
        const int64_t f = c.flops[col];
        if (f == 0) {
            if (c.colbin) c.colbin[col] = -1;
            continue;
        }
        const int64_t ub = f < c.m ? f : c.m;
        int64_t need = ub;
        if (c.exact) {
            need = c.exact[col];
        } else if (c.est) {
            double e = ceil((double)c.alpha * (double)c.est[col]) + 16.0;
            if (e < (double)need) need = (int64_t)e;
        }
        const int64_t nb = c.bcp[c.cb + col + 1] - c.bcp[c.cb + col];
        if (c.esc_max > 0 && c.force_bin < 0 && f <= c.esc_max) {
            // low compression factor: expand-sort-compress
            const double nest = c.exact ? (double)c.exact[col] : c.est ? (double)c.est[col] : (double)ub;
            if ((double)f < c.esc_cf * (nest > 1.0 ? nest : 1.0)) {
                c.esc_list[atomicAdd(c.esc_count, 1)] = (int32_t)col;
                if (c.colbin) c.colbin[col] = -1;
                atomicAdd(c.esc_flops, (unsigned long long)f);
                continue;
            }
        }
        int b = 0;
        while (b < kNumBins && (double)need > c.max_load * bin_cap(b)) b++;
        if (nb > c.fp64_terms) b = kNumBins;
        if (c.force_bin > b && c.force_bin <= kNumBins) b = c.force_bin;
        if ((b == kNumBins || need > c.split_min) && c.split_max > 0 && need <= c.split_max &&
            c.force_bin < 0) {
            // row-range split, sized by the virtual part count P (a power of two, parts of
            // ~kPartNeed distinct rows); P > 32 runs 32 parts with bigger tables
            int P = 2;
            while ((int64_t)P * c.split_part_need < need) P <<= 1;
            // long sums (T): only the dense fp64 variant accumulates in fp64
            if (nb > c.fp64_terms) P = (P < 128 ? 128 : P) | kSplitFp64;
            else if (P > c.dense_min_P) P |= kSplitDense;
            else if (c.split_big && P >= 4 && P <= 32) P = (P >> 1) | kSplitBig;
            // private-slice parts give each of 8 warps 1/(8P) of every segment: below
            // kShortSegment / 2 rows on average the lanes idle, so use the shared table
            else if (f < (int64_t)(kShortSegment / 2) * nb * 8 * P) P |= kSplitShared;
            c.split_P[col] = P;
            c.split_list[atomicAdd(c.split_count, 1)] = (int32_t)col;
            if (c.colbin) c.colbin[col] = -1;
            atomicAdd(&c.bin_flops[kNumBins], (unsigned long long)f);
            atomicAdd(&c.bin_nnzb[kNumBins], (unsigned long long)nb);
            continue;
        }
        // family: short average segments go to the CTA-shared atomic table
        const bool shortseg = f < (int64_t)kShortSegment * nb;
        const int fam = c.force_family >= 0 ? c.force_family : (shortseg ? 1 : 0);
        const int bb = fam * kFamily + b;
        const int pos = atomicAdd(&c.bin_count[bb], 1);
        c.lists[(int64_t)bb * c.list_stride + pos] = (int32_t)col;
        if (c.colbin) c.colbin[col] = bb;
        atomicAdd(&c.bin_flops[bb], (unsigned long long)f);
        atomicAdd(&c.bin_nnzb[bb], (unsigned long long)nb);
        if (b == kNumBins) {
            int64_t cap = 64 * (kGlobalThreads / 32);
            while ((double)need > c.max_load * cap) cap <<= 1;
            c.gcap_col[col] = (int32_t)cap;
        }
    }
}

cudaError_t launch_classify(const ClassifyArgs &c, cudaStream_t s) {
    if (c.n <= 0) return cudaSuccess;
    int64_t b = (c.n + 255) / 256;
    if (b > g_sms * 16) b = g_sms * 16;
    ++g_launches;
    k_classify<<<(int)b, 256, 0, s>>>(c);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ split columns
__global__ void k_split_items(int nsplit, const int32_t *split_list, const int32_t *split_P,
                              const int64_t *ioff, int32_t *item_col, int32_t *item_pr) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nsplit; s += gridDim.x * blockDim.x) {
        const int32_t col = split_list[s];
        const int P = split_parts(split_P[col]);
        const int step = 32 / P;
        const int64_t i0 = ioff[s];
        for (int p = 0; p < P; p++) {
            item_col[i0 + p] = col;
            item_pr[i0 + p] = (p * step) | ((p + 1) * step) << 8;
        }
    }
}
cudaError_t launch_split_items(int nsplit, const int32_t *split_list, const int32_t *split_P,
                               const int64_t *ioff, int32_t *item_col, int32_t *item_pr,
                               cudaStream_t s) {
    if (nsplit <= 0) return cudaSuccess;
    ++g_launches;
    k_split_items<<<(nsplit + 255) / 256, 256, 0, s>>>(nsplit, split_list, split_P, ioff, item_col,
                                                      item_pr);
    return cudaGetLastError();
}

__global__ void k_split_stitch(int nc, const int64_t *ioff, int64_t item0, const int32_t *item_col,
                               const int64_t *sioff, const int *col_flag, int64_t *ccp,
                               int32_t *colmap, const int64_t *stg_nnz, const int64_t *stg_m,
                               const double *stg_s, int64_t *fnnz, int64_t *fm, double *fs) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c <= nc; c += gridDim.x * blockDim.x) {
        const int64_t i = ioff[c] - item0;  // first item of chunk column c (or the end)
        ccp[c] = sioff[i];
        if (c < nc) {
            const int32_t col = item_col[i];
            colmap[c] = col_flag[col] ? -1 : col;
            if (stg_nnz) {  // candidates: the column's statistics are the sums over its parts
                const int64_t i1 = ioff[c + 1] - item0;
                int64_t n = 0, m = 0;
                double sm = 0.0;
                for (int64_t q = i; q < i1; q++) {
                    n += stg_nnz[q];
                    m += stg_m[q];
                    sm += stg_s[q];
                }
                fnnz[c] = n;
                fm[c] = m;
                fs[c] = sm;
            }
        }
    }
}
cudaError_t launch_split_stitch(int nc, const int64_t *ioff, int64_t item0, const int32_t *item_col,
                                const int64_t *sioff, const int *col_flag, int64_t *ccp,
                                int32_t *colmap, const int64_t *stg_nnz, const int64_t *stg_m,
                                const double *stg_s, int64_t *fnnz, int64_t *fm, double *fs,
                                cudaStream_t s) {
    ++g_launches;
    k_split_stitch<<<(nc + 256) / 256, 256, 0, s>>>(nc, ioff, item0, item_col, sioff, col_flag, ccp,
                                                   colmap, stg_nnz, stg_m, stg_s, fnnz, fm, fs);
    return cudaGetLastError();
}

// warp per item: copy its staged (sorted) entries to the stitched column
__global__ void k_split_gather(int64_t nitems, const int64_t *stg_cnt, const int64_t *stg_off,
                               const int32_t *stg_row, const float *stg_val, const int64_t *sioff,
                               int32_t *crow, float *cval) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w0; i < nitems; i += nw) {
        const int64_t n = stg_cnt[i];
        const int64_t src = stg_off[i], dst = sioff[i];
        for (int64_t e = lane; e < n; e += 32) {
            crow[dst + e] = stg_row[src + e];
            cval[dst + e] = stg_val[src + e];
        }
    }
}
cudaError_t launch_split_gather(int64_t nitems, const int64_t *stg_cnt, const int64_t *stg_off,
                                const int32_t *stg_row, const float *stg_val, const int64_t *sioff,
                                int32_t *crow, float *cval, cudaStream_t s) {
    if (nitems <= 0) return cudaSuccess;
    int64_t b = (nitems + 7) / 8;
    if (b > g_sms * 16) b = g_sms * 16;
    ++g_launches;
    k_split_gather<<<(int)b, 256, 0, s>>>(nitems, stg_cnt, stg_off, stg_row, stg_val, sioff, crow,
                                          cval);
    return cudaGetLastError();
}

__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
    h ^= h >> 16;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    h *= 0xc2b2ae35u;
    h ^= h >> 16;
    return h;
}

// warp per column: key[j] = min_{i in rows(B_*j)} fmix32(i)
__global__ void k_minhash_key(int64_t n, const int64_t *bcp, const int32_t *brow, int64_t cb,
                              uint32_t *key) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = w0; j < n; j += nw) {
        const int64_t q0 = bcp[cb + j], q1 = bcp[cb + j + 1];
        uint32_t k = 0xffffffffu;
        for (int64_t q = q0 + lane; q < q1; q += 32) {
            const uint32_t h = fmix32((uint32_t)__ldg(brow + q));
            k = h < k ? h : k;
        }
        k = __reduce_min_sync(0xffffffffu, k);
        if (lane == 0) key[j] = k;
    }
}

cudaError_t launch_minhash_key(int64_t n, const int64_t *bcp, const int32_t *brow, int64_t cb,
                               uint32_t *key, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    int64_t b = (n + 7) / 8;
    if (b > g_sms * 16) b = g_sms * 16;
    ++g_launches;
    k_minhash_key<<<(int)b, 256, 0, s>>>(n, bcp, brow, cb, key);
    return cudaGetLastError();
}

__device__ __forceinline__ int64_t order_bucket(int32_t bb, uint32_t key) {
    return ((int64_t)bb << kOrderBits) | (int64_t)(key >> (32 - kOrderBits));
}

__global__ void k_order_hist(int64_t n, const int32_t *cols, const int32_t *colbin,
                             const uint32_t *key, int64_t *hist) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t col = cols ? cols[i] : (int32_t)i;
        const int32_t bb = colbin[col];
        if (bb < 0) continue;
        atomicAdd(reinterpret_cast<unsigned long long *>(&hist[order_bucket(bb, key[col])]), 1ull);
    }
}

// offs: exclusive scan of hist (offs[b << kOrderBits] = start of bin b); hist is reused
// as the per-bucket cursor
__global__ void k_order_scatter(int64_t n, const int32_t *cols, const int32_t *colbin,
                                const uint32_t *key, const int64_t *offs, int64_t *cursor,
                                int32_t *lists, int64_t list_stride) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t col = cols ? cols[i] : (int32_t)i;
        const int32_t bb = colbin[col];
        if (bb < 0) continue;
        const int64_t bk = order_bucket(bb, key[col]);
        const int64_t pos = offs[bk] + (int64_t)atomicAdd(reinterpret_cast<unsigned long long *>(&cursor[bk]), 1ull);
        lists[(int64_t)bb * list_stride + (pos - offs[(int64_t)bb << kOrderBits])] = col;
    }
}

cudaError_t launch_order_lists(int64_t n, const int32_t *cols, const int32_t *colbin,
                               const uint32_t *key, int64_t *hist, int64_t *offs, void *scan_tmp,
                               int32_t *lists, int64_t list_stride, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int64_t nbk = (int64_t)kAllBins << kOrderBits;
    cudaError_t e = cudaMemsetAsync(hist, 0, sizeof(int64_t) * nbk, s);
    if (e != cudaSuccess) return e;
    int64_t b = (n + 255) / 256;
    if (b > g_sms * 16) b = g_sms * 16;
    ++g_launches;
    k_order_hist<<<(int)b, 256, 0, s>>>(n, cols, colbin, key, hist);
    if ((e = launch_scan_i64(hist, offs, nbk, scan_tmp, s)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(hist, 0, sizeof(int64_t) * nbk, s)) != cudaSuccess) return e;
    ++g_launches;
    k_order_scatter<<<(int)b, 256, 0, s>>>(n, cols, colbin, key, offs, hist, lists, list_stride);
    return cudaGetLastError();
}

__global__ void k_global_layout(int count, const int32_t *list, const int32_t *gcap_col,
                                int32_t *gcap, int64_t *gcap64) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        int32_t c = gcap_col[list[i]];
        gcap[i] = c;
        gcap64[i] = c;
    }
}
cudaError_t launch_global_layout(int count, const int32_t *list, const int32_t *gcap_col,
                                 int32_t *gcap, int64_t *gcap64, cudaStream_t s) {
    if (count <= 0) return cudaSuccess;
    ++g_launches;
    k_global_layout<<<(count + 255) / 256, 256, 0, s>>>(count, list, gcap_col, gcap, gcap64);
    return cudaGetLastError();
}

// staging capacity of a pruned column: min(max(S,R,1), min(f_j, m))
__global__ void k_kcap(int64_t ncols, const int64_t *f, int64_t m, int kmax, int64_t *kcap) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < ncols;
         j += (int64_t)gridDim.x * blockDim.x) {
        int64_t u = f[j] < m ? f[j] : m;
        kcap[j] = u < kmax ? u : kmax;
    }
}
cudaError_t launch_kcap(int64_t ncols, const int64_t *flops, int64_t m, int kmax, int64_t *kcap,
                        cudaStream_t s) {
    if (ncols <= 0) return cudaSuccess;
    ++g_launches;
    k_kcap<<<red_grid(ncols) * 4, 256, 0, s>>>(ncols, flops, m, kmax, kcap);
    return cudaGetLastError();
}

// staging capacity of a column of an unpruned CSC: min(kmax, nnz(C_*j))
__global__ void k_kcap_cp(int64_t ncols, const int64_t *cp, int kmax, int64_t *kcap) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < ncols;
         j += (int64_t)gridDim.x * blockDim.x) {
        int64_t u = cp[j + 1] - cp[j];
        kcap[j] = u < kmax ? u : kmax;
    }
}
cudaError_t launch_kcap_cp(int64_t ncols, const int64_t *cp, int kmax, int64_t *kcap, cudaStream_t s) {
    if (ncols <= 0) return cudaSuccess;
    ++g_launches;
    k_kcap_cp<<<red_grid(ncols) * 4, 256, 0, s>>>(ncols, cp, kmax, kcap);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ merge helpers
// col_ptr of list l inside the horizontal concatenation X = [P_0 | P_1 | ...]:
// out[j] = cp[j] + off for j in [0, n] (out is X.col_ptr + l*n).
__global__ void k_offset_colptr(int64_t n1, const int64_t *cp, int64_t off, int64_t *out) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n1;
         j += (int64_t)gridDim.x * blockDim.x)
        out[j] = cp[j] + off;
}
cudaError_t launch_offset_colptr(int64_t n1, const int64_t *cp, int64_t off, int64_t *out,
                                 cudaStream_t s) {
    if (n1 <= 0) return cudaSuccess;
    ++g_launches;
    k_offset_colptr<<<red_grid(n1) * 4, 256, 0, s>>>(n1, cp, off, out);
    return cudaGetLastError();
}
// E = [I; I; ...; I] (L*n x n): column j holds rows j, n+j, ..., (L-1)n+j with value 1,
// so that X * E = sum_l P_l (the merge of P:246 as a product).
__global__ void k_stack_identity(int64_t n, int L, int64_t *cp, int32_t *row, float *val) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= n;
         j += (int64_t)gridDim.x * blockDim.x) {
        cp[j] = (int64_t)L * j;
        if (j < n)
            for (int l = 0; l < L; l++) {
                row[(int64_t)L * j + l] = (int32_t)((int64_t)l * n + j);
                val[(int64_t)L * j + l] = 1.0f;
            }
    }
}
cudaError_t launch_stack_identity(int64_t n, int L, int64_t *cp, int32_t *row, float *val,
                                  cudaStream_t s) {
    ++g_launches;
    k_stack_identity<<<red_grid(n + 1) * 4, 256, 0, s>>>(n, L, cp, row, val);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ assembly
// Copy each column's cnt entries from its staging slot to the compact CSC.  Warp/column.
__global__ void k_copy_cols(int64_t ncols, const int64_t *__restrict__ cnt,
                            const int64_t *__restrict__ soff, const int32_t *__restrict__ srow,
                            const float *__restrict__ sval, const int64_t *__restrict__ cp,
                            int32_t *__restrict__ orow, float *__restrict__ oval) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = lane_id();
    for (int64_t col = w; col < ncols; col += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t n = cnt[col], src = soff[col], dst = cp[col];
        for (int64_t i = lane; i < n; i += 32) {
            orow[dst + i] = srow[src + i];
            oval[dst + i] = sval[src + i];
        }
    }
}
cudaError_t launch_copy_cols(int64_t ncols, const int64_t *cnt, const int64_t *soff,
                             const int32_t *srow, const float *sval, const int64_t *cp,
                             int32_t *orow, float *oval, cudaStream_t s) {
    if (ncols <= 0) return cudaSuccess;
    int64_t blocks = (ncols * 32 + 255) / 256;
    if (blocks > g_sms * 32) blocks = g_sms * 32;
    ++g_launches;
    k_copy_cols<<<(int)blocks, 256, 0, s>>>(ncols, cnt, soff, srow, sval, cp, orow, oval);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ standalone prune/inflate
// Alg. 1 lines 4-5 on an unpruned CSC column (rows already sorted): threshold stats,
// branch (Q5, Q7, Q8), exact top-K by radix select, renormalise + chaos (Q9), Hadamard
// power r and renormalise (Q1).  The kept entries are extracted in row
// order with a block scan, so the output stays sorted without a sort.
constexpr int kPruneNT = 256;
__global__ void __launch_bounds__(kPruneNT)
    k_prune(int64_t ncols, const int64_t *__restrict__ ccp, const int32_t *__restrict__ crow,
            const float *__restrict__ cval, const int64_t *__restrict__ soff,
            int32_t *__restrict__ srow, float *__restrict__ sval, int64_t *__restrict__ scnt,
            float *__restrict__ chaos_out, float *chaos_max, PruneParams pp,
            const int32_t *__restrict__ colmap, unsigned long long *out_count,
            const int64_t *__restrict__ fnnz, const int64_t *__restrict__ fm,
            const double *__restrict__ fs) {
    __shared__ unsigned hist[256];
    __shared__ int sint[4];
    __shared__ double sred[kPruneNT / 32];
    __shared__ int sscan[kPruneNT / 32];
    for (int64_t ci = blockIdx.x; ci < ncols; ci += gridDim.x) {
        // output column: colmap[ci] (split columns; -1 = skip), else ci
        const int64_t col = colmap ? (int64_t)colmap[ci] : ci;
        if (col < 0) continue;
        const int64_t base = ccp[ci];
        const int nnz = (int)(ccp[ci + 1] - base);
        if (fnnz)  // candidates of split parts + the whole column's statistics
            prune_column<kPruneNT>(crow + base, cval + base, nnz, col, soff, srow, sval, scnt,
                                   chaos_out, chaos_max, out_count, pp, hist, sint, sred, sscan,
                                   fnnz[ci], fm[ci], fs[ci]);
        else
            prune_column<kPruneNT>(crow + base, cval + base, nnz, col, soff, srow, sval, scnt,
                                   chaos_out, chaos_max, out_count, pp, hist, sint, sred, sscan);
    }
}

// Candidate mode (the fused 2D SUMMA, capi.cu): a stitched split column's candidates are cut
// back to its top-K (value desc, row asc) and written, rows ascending, to the column's staging
// slot; the column's statistics (nnz, m, s of all its entries) go to arrays indexed by column.
__global__ void __launch_bounds__(kPruneNT)
    k_cand_select(int64_t ncols, const int64_t *__restrict__ ccp, const int32_t *__restrict__ crow,
                  const float *__restrict__ cval, const int32_t *__restrict__ colmap, int K,
                  const int64_t *__restrict__ fnnz, const int64_t *__restrict__ fm,
                  const double *__restrict__ fs, const int64_t *__restrict__ soff,
                  int32_t *__restrict__ srow, float *__restrict__ sval, int64_t *__restrict__ scnt,
                  int64_t *__restrict__ onnz, int64_t *__restrict__ om, double *__restrict__ os,
                  unsigned long long *out_count) {
    __shared__ unsigned hist[256];
    __shared__ int sint[4];
    __shared__ int sscan[kPruneNT / 32];
    for (int64_t ci = blockIdx.x; ci < ncols; ci += gridDim.x) {
        const int64_t col = colmap[ci];
        if (col < 0) continue;
        const int64_t base = ccp[ci];
        const int n = (int)(ccp[ci + 1] - base);
        uint32_t t = 0;
        int rowcut = 0x7fffffff;
        if (n > K) radix_select_topk<kPruneNT, float>(crow + base, cval + base, n, K, t, rowcut, hist, sint);
        const int64_t dst = soff[col];
        int kept = 0;
        for (int c0 = 0; c0 < n; c0 += kPruneNT) {
            const int i = c0 + threadIdx.x;
            int f = 0, r = 0;
            float v = 0.f;
            if (i < n) {
                r = crow[base + i];
                v = cval[base + i];
                const uint32_t b = val_bits(v);
                f = n <= K || b > t || (b == t && r <= rowcut);
            }
            int tot;
            const int pos = block_excl_scan<kPruneNT>(f, sscan, tot);
            if (f) {
                srow[dst + kept + pos] = r;
                sval[dst + kept + pos] = v;
            }
            kept += tot;
        }
        if (threadIdx.x == 0) {
            scnt[col] = kept;
            onnz[col] = fnnz[ci];
            om[col] = fm[ci];
            os[col] = fs[ci];
            if (out_count) atomicAdd(out_count, (unsigned long long)kept);
        }
        __syncthreads();
    }
}

cudaError_t launch_cand_select(int64_t ncols, const int64_t *ccp, const int32_t *crow, const float *cval,
                               const int32_t *colmap, int K, const int64_t *fnnz, const int64_t *fm,
                               const double *fs, const int64_t *soff, int32_t *srow, float *sval,
                               int64_t *scnt, int64_t *onnz, int64_t *om, double *os,
                               unsigned long long *out_count, int grid, cudaStream_t s) {
    if (ncols <= 0) return cudaSuccess;
    ++g_launches;
    k_cand_select<<<grid, kPruneNT, 0, s>>>(ncols, ccp, crow, cval, colmap, K, fnnz, fm, fs, soff, srow,
                                            sval, scnt, onnz, om, os, out_count);
    return cudaGetLastError();
}

cudaError_t launch_prune(int64_t ncols, const int64_t *ccp, const int32_t *crow, const float *cval,
                         const int64_t *soff, int32_t *srow, float *sval, int64_t *scnt,
                         float *chaos, float *chaos_max, const PruneParams &pp, int grid,
                         cudaStream_t s, const int32_t *colmap, unsigned long long *out_count,
                         const int64_t *fnnz, const int64_t *fm, const double *fs) {
    if (ncols <= 0) return cudaSuccess;
    ++g_launches;
    k_prune<<<grid, kPruneNT, 0, s>>>(ncols, ccp, crow, cval, soff, srow, sval, scnt, chaos,
                                      chaos_max, pp, colmap, out_count, fnnz, fm, fs);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ Cohen estimator
// Philox-4x32-10 (Salmon et al., SC'11) -- 10 rounds of the 4x32 S-box with key bumps.
__device__ __forceinline__ uint4 philox4x32_10(uint4 x, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; r++) {
        const uint32_t lo0 = 0xD2511F53u * x.x, hi0 = __umulhi(0xD2511F53u, x.x);
        const uint32_t lo1 = 0xCD9E8D57u * x.z, hi1 = __umulhi(0xCD9E8D57u, x.z);
        x = make_uint4(hi1 ^ x.y ^ k.x, lo1, hi0 ^ x.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return x;
}

// Keys X[s][i] ~ Exp(lambda = 1): u = Philox(ctr=(i_lo,i_hi,s,0),
// key=(seed_lo,seed_hi)).x, X = (float)(-log((u + 0.5) * 2^-32)) evaluated in double.
// X is stored row-major [m][r] so one row's r keys are contiguous for the gathers.
__global__ void k_cohen_keys(int64_t m, int64_t row0, int r, uint64_t seed, float *X,
                             float *keys_out) {
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t gi = (uint64_t)(row0 + i);
        for (int s = 0; s < r; s++) {
            uint4 o = philox4x32_10(make_uint4((uint32_t)gi, (uint32_t)(gi >> 32), (uint32_t)s, 0u), key);
            const float x = (float)(-log(((double)o.x + 0.5) * (1.0 / 4294967296.0)));
            X[i * r + s] = x;
            if (keys_out) keys_out[(int64_t)s * m + i] = x;
        }
    }
}
cudaError_t launch_cohen_keys(int64_t m, int64_t row0, int r, uint64_t seed, float *X,
                              float *keys_out, cudaStream_t s) {
    if (m <= 0) return cudaSuccess;
    int64_t b = (m + 255) / 256;
    if (b > g_sms * 16) b = g_sms * 16;
    ++g_launches;
    k_cohen_keys<<<(int)b, 256, 0, s>>>(m, row0, r, seed, X, keys_out);
    return cudaGetLastError();
}

// One layer of min-propagation: out[j][s] = min_{i in inds(M_*j)} in[i][s].
// With est != nullptr (the output layer) also est_j = (r-1) / sum_s out[j][s], 0 when
// column j reaches nothing.  One warp per column; r <= 16 keys in registers.
__global__ void k_cohen_min(int64_t ncols, const int64_t *__restrict__ cp,
                            const int32_t *__restrict__ row, int64_t c0,
                            const float *__restrict__ in, int r, float *__restrict__ out,
                            float *__restrict__ est) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = lane_id();
    for (int64_t col = w; col < ncols; col += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        float mn[16];
#pragma unroll
        for (int s = 0; s < 16; s++) mn[s] = INFINITY;
        const int64_t q0 = cp[c0 + col], q1 = cp[c0 + col + 1];
        if ((r & 1) == 0) {
            // even r: 8-byte key loads (rows of r floats are 8-byte aligned), two entries per
            // lane per trip so both gathers are in flight together
            int64_t q = q0 + lane;
            for (; q + 32 < q1; q += 64) {
                const float2 *s0 = reinterpret_cast<const float2 *>(in + (int64_t)__ldg(row + q) * r);
                const float2 *s1 = reinterpret_cast<const float2 *>(in + (int64_t)__ldg(row + q + 32) * r);
#pragma unroll
                for (int s = 0; s < 8; s++)
                    if (2 * s < r) {
                        const float2 a = __ldg(s0 + s), b = __ldg(s1 + s);
                        mn[2 * s] = fminf(mn[2 * s], fminf(a.x, b.x));
                        mn[2 * s + 1] = fminf(mn[2 * s + 1], fminf(a.y, b.y));
                    }
            }
            if (q < q1) {
                const float2 *s0 = reinterpret_cast<const float2 *>(in + (int64_t)__ldg(row + q) * r);
#pragma unroll
                for (int s = 0; s < 8; s++)
                    if (2 * s < r) {
                        const float2 a = __ldg(s0 + s);
                        mn[2 * s] = fminf(mn[2 * s], a.x);
                        mn[2 * s + 1] = fminf(mn[2 * s + 1], a.y);
                    }
            }
        } else {
            for (int64_t q = q0 + lane; q < q1; q += 32) {
                const float *src = in + (int64_t)__ldg(row + q) * r;
#pragma unroll
                for (int s = 0; s < 16; s++)
                    if (s < r) mn[s] = fminf(mn[s], __ldg(src + s));
            }
        }
        double sum = 0.0;
#pragma unroll
        for (int s = 0; s < 16; s++) {
            if (s < r) {
                float v = warp_min(mn[s]);
                if (out && lane == 0) out[col * r + s] = v;
                sum += (double)v;
            }
        }
        if (est && lane == 0) est[col] = isinf(sum) ? 0.0f : (float)((double)(r - 1) / sum);
    }
}
cudaError_t launch_cohen_min(int64_t ncols, const int64_t *cp, const int32_t *row, int64_t c0,
                             const float *in, int r, float *out, float *est, cudaStream_t s) {
    if (ncols <= 0) return cudaSuccess;
    int64_t blocks = (ncols * 32 + 255) / 256;
    if (blocks > g_sms * 32) blocks = g_sms * 32;
    ++g_launches;
    k_cohen_min<<<(int)blocks, 256, 0, s>>>(ncols, cp, row, c0, in, r, out, est);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ preprocessing (Alg. 1 l.1)
__device__ __forceinline__ int64_t lower_bound_row(const int32_t *rows, int64_t lo, int64_t hi,
                                                   int32_t key) {
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (rows[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}
__global__ void k_pre_count(int64_t n, const int64_t *gcp, const int32_t *grow, int add_loops,
                            int64_t *cnt) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = gcp[j], b = gcp[j + 1];
        int64_t c = b - a;
        if (add_loops) {
            int64_t p = lower_bound_row(grow, a, b, (int32_t)j);
            if (!(p < b && grow[p] == (int32_t)j)) c += 1;
        }
        cnt[j] = c;
    }
}
cudaError_t launch_pre_count(int64_t n, const int64_t *gcp, const int32_t *grow, int add_loops,
                             int64_t *cnt, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    ++g_launches;
    k_pre_count<<<red_grid(n) * 4, 256, 0, s>>>(n, gcp, grow, add_loops, cnt);
    return cudaGetLastError();
}
// Warp per column: insert / add the self-loop of weight 1 (Q10), sum the column in
// fp64 and write w / sum (column-stochastic).
__global__ void k_pre_fill(int64_t n, const int64_t *__restrict__ gcp,
                           const int32_t *__restrict__ grow, const float *__restrict__ gw,
                           int add_loops, const int64_t *__restrict__ cp, int32_t *__restrict__ row,
                           float *__restrict__ val) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = lane_id();
    for (int64_t j = w; j < n; j += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t a = gcp[j], b = gcp[j + 1];
        int64_t p = b;
        bool has = false;
        if (add_loops) {
            p = lower_bound_row(grow, a, b, (int32_t)j);
            has = p < b && grow[p] == (int32_t)j;
        }
        const bool ins = add_loops && !has;
        double s = 0.0;
        for (int64_t t = a + lane; t < b; t += 32) {
            double x = (double)gw[t];
            if (add_loops && grow[t] == (int32_t)j) x += 1.0;
            s += x;
        }
        s = warp_sum(s);
        if (ins) s += 1.0;
        const int64_t o = cp[j];
        for (int64_t t = a + lane; t < b; t += 32) {
            double x = (double)gw[t];
            if (add_loops && grow[t] == (int32_t)j) x += 1.0;
            const int64_t d = o + (t - a) + ((ins && t >= p) ? 1 : 0);
            row[d] = grow[t];
            val[d] = (float)(x / s);
        }
        if (ins && lane == 0) {
            row[o + (p - a)] = (int32_t)j;
            val[o + (p - a)] = (float)(1.0 / s);
        }
    }
}
cudaError_t launch_pre_fill(int64_t n, const int64_t *gcp, const int32_t *grow, const float *gw,
                            int add_loops, const int64_t *cp, int32_t *row, float *val,
                            cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    int64_t blocks = (n * 32 + 255) / 256;
    if (blocks > g_sms * 32) blocks = g_sms * 32;
    ++g_launches;
    k_pre_fill<<<(int)blocks, 256, 0, s>>>(n, gcp, grow, gw, add_loops, cp, row, val);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ connected components
// Union-find with min-index hooking (a root is always its component's smallest vertex)
// and path halving; then canonical labels = rank of the root among roots (Q11).
__device__ __forceinline__ int32_t uf_find(int32_t *parent, int32_t x) {
    volatile int32_t *p = parent;
    int32_t px = p[x];
    while (px != x) {
        int32_t g = p[px];
        if (g != px) p[x] = g;
        x = px;
        px = p[x];
    }
    return x;
}
__global__ void k_cc_init(int64_t n, int32_t *parent) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        parent[i] = (int32_t)i;
}
__global__ void k_cc_hook(int64_t n, const int64_t *__restrict__ cp, const int32_t *__restrict__ row,
                          int32_t *parent) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = lane_id();
    for (int64_t j = w; j < n; j += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        for (int64_t t = cp[j] + lane; t < cp[j + 1]; t += 32) {
            int32_t a = row[t], b = (int32_t)j;
            for (;;) {
                a = uf_find(parent, a);
                b = uf_find(parent, b);
                if (a == b) break;
                int32_t hi = a > b ? a : b, lo = a > b ? b : a;
                int32_t old = atomicCAS(&parent[hi], hi, lo);
                if (old == hi) break;
                a = hi;
                b = lo;
            }
        }
    }
}
// After hooking the forest is static: roots are found read-only (a path-halving write
// here could overwrite another thread's stored root with a non-root ancestor).
__global__ void k_cc_flag(int64_t n, const int32_t *parent, int64_t *flag, int32_t *root) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t x = (int32_t)i, px = parent[x];
        while (px != x) {
            x = px;
            px = parent[x];
        }
        root[i] = x;
        flag[i] = (x == (int32_t)i) ? 1 : 0;
    }
}
__global__ void k_cc_label(int64_t n, const int64_t *rank, int32_t *labels) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        labels[i] = (int32_t)rank[labels[i]];
}
cudaError_t launch_cc(int64_t n, const int64_t *cp, const int32_t *row, int32_t *parent,
                      int64_t *flag, int64_t *rank, void *scan_tmp, int32_t *labels,
                      cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int g = red_grid(n) * 4;
    ++g_launches;
    k_cc_init<<<g, 256, 0, s>>>(n, parent);
    int64_t blocks = (n * 32 + 255) / 256;
    if (blocks > g_sms * 32) blocks = g_sms * 32;
    ++g_launches;
    k_cc_hook<<<(int)blocks, 256, 0, s>>>(n, cp, row, parent);
    ++g_launches;
    k_cc_flag<<<g, 256, 0, s>>>(n, parent, flag, labels);
    cudaError_t e = launch_scan_i64(flag, rank, n, scan_tmp, s);
    if (e != cudaSuccess) return e;
    ++g_launches;
    k_cc_label<<<g, 256, 0, s>>>(n, rank, labels);
    return cudaGetLastError();
}

}  // namespace mclx
