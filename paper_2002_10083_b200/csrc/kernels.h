// kernels.h -- host-side launch wrappers for the libmclx kernels (internal header).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "mclx_dev.cuh"

namespace mclx {

// Shared-memory bins: table capacity (slots) and CTA size.  Bin kNumBins is the
// global-memory (fp64) bin.  A column goes to the smallest bin whose table holds
// its size bound at load factor <= 1/2 (kLoadNum/kLoadDen).
constexpr int kNumBins = 6;
constexpr int kBinCap[kNumBins] = {512, 1024, 2048, 4096, 8192, 16384};
constexpr int kBinThreads[kNumBins] = {32, 32, 64, 128, 256, 512};
constexpr int kGlobalThreads = 512;
__host__ __device__ constexpr int bin_cap(int b) {
    return b == 0 ? 512 : b == 1 ? 1024 : b == 2 ? 2048 : b == 3 ? 4096 : b == 4 ? 8192 : 16384;
}

constexpr int kFp64Terms = 16384;  // nnz(B_*j) above which a column accumulates in fp64 (T)

// kPart: one row-range part of a split column (see run_bins): accumulate only the rows of
// rowparts [p0, p1) and write the part's entries, rows sorted, to its staging slot
enum Mode { kSym = 0, kNum = 1, kFused = 2, kPart = 3 };

// Host-side count of kernel launches issued by this library (reported in mcl_stats_t).
extern int64_t g_launches;
// Multiprocessor count of the current context's device (set by mcl_ctx_create); launch
// helpers size persistent grids as multiples of it.
extern int g_sms;

struct BinArgs {
    // operands: C = A * B[:, cb : cb + ncols_out)
    const int64_t *acp;
    const int32_t *arow;
    const float *aval;
    int64_t m;
    const int64_t *bcp;
    const int32_t *brow;
    const float *bval;
    int64_t cb;
    const int64_t *flops;  // [ncols_out]
    const int2 *apair;     // [nnz(A)] (row, value bits) pairs of A: one 8-byte gather per product
    const int *rowpart;    // [A.ncols][33] row-range index of A (see kernels_spgemm.cu)
    const int *rowpart_fine;  // [A.ncols][129] (split parts of the private family)
    // work list of this bin
    const int32_t *list;
    const int *count;
    int *counter;
    // global bin layout (per list index)
    const int64_t *goff;
    const int32_t *gcap;
    int *gkeys;
    double *gvals;
    // outputs
    int64_t *sym_nnz;                                   // kSym
    const int64_t *c_cp;                                // kNum
    int64_t *c_cnt;     // kNum with upper-bound slots: per-column counts (else exact c_cp)
    int32_t *c_row;
    float *c_val;
    const int64_t *soff;                                // kFused
    int32_t *s_row;
    float *s_val;
    int64_t *s_cnt;
    float *chaos;
    float *chaos_max;
    int32_t *retry_list;
    int *retry_count;
    int *err_flag;
    unsigned long long *bin_out;  // this bin's output-entry counter (kFused)
    PruneParams pp;
    // kPart: item i = part [p0, p1) (item_pr[i] = p0 | p1 << 8) of column list[i]
    const int32_t *item_pr;
    const int64_t *stg_off;                             // staging offset of each item
    int32_t *stg_row;
    float *stg_val;
    int64_t *stg_cnt;
    int *col_flag;                                      // [ncols_out] overflowed split columns
    // kPart with cand_k > 0: a part stages only its top-cand_k entries (value desc, row asc;
    // cand_k = max(S, R), so the column's kept set is among them for every branch of
    // Alg. 1 l.4) and reports the statistics of ALL its entries for the branch decision
    // kFused with cand_k > 0 (candidate mode, the 2D SUMMA's row blocks): the same epilogue per
    // output column -- its top-cand_k entries unscaled into (soff, s_row, s_val, s_cnt) and its
    // statistics into stg_nnz / stg_m / stg_s indexed by column; the prune runs after the
    // column communicator has summed the statistics of all row blocks (dist_prune)
    int cand_k;
    int64_t *stg_nnz;  // [items] entries of the part
    int64_t *stg_m;    // [items] entries >= theta
    double *stg_s;     // [items] their mass (fp64)
};
// the dense sweep's candidate buffer: a round of the tile compaction appends <= 1024 entries,
// and the buffer is cut back to cand_k (a radix select) when it could overflow, so the
// slack kCandBuf - 1024 - cand_k sets how often that happens (~every slack accepted entries)
constexpr int kCandBuf = 4096;
constexpr int kCandMax = 2048;
// the shared-table bin that runs the parts of split columns (table slots, threads)
constexpr int kPartCap = 8192;
constexpr int kPartThreads = 512;
constexpr int kPartNeed = kPartCap / 2;  // distinct rows a part is sized for (load 1/2)
constexpr int kParts = 32;  // row ranges of the rowpart index (k_rowpart)
constexpr int kFineParts = 128;  // the finer index used by private-slice split parts
// dense bin (kernels_dense.cu): kDenseParts row-range parts per column, each swept tile by
// tile with per-segment cursors (tile + kSweepSeg descriptors in shared memory)
constexpr int kDenseThreads = 1024;
constexpr int kDenseParts = 8;             // parts of a dense column (32 / 8 = 4 rowparts each)
constexpr int kSweepTileBytes = 163840;    // dense tile: 40960 fp32 / 20480 fp64 rows
constexpr int kSweepSeg = 2048;            // segment descriptors (cursor, end, b) per chunk
// split_P flag: the column needs fp64 accumulation (more than kFp64Terms segments)
constexpr int kSplitFp64 = 1 << 30;
// split_P flag: short sub-segments, run the parts in the CTA-shared-table family
constexpr int kSplitShared = 1 << 29;
// split_P flag: sweep the column's row ranges with dense tiles (kernels_dense.cu)
constexpr int kSplitDense = 1 << 28;
// split_P flag (MCLX_SPLIT_BIG=1): half as many parts, each in a 2*kPartCap-slot table
constexpr int kSplitBig = 1 << 27;
constexpr int kSplitFlags = kSplitFp64 | kSplitShared | kSplitDense | kSplitBig;
// work items (row-range parts) of a split column from its split_P entry: the dense variants
// (more than 64 virtual parts, or fp64) sweep kDenseParts ranges, hashed parts min(P, 32)
__host__ __device__ inline int split_parts(int Pf) {
    const int P = Pf & ~kSplitFlags;
    return (Pf & (kSplitFp64 | kSplitDense)) ? kDenseParts : (P < 32 ? P : 32);
}
cudaError_t launch_dense_part(bool fp64, const BinArgs &a, int grid, cudaStream_t s);
int dense_part_occupancy(bool fp64);
// part variants: 0 kPartCap-slot shared table, 1 2*kPartCap-slot shared table
// (variants 2 / 3, dense fp32 / fp64 row tiles: launch_dense_part)
cudaError_t launch_part(int variant, const BinArgs &a, int grid, cudaStream_t s);
int part_occupancy(int variant);

// Two kernel families share the bins: private row-range slices (bin b = 0..kNumBins) for
// columns whose average gathered segment is long, and a CTA-shared atomic table
// (bin kFamily + b) for short-segment (R-MAT-like) columns.
constexpr int kFamily = kNumBins + 1;
constexpr int kAllBins = 2 * kFamily;
constexpr int kShortSegment = 16;  // flops_j / nnz(B_*j) below this -> atomic family

// expand-sort-compress kernel of low-cf columns (kernels_esc.cu): one CTA per column of
// at most kEscCap products
constexpr int kEscCap = 1024;
constexpr int kEscThreads = 128;
cudaError_t launch_esc(int mode, const BinArgs &a, int grid, cudaStream_t s);
int esc_occupancy(int mode);

// One launch of bin `bin` (0..kAllBins-1) in mode `mode`; grid chosen from occupancy.
cudaError_t launch_bin(int mode, int bin, const BinArgs &a, int grid, cudaStream_t s);
// Max resident CTAs per SM for (mode, bin); also sets the dynamic smem attribute.
int bin_occupancy(int mode, int bin);
void prof_read(unsigned long long out[12], int reset);  // development counters (-DMCLX_PROF)
size_t bin_smem_bytes(int mode, int bin);

// rowpart[k][i] = first position in A_*k whose row >= ceil(i*m/32), i = 0..32
cudaError_t launch_rowpart(int64_t ncols, const int64_t *cp, const int32_t *row, int64_t m,
                           int *rowpart, cudaStream_t s, int nparts = 32);

// misc kernels (kernels_misc.cu)
// dst[i] = src[idx[i]]
cudaError_t launch_gather_i32(int64_t n, const int32_t *idx, const int32_t *src, int32_t *dst,
                              cudaStream_t s);
cudaError_t launch_gather_i64(int64_t n, const int32_t *idx, const int64_t *src, int64_t *dst,
                              cudaStream_t s);
// phase planner (capi.cu plan_phases): per-column byte estimates and the batch cuts
cudaError_t launch_affine_i64(int64_t n, const int64_t *x, int64_t a, int64_t b, int64_t *bytes,
                              bool accumulate, cudaStream_t s);
cudaError_t launch_affine_est(int64_t n, const float *est, double a, int64_t b, int64_t *bytes,
                              cudaStream_t s);
cudaError_t launch_phase_cuts(const int64_t *prefix, int64_t n, int h, int64_t *cut, cudaStream_t s);
// apair[q] = (row[q], bits of val[q]): the interleaved copy of A the private family gathers
cudaError_t launch_pack_pairs(int64_t nnz, const int32_t *row, const float *val, int2 *apair,
                              cudaStream_t s);
// CSC invariants of include/mclx.h (MCLX_VALIDATE); *flag |= 1 col_ptr, 2 row range,
// 4 row order, 8 value (not finite or <= 0)
cudaError_t launch_validate_csc(int64_t ncols, int64_t nrows, int64_t nnz, const int64_t *cp,
                                const int32_t *row, const float *val, int *flag, cudaStream_t s);
cudaError_t launch_flops(int64_t ncols, const int64_t *acp, const int64_t *bcp,
                         const int32_t *brow, int64_t cb, int64_t *f, cudaStream_t s);
cudaError_t launch_reduce_i64(const int64_t *x, int64_t n, unsigned long long *out, cudaStream_t s);
cudaError_t launch_reduce_f32(const float *x, int64_t n, double *out, cudaStream_t s);
// exclusive scan of in[0,n) into out[0,n], out[n] = total.  tmp: >= scan_tmp_bytes(n)
size_t scan_tmp_bytes(int64_t n);
cudaError_t launch_scan_i64(const int64_t *in, int64_t *out, int64_t n, void *tmp, cudaStream_t s);
struct ClassifyArgs {
    int64_t n;               // number of columns to classify
    const int32_t *cols;     // optional explicit column list (retry), else 0..n-1
    const int64_t *flops;
    const int64_t *bcp;
    int64_t cb;
    const float *est;        // optional
    const int64_t *exact;    // optional
    int64_t m;
    float alpha;
    float max_load;          // table load factor bound used for binning (<= 0.5 default)
    int force_bin;
    int force_family;        // -1 auto, 0 private slices, 1 atomic shared table
    int64_t list_stride;     // columns per bin list
    int *bin_count;          // [kAllBins]
    int32_t *lists;          // [kAllBins * list_stride]
    int32_t *gcap_col;       // [ncols_out]
    unsigned long long *bin_flops;  // [kNumBins + 1]
    unsigned long long *bin_nnzb;   // [kNumBins + 1] sum of nnz(B_*j)
    int32_t *colbin;         // optional [ncols_out]: the bin chosen for each column
    // split columns (kFused): global-bin columns with need <= split_max are processed
    // as split_P[col] row-range parts (a power of two, 2..32) instead
    int64_t split_max;       // 0 disables
    int64_t split_min;       // also split smaller columns with need > split_min (tests)
    int64_t split_part_need; // distinct rows a part is sized for (kPartNeed)
    int dense_min_P;         // virtual part counts above this (<= 64) take the dense sweep
    int split_big;           // P in [4, 32]: P/2 parts of 2*kPartCap-slot tables (kSplitBig)
    int64_t fp64_terms;      // nnz(B_*j) above which a column accumulates in fp64 (kFp64Terms)
    // low-cf columns (kernels_esc.cu): f_j <= esc_max and f_j < esc_cf x (estimated or exact
    // nnz_j) run the expand-sort-compress kernel; esc_max = 0 disables
    int64_t esc_max;
    double esc_cf;
    int *esc_count;
    int32_t *esc_list;
    unsigned long long *esc_flops;
    int *split_count;
    int32_t *split_list;
    int32_t *split_P;
};
// items of the split columns: item ioff[s] + p = part p of split column s
cudaError_t launch_split_items(int nsplit, const int32_t *split_list, const int32_t *split_P,
                               const int64_t *ioff, int32_t *item_col, int32_t *item_pr,
                               cudaStream_t s);
// stitch the parts of split columns [s0, s0 + nc) (items from ioff[s0]) into an unpruned
// CSC: ccp from the scanned part counts sioff; colmap = product column, or -1 when a part
// overflowed (the column is re-run in a later round)
// with stg_nnz (candidates) also the column sums of the parts' statistics -> fnnz, fm, fs
cudaError_t launch_split_stitch(int nc, const int64_t *ioff, int64_t item0, const int32_t *item_col,
                                const int64_t *sioff, const int *col_flag, int64_t *ccp,
                                int32_t *colmap, const int64_t *stg_nnz, const int64_t *stg_m,
                                const double *stg_s, int64_t *fnnz, int64_t *fm, double *fs,
                                cudaStream_t s);
cudaError_t launch_split_gather(int64_t nitems, const int64_t *stg_cnt, const int64_t *stg_off,
                                const int32_t *stg_row, const float *stg_val, const int64_t *sioff,
                                int32_t *crow, float *cval, cudaStream_t s);
cudaError_t launch_classify(const ClassifyArgs &c, cudaStream_t s);
// Locality order of the bin work lists: key[j] = min over rows i of B_*j of a hash of
// i (a MinHash of the column's row set, so columns with similar row sets -- the same
// family / cluster -- get equal keys); the lists are rewritten sorted by (bin, key >> 16).
constexpr int kOrderBits = 16;
cudaError_t launch_minhash_key(int64_t n, const int64_t *bcp, const int32_t *brow, int64_t cb,
                               uint32_t *key, cudaStream_t s);
cudaError_t launch_order_lists(int64_t n, const int32_t *cols, const int32_t *colbin,
                               const uint32_t *key, int64_t *hist, int64_t *offs, void *scan_tmp,
                               int32_t *lists, int64_t list_stride, cudaStream_t s);
cudaError_t launch_global_layout(int count, const int32_t *list, const int32_t *gcap_col,
                                 int32_t *gcap, int64_t *gcap64, cudaStream_t s);
cudaError_t launch_kcap(int64_t ncols, const int64_t *flops, int64_t m, int kmax, int64_t *kcap,
                        cudaStream_t s);
cudaError_t launch_kcap_cp(int64_t ncols, const int64_t *cp, int kmax, int64_t *kcap,
                           cudaStream_t s);
cudaError_t launch_offset_colptr(int64_t n1, const int64_t *cp, int64_t off, int64_t *out,
                                 cudaStream_t s);
cudaError_t launch_stack_identity(int64_t n, int L, int64_t *cp, int32_t *row, float *val,
                                  cudaStream_t s);
cudaError_t launch_copy_cols(int64_t ncols, const int64_t *cnt, const int64_t *soff,
                             const int32_t *srow, const float *sval, const int64_t *cp,
                             int32_t *orow, float *oval, cudaStream_t s);
// candidate mode: cut stitched split columns to their top-K, write them to the staging slots
// and scatter their statistics to column-indexed arrays (onnz, om, os)
cudaError_t launch_cand_select(int64_t ncols, const int64_t *ccp, const int32_t *crow, const float *cval,
                               const int32_t *colmap, int K, const int64_t *fnnz, const int64_t *fm,
                               const double *fs, const int64_t *soff, int32_t *srow, float *sval,
                               int64_t *scnt, int64_t *onnz, int64_t *om, double *os,
                               unsigned long long *out_count, int grid, cudaStream_t s);
cudaError_t launch_prune(int64_t ncols, const int64_t *ccp, const int32_t *crow, const float *cval,
                         const int64_t *soff, int32_t *srow, float *sval, int64_t *scnt,
                         float *chaos, float *chaos_max, const PruneParams &pp, int grid,
                         cudaStream_t s, const int32_t *colmap = nullptr,
                         unsigned long long *out_count = nullptr, const int64_t *fnnz = nullptr,
                         const int64_t *fm = nullptr, const double *fs = nullptr);
cudaError_t launch_cohen_keys(int64_t m, int64_t row0, int r, uint64_t seed, float *X,
                              float *keys_out, cudaStream_t s);
cudaError_t launch_cohen_min(int64_t ncols, const int64_t *cp, const int32_t *row, int64_t c0,
                             const float *in, int r, float *out, float *est, cudaStream_t s);
cudaError_t launch_pre_count(int64_t n, const int64_t *gcp, const int32_t *grow, int add_loops,
                             int64_t *cnt, cudaStream_t s);
cudaError_t launch_pre_fill(int64_t n, const int64_t *gcp, const int32_t *grow, const float *gw,
                            int add_loops, const int64_t *cp, int32_t *row, float *val,
                            cudaStream_t s);
cudaError_t launch_cc(int64_t n, const int64_t *cp, const int32_t *row, int32_t *parent,
                      int64_t *flag, int64_t *rank, void *scan_tmp, int32_t *labels,
                      cudaStream_t s);

// SUMMA kernels (kernels_summa.cu)
constexpr int kMaxStages = 16;
struct VStack {  // s <= kMaxStages B-panels (row ranges starting at k0[q]) of one column stripe
    const int64_t *cp[kMaxStages];
    const int32_t *row[kMaxStages];
    const float *val[kMaxStages];
    int64_t k0[kMaxStages];
    int s;
};
// count_only: cnt[j] = nnz of stacked column j; else copy into (ocp, orow, oval)
cudaError_t launch_vstack(int64_t nj, const VStack &v, int64_t *cnt, const int64_t *ocp, int32_t *orow,
                          float *oval, bool count_only, cudaStream_t s);
cudaError_t launch_rebase_colptr(int64_t n1, const int64_t *cp, int64_t *out, cudaStream_t s);
cudaError_t launch_rowslice_count(int64_t ncols, const int64_t *cp, const int32_t *rows, int64_t r0,
                                  int64_t r1, int64_t *first, int64_t *cnt, cudaStream_t s);
cudaError_t launch_rowslice_copy(int64_t ncols, const int64_t *first, const int64_t *ocp,
                                 const int32_t *rows, const float *vals, int64_t r0, int32_t *orow,
                                 float *oval, cudaStream_t s);
cudaError_t launch_dp_stats(int64_t ncols, const int64_t *cp, const float *vals, double theta,
                            int64_t *nnz, int64_t *m, double *sm, int grid, cudaStream_t s);
cudaError_t launch_dp_branch(int64_t ncols, const int64_t *nnz, const int64_t *m, const double *sm,
                             const PruneParams &pp, int64_t *K, int8_t *mode, int32_t *rem,
                             uint32_t *prefix, int32_t *rowcut, cudaStream_t s);
// ccnt (dp_hist / dp_keepstats / dp_write): column j's entries are [cp[j], cp[j] + ccnt[j])
// (staging slots) instead of [cp[j], cp[j + 1]) (compact CSC).
// packed: histograms as 128 words per column, bins b and b + 128 in the low / high 16 bits
// (the caller guarantees every global count < 2^16: candidate columns, <= ranks x max(S, R))
cudaError_t launch_dp_hist(int64_t nsel, const int32_t *sel, const int64_t *cp, const int32_t *rows,
                           const float *vals, int64_t row0, const int8_t *mode, const uint32_t *vprefix,
                           const uint32_t *rprefix, const int32_t *done, int pass, unsigned *hist,
                           int grid, cudaStream_t s, int packed = 0, const int64_t *ccnt = nullptr);
cudaError_t launch_dp_sellist(int64_t ncols, const int8_t *mode, int64_t *flag, int64_t *pos,
                              int32_t *sel, void *tmp, cudaStream_t s);
cudaError_t launch_dp_undone(int64_t nsel, const int32_t *sel, const int32_t *done,
                             unsigned long long *cnt, cudaStream_t s);
cudaError_t launch_dp_digit(int64_t nsel, const int32_t *sel, const unsigned *hist, int pass,
                            uint32_t *vprefix, uint32_t *rprefix, int32_t *rem, int32_t *done,
                            int32_t *rowcut, cudaStream_t s, int packed = 0);
cudaError_t launch_dp_keepstats(int64_t ncols, const int64_t *cp, const int32_t *rows,
                                const float *vals, int64_t row0, const int8_t *mode,
                                const uint32_t *vprefix, const int32_t *rowcut, const PruneParams &pp,
                                int64_t *kcnt, double *sums, int grid, cudaStream_t s,
                                const int64_t *ccnt = nullptr);
cudaError_t launch_dp_write(int64_t ncols, const int64_t *cp, const int32_t *rows, const float *vals,
                            int64_t row0, const int8_t *mode, const uint32_t *vprefix,
                            const int32_t *rowcut, const PruneParams &pp, const double *gsums,
                            const int64_t *gkcnt, const int64_t *soff, int32_t *srow, float *sval,
                            int64_t *scnt, float *chaos, float *chaos_max, int grid, cudaStream_t s,
                            const int64_t *ccnt = nullptr);

}  // namespace mclx
