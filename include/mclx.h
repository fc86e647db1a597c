/*
 * mclx.h -- C ABI of libmclx.so, the B200-native (sm_100a) hot path of HipMCL's
 * Markov Cluster method (Selvitopi, Hussain, Azad, Buluc; arXiv:2002.10083).
 *
 * Citations are to /root/reference/PAPER.md as P:<line> with the enclosing
 * section / algorithm, and to DESIGN.md readings Q1..Q20 where the paper is
 * silent.  The path (Alg. 1 lines 3-5) is one MCL iteration:
 *   expansion B = A*A (SpGEMM), prune (threshold + top-k, P:161, P:187-188,
 *   recovery Q7), inflation (Hadamard power r) and column
 *   renormalisation (Q1), plus the cluster extraction of Alg. 1 line 6.
 *
 * Conventions common to every call
 *  - Matrices are CSC (§III-B: CSC in, CSC out, C = AB formed
 *    column-by-column, no transpose).  All pointers inside mcl_csc_t are DEVICE
 *    pointers on the context's device.  col_ptr is int64 [ncols+1] with
 *    col_ptr[0] = 0 and non-decreasing; row_idx is int32 [nnz], strictly
 *    increasing inside each column; val is fp32 [nnz], finite and > 0 (>= 0 for an
 *    unpruned product, whose entries may underflow to 0, Q13).
 *  - Inputs are BORROWED: owned by the caller, valid in stream order for the
 *    duration of the call, never modified.
 *  - Outputs (mcl_csc_t *out arguments) are ALLOCATED BY THE LIBRARY through
 *    the context's allocator callback and become caller-owned on return; free
 *    them with mcl_csc_release (which calls the free callback).
 *  - All device work is enqueued on the context stream.  Calls that must size
 *    an output (mcl_expand, mcl_spgemm, mcl_prune_inflate, mcl_iterate,
 *    mcl_merge, mcl_preprocess) synchronise that stream a small, fixed number of
 *    times to read sizes; results are valid in stream order when the call returns.
 *  - Every call returns MCL_OK (0) or a negative MCL_ERR_* code.  On error, out
 *    matrices are zeroed (nnz 0, NULL pointers), nothing leaks, and
 *    mcl_last_error(ctx) describes the failure.  The library never aborts and
 *    never prints.
 *  - There is no CPU fallback: every arithmetic step runs in the library's own
 *    sm_100a kernels.  A context refuses to be created on a device that is not
 *    compute capability 10.0 (MCL_ERR_UNSUPPORTED_DEVICE).
 */
#ifndef MCLX_H
#define MCLX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCLX_VERSION 1

enum {
    MCL_OK = 0,
    MCL_ERR_INVALID_ARG = -1,       /* NULL pointer, r <= 1, S < 1, pct outside [0,1], theta < 0, ... */
    MCL_ERR_DIM = -2,               /* A.ncols != B.nrows, non-square where A*A is needed, bad range */
    MCL_ERR_FORMAT = -3,            /* only with env MCLX_VALIDATE=1 (checked on the device for every
                                       input matrix): col_ptr not 0-based / non-decreasing / ending at
                                       nnz, a row outside [0, nrows) or not strictly increasing in its
                                       column, a negative or non-finite value          */
    MCL_ERR_OOM = -4,               /* allocator returned NULL                                          */
    MCL_ERR_CUDA = -5,              /* a CUDA runtime error (message in mcl_last_error)                 */
    MCL_ERR_NCCL = -6,              /* an NCCL error                                                    */
    MCL_ERR_UNSUPPORTED_DEVICE = -7,/* device is not sm_100 (B200)                                      */
    MCL_ERR_NOT_IMPLEMENTED = -8,
    MCL_ERR_INTERNAL = -9           /* a device consistency check failed, or a hash table overflowed
                                       even at the exact size bound min(f_j, m) (a library bug)     */
};

/* A CSC block.  (row0, col0, n_global) place the block in a global matrix for the
 * multi-GPU partition (all 0 / n on one GPU); row0 also offsets the Cohen key
 * counters so that a block's keys equal the global matrix's keys. */
typedef struct {
    int64_t nrows, ncols, nnz;
    int64_t row0, col0, n_global;
    int64_t *col_ptr; /* device, [ncols+1] */
    int32_t *row_idx; /* device, [nnz]     */
    float *val;       /* device, [nnz]     */
} mcl_csc_t;

/* Parameters of one MCL iteration.  Defaults (mcl_params_default) in brackets. */
typedef struct {
    double inflation;        /* r > 1 [2.0]  Hadamard power, r = 2 at P:770 (Q2)   */
    double prune_threshold;  /* theta >= 0 [1e-4]  keep v >= theta, "user supplied" (Q3,Q4) */
    int32_t select_k;        /* S >= 1 [1100]  top-S when more than S survive, P:188 (Q5,Q6)  */
    int32_t recover_k;       /* R >= 0 [1400]  0 disables recovery (Q7)                        */
    double recover_pct;      /* pct in [0,1] [0.9]  recover when kept mass < pct (Q7)          */
    double chaos_eps;        /* [1e-3] convergence threshold used by the caller's loop (Q9)    */
    int32_t est_keys;        /* r for Cohen, 2..16 [10]                           */
    double est_cf_threshold; /* [2.0] exact symbolic sizing when estimated cf < this  */
    uint64_t seed;           /* [0x5eed] Philox key of the Cohen exponential keys (Q14)        */
    double mem_safety;       /* [0.9] fraction of free HBM the phase planner may use (Q15)     */
    int32_t estimator;       /* [0] 0 = policy of P:1076-1077, 1 = always exact symbolic,
                                2 = always Cohen (with overflow retry)                        */
    int32_t force_bin;       /* [-1] >= 0 forces every non-empty column into bin (force_bin % 7)
                                or a bigger one (6 = the fp64 global-memory bin), of kernel
                                family force_bin / 7 (0 private row-range slices, 1 CTA-shared
                                atomic table) -- for bin-invariance tests                      */
} mcl_params_t;

#define MCL_NUM_BINS 6 /* shared-memory bins; bin index MCL_NUM_BINS is the global-memory bin */

/* Filled by the calls that take it (NULL allowed).  -1 = not computed. */
typedef struct {
    int64_t flops;           /* sum_j sum_{k in inds(B_*j)} nnz(A_*k)              */
    int64_t nnz_in;          /* nnz(A)                                                          */
    int64_t nnz_unpruned;    /* nnz(A*A) when known (expand, exact symbolic), else -1           */
    int64_t nnz_out;         /* nnz of the returned matrix                                      */
    double est_nnz;          /* Cohen estimate of nnz(A*A) (sum over columns), -1 if not run    */
    double cf;               /* flops / nnz_unpruned (or / est_nnz)                             */
    float chaos;             /* max_j chaos_j of the pruned, renormalised columns (Q9)          */
    int32_t phases;          /* column batches ("phases") the call ran: the planner cuts
                                the output columns into batches of near-equal estimated bytes
                                within mem_safety x free HBM (env MCLX_PHASES=h forces h)       */
    int32_t retries;         /* columns re-run after a hash-table overflow                      */
    int32_t estimator_used;  /* 1 exact symbolic, 2 Cohen, 3 Cohen-binned numeric into upper-bound
                                slots min(f_j, m) + compaction (unfused products, no symbolic) */
    int64_t bin_cols[MCL_NUM_BINS + 1];
    int64_t bin_flops[MCL_NUM_BINS + 1];
    float ms[8];             /* per stage: 0 flops/bin, 1 estimate, 2 symbolic, 3 numeric
                                (fused numeric+select+inflate in mcl_iterate), 4 select/inflate
                                (unfused), 5 assemble, 6 total, 7 numeric launches count.
                                mcl_summa_iterate with pr > 1: 0-2 and 5 the last phase's
                                distributed prune (stats, top-K cut, kept sums, write),
                                3 set-up (panels, broadcast wait, stacking, phase plan),
                                4 products of all phases, 7 distributed prunes of all phases  */
    int64_t peak_bytes;      /* peak scratch bytes held by the context                          */
    int64_t launches;        /* kernels this call launched                                      */
    float bin_ms[MCL_NUM_BINS + 1];          /* device time of each bin's kernel(s) (events)    */
    int64_t bin_nnzb[MCL_NUM_BINS + 1];      /* sum of nnz(B_*j) over the bin's columns         */
    int64_t bin_out[MCL_NUM_BINS + 1];       /* entries the bin wrote (fused: kept entries)     */
    int64_t comm_bytes;      /* bytes this rank received in SUMMA broadcasts                    */
    int64_t peak_partial;    /* peak live nnz of SUMMA stage partials (Alg. 2 schedule)         */
    int64_t split_cols;      /* columns run as row-range parts (counted in bin MCL_NUM_BINS too) */
    int64_t split_items;     /* row-range parts run                                             */
    float split_ms;          /* device time of the split path (included in bin_ms[MCL_NUM_BINS])*/
    int64_t split_vcols[3];  /* split columns per part variant: 8192-slot shared tables,
                                16384-slot shared tables, fp64 global tables                    */
    float split_vms[3];      /* device time per part variant (parts + stitch + prune)           */
    int32_t stages;          /* SUMMA inner panels (stage products per phase), 0 if none        */
    int64_t esc_cols;        /* low-cf columns run by expand-sort-compress (env MCLX_ESC_CF = the
                                cf threshold, default 1.5; 0 turns it off), not in bin_*       */
    int64_t esc_flops;
    int64_t esc_out;         /* entries the ESC kernel wrote (fused: kept entries)             */
    float esc_ms;            /* its device time                                                */
} mcl_stats_t;

/* Allocator callbacks: device memory, stream-ordered.  NULL callbacks select the
 * built-in cudaMallocAsync/cudaFreeAsync pool. */
typedef void *(*mcl_alloc_fn)(void *state, size_t bytes, void *stream);
typedef void (*mcl_free_fn)(void *state, void *ptr, size_t bytes, void *stream);

typedef struct mcl_ctx *mcl_ctx_t;

int mcl_version(void);
void mcl_params_default(mcl_params_t *p);

/* Create a context on `device` enqueuing on `stream` (a cudaStream_t; NULL = the
 * legacy default stream).  Fails with MCL_ERR_UNSUPPORTED_DEVICE off sm_100. */
int mcl_ctx_create(mcl_ctx_t *ctx, int device, void *stream, mcl_alloc_fn alloc,
                   mcl_free_fn free_fn, void *alloc_state);
int mcl_ctx_set_stream(mcl_ctx_t ctx, void *stream);
int mcl_ctx_destroy(mcl_ctx_t ctx);
const char *mcl_last_error(mcl_ctx_t ctx);

/* Free a matrix returned by this library (no-op on an all-zero struct). */
int mcl_csc_release(mcl_ctx_t ctx, mcl_csc_t *m);

/* Alg. 1 line 1: A = column-stochastic version of the weighted
 * adjacency matrix G (square, weights > 0).  add_loops != 0 adds a self-loop of
 * weight 1.0 to every vertex first, summed onto an existing diagonal (Q10).
 * Empty columns (add_loops == 0) stay empty. */
int mcl_preprocess(mcl_ctx_t ctx, const mcl_csc_t *G, int add_loops, mcl_csc_t *A_out);

/* flops per column: flops_j = sum_{k in inds(B_*j)} nnz(A_*k).
 * flops_dev: optional device int64 [B.ncols]; total: optional host int64. */
int mcl_flops(mcl_ctx_t ctx, const mcl_csc_t *A, const mcl_csc_t *B, int64_t *flops_dev,
              int64_t *total);

/* Cohen's probabilistic size estimate of C = A*B (§V; lambda = 1 and
 * r keys per first-layer vertex).  est_dev: device fp32 [B.ncols]
 * receives (r-1)/sum_s c_j[s] (0 for an unreachable column).  keys_dev (optional,
 * device fp32 [r * A.nrows], plane-major [s][i]) receives the exponential keys
 * X[s][i] = (float)(-log((u+0.5) 2^-32)), u = Philox4x32-10(ctr=(i_lo,i_hi,s,0),
 * key=(seed_lo,seed_hi))[0], i = A.row0 + local row (Q14).  total: optional host sum. */
int mcl_estimate(mcl_ctx_t ctx, const mcl_csc_t *A, const mcl_csc_t *B, int32_t r,
                 uint64_t seed, float *est_dev, float *keys_dev, double *total);

/* Exact symbolic pass (§V): nnz_dev (device int64
 * [B.ncols]) receives |union_{k in inds(B_*j)} inds(A_*k)|. */
int mcl_symbolic(mcl_ctx_t ctx, const mcl_csc_t *A, const mcl_csc_t *B, int64_t *nnz_dev,
                 int64_t *total);

/* Unpruned product C[:, b:e) = A * B[:, b:e) (rectangular blocks for the
 * Sparse-SUMMA stages).  Exact sizes from the symbolic pass; rows
 * sorted ascending; values fp32 (fp64 accumulation for columns with
 * nnz(B_*j) > 16384).  C_out->ncols = e - b. */
int mcl_spgemm(mcl_ctx_t ctx, const mcl_csc_t *A, const mcl_csc_t *B, int64_t col_begin,
               int64_t col_end, const mcl_params_t *p, mcl_csc_t *C_out, mcl_stats_t *st);

/* The expansion of Alg. 1 line 3: mcl_spgemm(A, A, ...).  A square. */
int mcl_expand(mcl_ctx_t ctx, const mcl_csc_t *A, int64_t col_begin, int64_t col_end,
               const mcl_params_t *p, mcl_csc_t *C_out, mcl_stats_t *st);

/* Alg. 1 lines 4-5 on an unpruned C (readings Q1-Q9): per column, threshold,
 * top-S select / recovery / argmax fallback, renormalise, Hadamard power r,
 * renormalise.  st->chaos = max_j chaos_j.  chaos_dev (optional, device fp32
 * [C.ncols]) receives chaos_j. */
int mcl_prune_inflate(mcl_ctx_t ctx, const mcl_csc_t *C, const mcl_params_t *p,
                      mcl_csc_t *A_next, float *chaos_dev, mcl_stats_t *st);

/* One fused MCL iteration (Alg. 1 lines 3-5): flop count and binning, size
 * estimate (Cohen or exact symbolic by the P:1076-1077 policy), numeric hash
 * SpGEMM whose epilogue selects / prunes / recovers / inflates / renormalises each
 * column while it is still in shared memory, then assembly of A_next.  The
 * unpruned product never reaches HBM. */
int mcl_iterate(mcl_ctx_t ctx, const mcl_csc_t *A, const mcl_params_t *p, mcl_csc_t *A_next,
                mcl_stats_t *st);

/* mcl_iterate restricted to the output columns [col_begin, col_end) (A square):
 * A_next = the pruned, inflated columns b..e-1 of the next iterate (ncols = e - b,
 * col0 = A.col0 + b).  Columns are independent given A (pruning is per column,
 * P:208; inflation per entry), which is what the phases of P:212-218 and the
 * column partition across GPUs of P:401-406 rely on. */
int mcl_iterate_range(mcl_ctx_t ctx, const mcl_csc_t *A, int64_t col_begin, int64_t col_end,
                      const mcl_params_t *p, mcl_csc_t *A_next, mcl_stats_t *st);

/* Alg. 1 line 6: weak connected components of the pattern of A (Q11).
 * labels_dev: caller-owned device int32 [A.ncols]; components are numbered in
 * order of their smallest vertex.  ncl: host. */
int mcl_clusters(mcl_ctx_t ctx, const mcl_csc_t *A, int32_t *labels_dev, int64_t *ncl);

/* Merge L equally shaped CSC blocks into their sum (the "merge all lists
 * in L" step of Alg. 2).  Rows sorted, duplicate rows summed. */
int mcl_merge(mcl_ctx_t ctx, int32_t L, const mcl_csc_t *lists, mcl_csc_t *out);

/* ---------------------------------------------------------------- 2D Sparse SUMMA
 * P:222-246 §II "Overview of Sparse SUMMA", generalised to a pr x pc grid (Q17): rank
 * r = i*pc + j owns block (i, j) = rows [i n/pr, (i+1) n/pr) x cols [j n/pc, (j+1) n/pc)
 * of every iterate.  The inner dimension is cut into s = lcm(pr, pc) panels K_q; at stage
 * q rank (i, floor(q pc/s)) broadcasts A[rows_i, K_q] along its row communicator and rank
 * (floor(q pr/s), j) broadcasts A[K_q, cols_j] along its column communicator (NCCL over
 * NVLink).  Forms of the local product:
 *   pr = 1: every column of C lives on one rank; all stages accumulate in the fused kernel
 *     and the prune is local.
 *   pr > 1 (default): the resident panels are stacked into A[rows_i, :] and A[:, cols_j] and
 *     ONE fused product in candidate mode yields each column's top-max(S, R) entries plus
 *     the statistics of all its entries (the stage partials merge in the hash tables).
 *   pr > 1 with MCLX_SUMMA_STAGED=1: a product per stage (mcl_spgemm) and the Alg. 2 binary
 *     merge on the device.
 * The pruning of a column split over pr ranks exchanges only fixed-size all-reduces
 * (per-column counts and sums, radix-select digit histograms for the exact top-k cut).
 */

/* out = A[r0:r1, c0:c1] (local index ranges) as a block: row ids rebased to r0, row0 / col0
 * advanced by r0 / c0, n_global kept.  Used to distribute an iterate over the grid. */
int mcl_block(mcl_ctx_t ctx, const mcl_csc_t *A, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
              mcl_csc_t *out);
/* Development counters of the SpGEMM kernel (all zero unless libmclx was built with
 * -DMCLX_PROF): [0] warp insert calls, [1] probe-loop passes, [2] products, [3] accumulate
 * cycles summed over warps, [4] epilogue cycles summed over CTAs, [5] columns, epilogue
 * phases: [6] table compaction, [7] stats + select + kept compaction, [8] sums, [9] sort
 * and write; [10], [11] reserved. */
int mcl_prof_read(uint64_t out[12], int reset);
/* rank 0 creates the id and shares it (e.g. through torch.distributed) */
int mcl_nccl_unique_id(unsigned char out[128]);
/* collective over the pr*pc ranks: creates the world, row and column communicators */
int mcl_ctx_set_grid(mcl_ctx_t ctx, int pr, int pc, int rank, const unsigned char id[128]);
/* One MCL iteration (Alg. 1 lines 3-5) on the distributed iterate.  A: this rank's block
 * (row0/col0/n_global set as above); A_next: its block of the next iterate.  Collective;
 * st->chaos is the global chaos. */
int mcl_summa_iterate(mcl_ctx_t ctx, const mcl_csc_t *A, const mcl_params_t *p, mcl_csc_t *A_next,
                      mcl_stats_t *st);

/* The schedule mcl_summa_iterate runs (host arithmetic only; no device, no NCCL): for rank
 * `rank` of a pr x pc grid over n vertices with s = lcm(pr, pc) x stage_mult inner panels,
 * out[0..3] = the rank's block rows [r0, r1) and columns [c0, c1); then for every stage q,
 * out[4 + 5q ..] = k0, k1 (the inner panel K_q), the grid column of the A-panel's owner in the
 * rank's row, the grid row of the B-panel's owner in its column, and Alg. 2's nmerges after
 * pushing stage q's partial.  cap: entries of out (>= 4 + 5 s).  Returns s. */
int mcl_summa_schedule(int pr, int pc, int rank, int64_t n, int stage_mult, int64_t *out, int64_t cap);

/* Host-memory-backed iteration: the Pipelined Sparse SUMMA of P:337-363
 * §III on one GPU, for an iterate larger than the device's memory.  A_host is a square CSC in
 * HOST memory (pinned memory lets the copies run asynchronously).  The output columns run in
 * `phases` batches of near-equal nnz; within a phase the inner dimension is cut
 * into `stages` panels: the column panel A[:, K_q] is copied to the device on a copy stream,
 * double-buffered so that stage q+1's copy overlaps stage q's product; the rows K_q
 * of the phase's columns (copied once per phase) are sliced on the device; the partial
 * products are merged on the device by Alg. 2 -- the paper merges them on the
 * host, this library does no arithmetic on the CPU -- and the merged batch is pruned /
 * inflated and copied back to host memory.  The device holds two A-panels, one phase's
 * columns, its partials and staging, not A.  stages / phases <= 0: chosen from
 * mem_safety x free HBM.  A_next_host receives pinned HOST arrays allocated by the library,
 * freed with mcl_host_csc_release.  st->stages / phases / peak_partial; st->comm_bytes = the
 * host -> device bytes. */
int mcl_iterate_hostmem(mcl_ctx_t ctx, const mcl_csc_t *A_host, const mcl_params_t *p,
                        int32_t stages, int32_t phases, mcl_csc_t *A_next_host, mcl_stats_t *st);
int mcl_host_csc_release(mcl_csc_t *m);

/* ------------------------------------------------------------------ I/O around the kernel
 * Host-side (no CUDA) ingestion of a weighted graph and the cluster output file (SURVEY §8(f)
 * row 4; SPEC S:547-559 load_graph / run).  All arrays are HOST memory owned by the struct. */
typedef struct {
    int64_t n, nnz;
    int64_t *col_ptr;  /* host [n+1]                                                       */
    int32_t *row_idx;  /* host [nnz], strictly increasing inside each column               */
    float *val;        /* host [nnz], > 0                                                   */
    char **labels;     /* host [n] vertex labels of a TSV input, NULL for MatrixMarket     */
} mcl_graph_t;

/* Read a graph: MatrixMarket coordinate (real / integer / pattern -> 1.0, general /
 * symmetric, 1-based) or a labelled edge list "src dst [weight]" (TSV or spaces; labels get
 * dense ids in order of first appearance; column = src, row = dst).  Duplicates are summed,
 * exact zeros dropped; symmetrize != 0 returns max(A, A^T).  On error g is zeroed, err
 * (optional, errlen bytes) names the file and line: MCL_ERR_FORMAT (malformed line, negative
 * weight, symmetric-marker violation, entry count), MCL_ERR_DIM (non-square), MCL_ERR_OOM,
 * MCL_ERR_INVALID_ARG (unreadable file). */
int mcl_graph_read(const char *path, int symmetrize, mcl_graph_t *g, char *err, size_t errlen);
void mcl_graph_free(mcl_graph_t *g);
/* Write the clusters of `labels` (host int32 [n], cluster ids 0..k-1 as mcl_clusters numbers
 * them, i.e. by smallest member): one line per cluster, its members in ascending vertex order
 * separated by single spaces -- the graph's labels, or 1-based vertex ids (g NULL or without
 * labels). */
int mcl_clusters_write(const char *path, const int32_t *labels, int64_t n, const mcl_graph_t *g);

#ifdef __cplusplus
}
#endif
#endif /* MCLX_H */
