// capi.cu -- the C ABI of libmclx.so (include/mclx.h): context, allocation, and the
// host orchestration of each entry point (which kernels, in what order, which few
// small read-backs).  No arithmetic of the method happens on the host.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <functional>
#include <string>
#include <unordered_map>
#include <vector>

#include <nccl.h>

#include "kernels.h"
#include "mclx.h"

using namespace mclx;

struct Buf {
    void *p = nullptr;
    size_t bytes = 0;
};

struct mcl_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    mcl_alloc_fn alloc = nullptr;
    mcl_free_fn free_fn = nullptr;
    void *state = nullptr;
    std::string err;
    int sms = 148;
    std::unordered_map<std::string, Buf> scratch;
    size_t cur = 0, peak = 0;
    int occ[3][kAllBins] = {};
    void *pin = nullptr;     // mapped pinned read-back buffer (readback)
    size_t pin_bytes = 0;
    void *pin_up = nullptr;  // mapped pinned upload buffer (upload)
    size_t pin_up_bytes = 0;
    cudaEvent_t up_ev = nullptr;
    cudaEvent_t ev[8] = {};
    cudaEvent_t bev[2 * kAllBins + 2] = {};  // per bin (+ the ESC kernel)
    cudaEvent_t pev[6] = {};  // phases of the distributed prune
    cudaEvent_t sev[3] = {};  // SUMMA iteration (ev[] is reused by the stage products)
    cudaEvent_t vev[2] = {};  // split path, per part variant
    // 2D Sparse-SUMMA grid (mcl_ctx_set_grid): world / row / column communicators
    int pr = 1, pc = 1, rank = 0;
    ncclComm_t world = nullptr, rowc = nullptr, colc = nullptr;
    cudaStream_t cstream = nullptr;          // SUMMA stage broadcasts (pipelined)
    float *cohen_M_pre = nullptr;            // a precomputed Cohen first layer for the next call
    int cohen_M_r = 0;
    cudaEvent_t qev[5] = {};                 // ready[2], free[2], start
    int64_t gbin_budget = (int64_t)32 << 30;  // bytes of fp64 global-bin tables live at once
    float alpha = 1.2f;     // table sizing: need = alpha * Cohen estimate + 16
    float max_load = 0.5f;  // bin when need <= max_load * cap
    bool order_lists = true;  // MinHash locality order of the bin work lists
    bool split = true;        // row-range split of big fused columns (MCLX_SPLIT=0: off)
    int64_t split_budget = (int64_t)4 << 30;  // staging bytes per chunk of split parts
    int64_t split_min_need = INT64_MAX;       // MCLX_SPLIT_MIN_NEED: split smaller columns too
    int64_t split_part_need = kPartNeed;      // MCLX_SPLIT_PART_NEED (<= kPartNeed; tests)
    int64_t fp64_terms = kFp64Terms;          // MCLX_FP64_TERMS (tests)
    int64_t cap_budget = (int64_t)48 << 30;   // unfused products: upper-bound slots up to this
    bool split_private = true;                // MCLX_SPLIT_PRIVATE=0: P <= 4 parts shared-table too
    bool validate = false;                    // MCLX_VALIDATE=1: check input CSC invariants
    bool split_cand = true;                   // MCLX_SPLIT_CAND=0: split parts stage every entry
    int dense_min_P = 64;                     // MCLX_DENSE_MIN_P: split columns of more parts go dense
    int split_big = 0;                        // MCLX_SPLIT_BIG=1: half the parts, 2x tables (A/B)
    double esc_cf = 1.5;                      // MCLX_ESC_CF: cf below which a small column runs ESC (0: off)
    double esc_iter_cf = 2.0;                 // MCLX_ESC_ITER_CF: ... when the product's cf is below this
    int force_phases = 0;                     // MCLX_PHASES=h forces h column batches (tests)
    int64_t phase_budget = -1;                // MCLX_PHASE_BUDGET_MB: bytes per batch (else
                                              // mem_safety x free HBM)
    size_t free_seen = 0;                     // free HBM at the last cudaMemGetInfo (phase_budget)
    int family = -1;                          // MCLX_FAMILY=0/1 forces a kernel family (A/B runs)
};

namespace {

int fail(mcl_ctx *c, int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    return code;
}

// MCLX_TRACE_SYNC=<ms>: report host syncs slower than <ms> (source line, bytes, wall ms) on
// stderr -- a diagnostic for host stalls that leave the GPU idle
static double g_trace_ms = -1.0;
static void trace_init() {
    static bool done = false;
    if (done) return;
    done = true;
    if (const char *e = getenv("MCLX_TRACE_SYNC")) g_trace_ms = atof(e);
}
static double now_ms() {
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return t.tv_sec * 1e3 + t.tv_nsec * 1e-6;
}

// host gaps between traced calls (the host busy or descheduled while the GPU may idle)
static double g_trace_last = 0.0;
static int g_trace_last_line = 0;
static void trace_gap(int line, double t0) {
    if (g_trace_last > 0.0 && t0 - g_trace_last > g_trace_ms)
        fprintf(stderr, "[mclx sync] gap line %d -> %d %.3f ms\n", g_trace_last_line, line,
                t0 - g_trace_last);
}
static void trace_end(int line) {
    g_trace_last = now_ms();
    g_trace_last_line = line;
}
static void trace_call(int line, double t0) {
    const double dt = now_ms() - t0;
    trace_gap(line, t0);
    if (dt > g_trace_ms) fprintf(stderr, "[mclx sync] call line %d %.3f ms\n", line, dt);
    trace_end(line);
}

#define CK(call)                                                                              \
    do {                                                                                      \
        const double tq_ = g_trace_ms >= 0 ? now_ms() : 0.0;                                  \
        cudaError_t e_ = (call);                                                              \
        if (g_trace_ms >= 0) trace_call(__LINE__, tq_);                                       \
        if (e_ != cudaSuccess)                                                                \
            return fail(c, MCL_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,         \
                        cudaGetErrorString(e_));                                              \
    } while (0)

#define RC(call)                   \
    do {                           \
        int r_ = (call);           \
        if (r_ != MCL_OK) return r_; \
    } while (0)

void *dalloc(mcl_ctx *c, size_t bytes) {
    if (bytes == 0) bytes = 16;
    void *p = nullptr;
    if (c->alloc) {
        trace_init();
        const double t0 = g_trace_ms >= 0 ? now_ms() : 0.0;
        p = c->alloc(c->state, bytes, (void *)c->stream);
        if (g_trace_ms >= 0) {
            trace_gap(-1, t0);
            if (now_ms() - t0 > g_trace_ms)
                fprintf(stderr, "[mclx sync] alloc bytes %zu %.3f ms\n", bytes, now_ms() - t0);
            trace_end(-1);
        }
    } else if (cudaMallocAsync(&p, bytes, c->stream) != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
    }
    return p;
}
void dfree(mcl_ctx *c, void *p, size_t bytes) {
    if (!p) return;
    if (c->free_fn) {
        const double t0 = g_trace_ms >= 0 ? now_ms() : 0.0;
        c->free_fn(c->state, p, bytes, (void *)c->stream);
        if (g_trace_ms >= 0) {
            trace_gap(-2, t0);
            if (now_ms() - t0 > g_trace_ms)
                fprintf(stderr, "[mclx sync] free bytes %zu %.3f ms\n", bytes, now_ms() - t0);
            trace_end(-2);
        }
    } else {
        cudaFreeAsync(p, c->stream);
    }
}

// Named, growing scratch buffers owned by the context.
int scratch(mcl_ctx *c, const char *name, size_t bytes, void **out) {
    Buf &b = c->scratch[name];
    if (b.bytes < bytes) {
        if (b.p) {
            dfree(c, b.p, b.bytes);
            c->cur -= b.bytes;
        }
        size_t nb = bytes + bytes / 8 + 4096;
        b.p = dalloc(c, nb);
        if (!b.p) {
            b.bytes = 0;
            return fail(c, MCL_ERR_OOM, "scratch '%s': cannot allocate %zu bytes", name, nb);
        }
        b.bytes = nb;
        c->cur += nb;
        c->peak = std::max(c->peak, c->cur);
    }
    *out = b.p;
    return MCL_OK;
}
template <typename T>
int scratch_t(mcl_ctx *c, const char *name, size_t count, T **out) {
    return scratch(c, name, count * sizeof(T), (void **)out);
}

// Host <-> device transfers of the orchestration (sizes, work lists, plans) go through
// mapped pinned buffers copied by KERNELS, not cudaMemcpy: copy-engine work is served in
// order, so a memcpy here would queue behind a caller's large transfer on another stream (the
// e2e bench's result read-back of the previous step / input upload of the next) and stall the
// iteration at each of its host syncs.  The buffers grow on demand.
constexpr size_t kPinBytes = 65536;  // initial size of each mapped pinned buffer

__global__ void k_copy_bytes(const unsigned char *__restrict__ src, unsigned char *__restrict__ dst,
                             size_t n) {
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
    if ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) {
        const size_t n16 = n >> 4;
        for (size_t i = t; i < n16; i += nt)
            reinterpret_cast<uint4 *>(dst)[i] = reinterpret_cast<const uint4 *>(src)[i];
        for (size_t i = (n16 << 4) + t; i < n; i += nt) dst[i] = src[i];
    } else {
        for (size_t i = t; i < n; i += nt) dst[i] = src[i];
    }
}

void launch_copy_bytes(const void *src, void *dst, size_t n, cudaStream_t s) {
    const size_t blocks = std::min<size_t>(std::max<size_t>((n + 4095) / 4096, 1), 256);
    ++g_launches;
    k_copy_bytes<<<(unsigned)blocks, 256, 0, s>>>((const unsigned char *)src, (unsigned char *)dst, n);
}

// grow a mapped pinned buffer to >= bytes (its contents are not kept)
int ensure_pin(mcl_ctx *c, void **buf, size_t *cap, size_t bytes) {
    if (*cap >= bytes) return MCL_OK;
    if (*buf) cudaFreeHost(*buf);
    *buf = nullptr;
    *cap = 0;
    const size_t nb = std::max(bytes + bytes / 2, kPinBytes);
    if (cudaHostAlloc(buf, nb, cudaHostAllocMapped) != cudaSuccess) {
        cudaGetLastError();
        return fail(c, MCL_ERR_OOM, "cannot allocate %zu bytes of pinned host memory", nb);
    }
    *cap = nb;
    return MCL_OK;
}

// Copy `bytes` from device to host through the mapped read-back buffer; waits for the stream.
int readback_at(int line, mcl_ctx *c, const void *dev, size_t bytes, void *host) {
    if (bytes == 0) return MCL_OK;
    if (!dev) return fail(c, MCL_ERR_INVALID_ARG, "readback from a NULL device pointer");
    trace_init();
    const double t0 = g_trace_ms >= 0 ? now_ms() : 0.0;
    RC(ensure_pin(c, &c->pin, &c->pin_bytes, bytes));
    launch_copy_bytes(dev, c->pin, bytes, c->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
    memcpy(host, c->pin, bytes);
    if (g_trace_ms >= 0) {
        const double dt = now_ms() - t0;
        trace_gap(line, t0);
        if (dt > g_trace_ms) fprintf(stderr, "[mclx sync] readback line %d bytes %zu %.3f ms\n", line, bytes, dt);
        trace_end(line);
    }
    return MCL_OK;
}
#define readback(...) readback_at(__LINE__, __VA_ARGS__)

// Copy `bytes` from host to device through the mapped upload buffer, stream-ordered (the
// host buffer may be reused at return; the upload buffer is reused after its copy ran).
int upload_at(int line, mcl_ctx *c, const void *host, size_t bytes, void *dev) {
    if (bytes == 0) return MCL_OK;
    if (!dev) return fail(c, MCL_ERR_INVALID_ARG, "upload to a NULL device pointer");
    trace_init();
    const double t0 = g_trace_ms >= 0 ? now_ms() : 0.0;
    CK(cudaEventSynchronize(c->up_ev));  // the previous upload's copy has read the buffer
    RC(ensure_pin(c, &c->pin_up, &c->pin_up_bytes, bytes));
    memcpy(c->pin_up, host, bytes);
    launch_copy_bytes(c->pin_up, dev, bytes, c->stream);
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->up_ev, c->stream));
    if (g_trace_ms >= 0) {
        const double dt = now_ms() - t0;
        trace_gap(line, t0);
        if (dt > g_trace_ms) fprintf(stderr, "[mclx sync] upload line %d bytes %zu %.3f ms\n", line, bytes, dt);
        trace_end(line);
    }
    return MCL_OK;
}
#define upload(...) upload_at(__LINE__, __VA_ARGS__)

void zero_csc(mcl_csc_t *m) {
    if (m) memset(m, 0, sizeof *m);
}

void free_csc(mcl_ctx *c, mcl_csc_t *m) {
    dfree(c, m->col_ptr, 0);
    dfree(c, m->row_idx, 0);
    dfree(c, m->val, 0);
    zero_csc(m);
}

// Frees an output matrix on every early return unless release()d: the header's "on
// error, outputs are zeroed and nothing leaks" contract for the entry points.
struct OutGuard {
    mcl_ctx *c;
    mcl_csc_t *m;
    bool armed = true;
    OutGuard(mcl_ctx *c_, mcl_csc_t *m_) : c(c_), m(m_) {}
    ~OutGuard() {
        if (armed && m) free_csc(c, m);
    }
    void release() { armed = false; }
};

int alloc_rows_vals(mcl_ctx *c, mcl_csc_t *m, int64_t nnz) {
    m->nnz = nnz;
    m->row_idx = (int32_t *)dalloc(c, (size_t)std::max<int64_t>(nnz, 1) * sizeof(int32_t));
    m->val = (float *)dalloc(c, (size_t)std::max<int64_t>(nnz, 1) * sizeof(float));
    if (!m->row_idx || !m->val) return fail(c, MCL_ERR_OOM, "cannot allocate %lld nnz", (long long)nnz);
    return MCL_OK;
}

int check_csc(mcl_ctx *c, const mcl_csc_t *m, const char *what) {
    if (!m) return fail(c, MCL_ERR_INVALID_ARG, "%s is NULL", what);
    if (m->nrows < 0 || m->ncols < 0 || m->nnz < 0)
        return fail(c, MCL_ERR_INVALID_ARG, "%s has negative dimensions", what);
    if (!m->col_ptr) return fail(c, MCL_ERR_INVALID_ARG, "%s.col_ptr is NULL", what);
    if (m->nnz > 0 && (!m->row_idx || !m->val))
        return fail(c, MCL_ERR_INVALID_ARG, "%s has nnz > 0 but NULL arrays", what);
    if (m->nrows > 0x7ffffffeLL) return fail(c, MCL_ERR_DIM, "%s: more than 2^31-2 rows", what);
    if (c->validate) {  // MCLX_VALIDATE=1: the CSC invariants, checked on the device
        int *flag;
        RC(scratch_t(c, "validate_flag", 1, &flag));
        CK(cudaMemsetAsync(flag, 0, sizeof(int), c->stream));
        CK(launch_validate_csc(m->ncols, m->nrows, m->nnz, m->col_ptr, m->row_idx, m->val, flag,
                               c->stream));
        int h = 0;
        RC(readback(c, flag, sizeof(int), &h));
        if (h)
            return fail(c, MCL_ERR_FORMAT, "%s is not a valid CSC:%s%s%s%s", what,
                        (h & 1) ? " col_ptr not 0-based / non-decreasing / ending at nnz;" : "",
                        (h & 2) ? " row index out of range;" : "",
                        (h & 4) ? " rows not strictly increasing in a column;" : "",
                        (h & 8) ? " a value is negative or not finite;" : "");
    }
    return MCL_OK;
}

int check_params(mcl_ctx *c, const mcl_params_t *p) {
    if (!(p->inflation > 1.0)) return fail(c, MCL_ERR_INVALID_ARG, "inflation must be > 1");
    if (!(p->prune_threshold >= 0.0)) return fail(c, MCL_ERR_INVALID_ARG, "prune_threshold < 0");
    if (p->select_k < 1) return fail(c, MCL_ERR_INVALID_ARG, "select_k must be >= 1");
    if (p->recover_k < 0) return fail(c, MCL_ERR_INVALID_ARG, "recover_k must be >= 0");
    if (!(p->recover_pct >= 0.0 && p->recover_pct <= 1.0))
        return fail(c, MCL_ERR_INVALID_ARG, "recover_pct outside [0,1]");
    if (p->est_keys < 2 || p->est_keys > 16)
        return fail(c, MCL_ERR_INVALID_ARG, "est_keys must be in [2,16]");
    return MCL_OK;
}

PruneParams prune_params(const mcl_params_t *p) {
    PruneParams pp;
    pp.theta = p->prune_threshold;
    pp.S = p->select_k;
    pp.R = p->recover_k;
    pp.pct = p->recover_pct;
    pp.r = p->inflation;
    pp.r_is_2 = p->inflation == 2.0;
    pp.kmax = std::max(1, std::max(p->select_k, p->recover_k));
    return pp;
}

float elapsed(mcl_ctx *c, int a, int b) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c->ev[a], c->ev[b]) != cudaSuccess) {
        cudaGetLastError();
        return -1.f;
    }
    return ms;
}

void init_stats(mcl_stats_t *st) {
    if (!st) return;
    memset(st, 0, sizeof *st);
    st->nnz_unpruned = -1;
    st->est_nnz = -1;
    st->cf = -1;
    st->phases = 1;
    for (int i = 0; i < 8; i++) st->ms[i] = -1.f;
}

// Operands of one product C = A * B[:, cb : cb + n).
struct Prod {
    const mcl_csc_t *A, *B;
    int64_t cb, n;
};

// Cohen estimate for the output columns of a product.
int cohen(mcl_ctx *c, const Prod &pr, int r, uint64_t seed, float *est, float *keys_out) {
    float *M;
    if (c->cohen_M_pre && c->cohen_M_r == r) {
        // the first layer was computed distributedly (SUMMA 1 x N: each rank its own
        // column block, then broadcast), see mcl_summa_iterate
        M = c->cohen_M_pre;
        c->cohen_M_pre = nullptr;
    } else {
        float *X;
        RC(scratch_t(c, "cohen_X", (size_t)std::max<int64_t>(pr.A->nrows, 1) * r, &X));
        RC(scratch_t(c, "cohen_M", (size_t)std::max<int64_t>(pr.A->ncols, 1) * r, &M));
        CK(launch_cohen_keys(pr.A->nrows, pr.A->row0, r, seed, X, keys_out, c->stream));
        CK(launch_cohen_min(pr.A->ncols, pr.A->col_ptr, pr.A->row_idx, 0, X, r, M, nullptr, c->stream));
    }
    CK(launch_cohen_min(pr.n, pr.B->col_ptr, pr.B->row_idx, pr.cb, M, r, nullptr, est, c->stream));
    return MCL_OK;
}

// Split columns (fused mode): a column too big for one CTA's shared-memory table is
// processed as P row-range parts (rowparts [p 32/P, (p+1) 32/P)), one CTA each with a
// shared-memory table (kPart), which writes the part's entries, rows sorted, to a
// staging slot.  Per chunk of columns (staging bounded by split_budget) the parts are
// stitched -- parts are row ranges, so concatenation keeps rows sorted -- into an
// unpruned CSC that k_prune turns into the pruned / inflated columns (Alg. 1 l.4-5).
// The tables stay on chip, unlike the global bin's, and a column's work spreads over P
// SMs.  A part that overflows flags its column for the next round.
int run_split(mcl_ctx *c, const Prod &pr, int nsplit, int32_t *split_list,
              const int32_t *split_P, BinArgs a, unsigned long long *out_count,
              int64_t *nitems_out, mcl_stats_t *st) {
    // the split columns and their part counts (gathered on the device: nsplit entries, not n)
    std::vector<int32_t> hl((size_t)nsplit), hPl((size_t)nsplit);
    {
        int32_t *pl;
        RC(scratch_t(c, "split_Pl", (size_t)nsplit, &pl));
        CK(launch_gather_i32(nsplit, split_list, split_P, pl, c->stream));
        RC(readback(c, split_list, sizeof(int32_t) * nsplit, hl.data()));
        RC(readback(c, pl, sizeof(int32_t) * nsplit, hPl.data()));
    }
    std::unordered_map<int32_t, int32_t> hP;
    hP.reserve((size_t)nsplit * 2);
    for (int s2 = 0; s2 < nsplit; s2++) hP[hl[s2]] = hPl[s2];
    // variant by the virtual part count P (parts sized for T = split_part_need distinct
    // rows): <= 32 parts of kPartCap slots; 64: 32 parts of 2 kPartCap slots; more
    // (outputs dense in a sizable share of the rows, or long fp64 sums): kDenseParts row
    // ranges swept by dense fp32 / fp64 tiles (kernels_dense.cu), staging capacity
    // min(part rows, 2 P T / kDenseParts + 256)
    // variants: 4 (P <= 16: private row-range slices, 8 warps over the part's >= 8 rowparts
    // of the 128-way index), 0 (P = 32, or MCLX_SPLIT_PRIVATE=0: CTA-shared tables), 1, 2, 3
    // (the private family addresses A with 32-bit offsets; its 128-way row index costs a
    // pass over A, so it is built only when enough columns use it)
    auto priv_ok = [&](int Pf) {
        return (Pf & ~kSplitFlags) <= 16 && !(Pf & kSplitFlags);
    };
    int64_t npriv = 0;
    for (int s2 = 0; s2 < nsplit; s2++) npriv += priv_ok(hP[hl[s2]]);
    const bool priv = c->split_private && pr.A->nnz < ((int64_t)1 << 32) &&
                      (npriv >= 4096 || c->split_min_need != INT64_MAX);
    auto variant_of = [&](int Pf) {
        const int P = Pf & ~kSplitFlags;
        return (Pf & kSplitFp64) ? 3
               : (Pf & kSplitDense) ? 2
               : (Pf & kSplitBig) ? 1
               : priv && priv_ok(Pf) ? 4
               : P <= 32 ? 0 : 1;
    };
    const int vorder[5] = {4, 0, 1, 2, 3};
    for (int o = 4; o >= 0; o--)  // stable: variant order 4, 0, 1, 2, 3; columns keep their order
        std::stable_partition(hl.begin(), hl.end(),
                              [&](int32_t col) { return variant_of(hP[col]) == vorder[o]; });
    const int64_t cap_of[2] = {kPartCap, 2 * kPartCap};
    // candidates: each part stages only its top max(S, R) entries plus the statistics of all
    // of them (exact: the column's kept set lies in the union of its parts' top-max(S, R)
    // for every branch of Alg. 1 l.4, readings Q5-Q8), so the stitched columns k_prune reads
    // are short; MCLX_SPLIT_CAND=0 stages every entry instead
    // candidate mode (a.cand_k > 0, run_bins): the stitched columns are cut to their top
    // max(S, R) unscaled (k_cand_select) instead of pruned, so the parts always stage candidates
    const bool candm = a.cand_k > 0;
    const int cand_k = ((c->split_cand || candm) && a.pp.kmax <= kCandMax) ? a.pp.kmax : 0;
    std::vector<int64_t> hoff((size_t)nsplit + 1, 0);   // first item of each column
    std::vector<int64_t> hstg;                          // staging offset of each item
    hstg.reserve((size_t)nsplit * 4 + 1);
    int64_t stg = 0;
    for (int s2 = 0; s2 < nsplit; s2++) {
        const int v = variant_of(hP[hl[s2]]), P = hP[hl[s2]] & ~kSplitFlags;
        const int parts = split_parts(hP[hl[s2]]);
        hoff[s2 + 1] = hoff[s2] + parts;
        // a dense part's slot: its rows, or twice its share of the column's size bound
        const int64_t prow = (pr.A->nrows + kDenseParts - 1) / kDenseParts + 1;
        const int64_t dcap =
            std::min<int64_t>(prow, (int64_t)P * c->split_part_need * 2 / kDenseParts + 256);
        for (int q = 0; q < parts; q++) {
            hstg.push_back(stg);
            // the 7/8 fill limit bounds a hashed part's entries
            const int64_t tc = v == 1 ? cap_of[1] : cap_of[0];
            const int64_t slot = (v == 2 || v == 3) ? dcap : tc - tc / 8;
            stg += cand_k > 0 ? std::min<int64_t>(slot, cand_k) : slot;
        }
    }
    hstg.push_back(stg);
    const int64_t nitems = hoff[nsplit];
    *nitems_out = nitems;
    // chunks: whole columns of one variant, staging (x2: staged + stitched) within budget
    const int64_t budget = std::max<int64_t>(c->split_budget / 16, 1 << 16);  // entries
    std::vector<int> cuts{0};
    for (int s2 = 0; s2 < nsplit; s2++) {
        const int s0 = cuts.back();
        if (s2 == s0) continue;
        const bool vchange = variant_of(hP[hl[s2]]) != variant_of(hP[hl[s0]]);
        const bool full = hstg[hoff[s2 + 1]] - hstg[hoff[s0]] > budget;
        if (vchange || full) cuts.push_back(s2);
    }
    cuts.push_back(nsplit);
    const int nchunks = (int)cuts.size() - 1;
    int64_t chunk_items = 0, chunk_stg = 0;
    for (int q = 0; q < nchunks; q++) {
        const int64_t i0 = hoff[cuts[q]], i1 = hoff[cuts[q + 1]];
        chunk_items = std::max(chunk_items, i1 - i0);
        chunk_stg = std::max(chunk_stg, hstg[i1] - hstg[i0]);
    }
    // device copies: reordered column list, item layout
    int64_t *ioff, *stg_off, *stg_cnt, *sioff, *ccp;
    int32_t *item_col, *item_pr, *stg_row, *crow, *colmap;
    float *stg_val, *cval;
    int *ccount;
    void *tmp;
    RC(scratch_t(c, "split_ioff", (size_t)nsplit + 1, &ioff));
    RC(scratch_t(c, "split_stg_off", (size_t)nitems + 1, &stg_off));
    RC(scratch_t(c, "split_item_col", (size_t)nitems, &item_col));
    RC(scratch_t(c, "split_item_pr", (size_t)nitems, &item_pr));
    RC(scratch_t(c, "split_counts", (size_t)2 * nchunks, &ccount));
    RC(scratch_t(c, "split_stg_cnt", (size_t)chunk_items, &stg_cnt));
    RC(scratch_t(c, "split_sioff", (size_t)chunk_items + 1, &sioff));
    RC(scratch_t(c, "split_stg_row", (size_t)chunk_stg, &stg_row));
    RC(scratch_t(c, "split_stg_val", (size_t)chunk_stg, &stg_val));
    RC(scratch_t(c, "split_crow", (size_t)chunk_stg, &crow));
    RC(scratch_t(c, "split_cval", (size_t)chunk_stg, &cval));
    RC(scratch_t(c, "split_ccp", (size_t)nsplit + 1, &ccp));
    RC(scratch_t(c, "split_colmap", (size_t)nsplit, &colmap));
    int64_t *stg_nnz = nullptr, *stg_m = nullptr, *fnnz = nullptr, *fm = nullptr;
    double *stg_s = nullptr, *fs = nullptr;
    if (cand_k > 0) {
        RC(scratch_t(c, "split_stg_nnz", (size_t)chunk_items, &stg_nnz));
        RC(scratch_t(c, "split_stg_m", (size_t)chunk_items, &stg_m));
        RC(scratch_t(c, "split_stg_s", (size_t)chunk_items, &stg_s));
        RC(scratch_t(c, "split_fnnz", (size_t)nsplit, &fnnz));
        RC(scratch_t(c, "split_fm", (size_t)nsplit, &fm));
        RC(scratch_t(c, "split_fs", (size_t)nsplit, &fs));
    }
    RC(scratch(c, "split_scan_tmp", scan_tmp_bytes(chunk_items + 1), &tmp));
    std::vector<int> hcnt((size_t)2 * nchunks, 0);
    for (int q = 0; q < nchunks; q++) hcnt[q] = (int)(hoff[cuts[q + 1]] - hoff[cuts[q]]);
    RC(upload(c, hl.data(), sizeof(int32_t) * nsplit, split_list));
    RC(upload(c, hoff.data(), sizeof(int64_t) * (nsplit + 1), ioff));
    RC(upload(c, hstg.data(), sizeof(int64_t) * (nitems + 1), stg_off));
    RC(upload(c, hcnt.data(), sizeof(int) * 2 * nchunks, ccount));
    CK(launch_split_items(nsplit, split_list, split_P, ioff, item_col, item_pr, c->stream));
    bool any_private = false;
    for (int s2 = 0; s2 < nsplit && !any_private; s2++) any_private = variant_of(hP[hl[s2]]) == 4;
    if (any_private) {  // the 128-way row index of A for private-slice parts
        int *rp_fine;
        RC(scratch_t(c, "rowpart_fine", (size_t)std::max<int64_t>(pr.A->ncols, 1) * (kFineParts + 1),
                     &rp_fine));
        CK(launch_rowpart(pr.A->ncols, pr.A->col_ptr, pr.A->row_idx, pr.A->nrows, rp_fine, c->stream,
                          kFineParts));
        a.rowpart_fine = rp_fine;
    }
    int occ[5];
    for (int v = 0; v < 2; v++) occ[v] = std::max(1, part_occupancy(v));
    occ[4] = std::max(1, part_occupancy(4));
    occ[2] = std::max(1, dense_part_occupancy(false));
    occ[3] = std::max(1, dense_part_occupancy(true));
    const int pgrid = (int)std::min<int64_t>(std::max<int64_t>(pr.n, 1), (int64_t)c->sms * 8);
    int vprev = -1;
    for (int q = 0; q <= nchunks; q++) {
        const int vq = q < nchunks ? variant_of(hP[hl[cuts[q]]]) : -1;
        if (st && vq != vprev) {  // per-variant device time (chunks are grouped by variant)
            if (vprev >= 0) {
                CK(cudaEventRecord(c->vev[1], c->stream));
                CK(cudaEventSynchronize(c->vev[1]));
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, c->vev[0], c->vev[1]));
                st->split_vms[vprev == 4 ? 0 : vprev < 3 ? vprev : 2] += ms;
            }
            if (vq >= 0) CK(cudaEventRecord(c->vev[0], c->stream));
        }
        vprev = vq;
        if (q == nchunks) break;
        const int s0 = cuts[q], nc = cuts[q + 1] - cuts[q];
        const int64_t item0 = hoff[s0], nit = hoff[cuts[q + 1]] - item0;
        const int v = vq;
        if (st) st->split_vcols[v == 4 ? 0 : v < 3 ? v : 2] += nc;
        // staging offsets relative to the chunk: stg_off[i] - stg_off[item0]
        BinArgs ap = a;
        ap.list = item_col + item0;
        ap.item_pr = item_pr + item0;
        ap.count = ccount + q;
        ap.counter = ccount + nchunks + q;
        ap.stg_off = stg_off + item0;
        ap.stg_row = stg_row - hstg[item0];
        ap.stg_val = stg_val - hstg[item0];
        ap.stg_cnt = stg_cnt;
        ap.cand_k = cand_k;
        ap.stg_nnz = stg_nnz;
        ap.stg_m = stg_m;
        ap.stg_s = stg_s;
        const int grid = (int)std::min<int64_t>(nit, (int64_t)occ[v] * c->sms);
        if (v == 2 || v == 3) CK(launch_dense_part(v == 3, ap, grid, c->stream));
        else CK(launch_part(v, ap, grid, c->stream));
        CK(launch_scan_i64(stg_cnt, sioff, nit, tmp, c->stream));
        CK(launch_split_stitch(nc, ioff + s0, item0, item_col + item0, sioff, a.col_flag, ccp, colmap,
                               stg_nnz, stg_m, stg_s, fnnz, fm, fs, c->stream));
        CK(launch_split_gather(nit, stg_cnt, stg_off + item0, stg_row - hstg[item0],
                               stg_val - hstg[item0], sioff, crow, cval, c->stream));
        if (candm)
            CK(launch_cand_select(nc, ccp, crow, cval, colmap, a.cand_k, fnnz, fm, fs, a.soff, a.s_row,
                                  a.s_val, a.s_cnt, a.stg_nnz, a.stg_m, a.stg_s, out_count, pgrid,
                                  c->stream));
        else
            CK(launch_prune(nc, ccp, crow, cval, a.soff, a.s_row, a.s_val, a.s_cnt, a.chaos,
                            a.chaos_max, a.pp, pgrid, c->stream, colmap, out_count, fnnz, fm, fs));
    }
    return MCL_OK;
}

// Classify the columns of a product into bins and run every bin kernel in `mode`;
// columns whose table overflowed (estimate too small) are re-binned with the exact
// bound min(f_j, m) and re-run.  `base` carries the mode's outputs.
// product_cf: the multiplication's estimated compression factor (flops / sum of the size
// estimates; <= 0 unknown).  The ESC kernel is considered only for a product whose cf is below
// c->esc_iter_cf -- HipMCL's hybrid picks the kernel per multiplication by cf (P:789-794,
// P:812-815) -- and then per column (c->esc_cf).
int run_bins(mcl_ctx *c, int mode, const Prod &pr, const int64_t *f, const float *est,
             const int64_t *exact, int force_bin, BinArgs base, mcl_stats_t *st,
             double product_cf = -1.0) {
    const int64_t n = pr.n;
    const int NB1 = kAllBins;  // both kernel families
    int *counts, *counters, *retry_count, *err;
    unsigned long long *bflops;
    int32_t *lists, *gcap_col, *retry_list, *retry_in;
    // the bins' metadata in ONE buffer, so a round reads it back with one host sync after
    // the classification and one after the kernels.  ints: [0, NB1) bin counts, [NB1, 2 NB1)
    // work counters, 2 NB1 retry count, +1 error flag, +2 / +3 ESC count / counter, +4 split
    // count; then unsigned long longs: bin flops, bin nnz(B_*j), bin outputs, ESC flops / out
    const int kInts = 2 * NB1 + 6;
    const size_t ints_bytes = ((size_t)kInts * sizeof(int) + 15) & ~(size_t)15;
    const size_t ulls_bytes = sizeof(unsigned long long) * (3 * NB1 + 2);
    unsigned char *meta;
    RC(scratch(c, "bin_meta", ints_bytes + ulls_bytes, (void **)&meta));
    counts = reinterpret_cast<int *>(meta);
    counters = counts + NB1;
    retry_count = counters + NB1;
    err = retry_count + 1;
    bflops = reinterpret_cast<unsigned long long *>(meta + ints_bytes);
    unsigned long long *bnnzb = bflops + NB1, *bout = bflops + 2 * NB1;
    // low-cf columns: expand-sort-compress list (kernels_esc.cu), round 0 only
    unsigned long long *esc_flops = bflops + 3 * NB1, *esc_out = esc_flops + 1;
    int *esc_count = counts + 2 * NB1 + 2, *esc_counter = esc_count + 1;
    int32_t *esc_list = nullptr;
    // candidate mode (base.cand_k > 0, kFused): every kernel writes top-max(S, R) candidates and
    // column statistics instead of pruned columns; the ESC kernel has no such epilogue
    const bool candm = mode == kFused && base.cand_k > 0;
    const bool use_esc = c->esc_cf > 0.0 && mode != kPart && !candm &&
                         (product_cf > 0.0 ? product_cf : 1e300) < c->esc_iter_cf;
    if (use_esc) RC(scratch_t(c, "esc_list", (size_t)std::max<int64_t>(n, 1), &esc_list));
    RC(scratch_t(c, "bin_lists", (size_t)NB1 * std::max<int64_t>(n, 1), &lists));
    RC(scratch_t(c, "gcap_col", (size_t)std::max<int64_t>(n, 1), &gcap_col));
    RC(scratch_t(c, "retry_list", (size_t)std::max<int64_t>(n, 1), &retry_list));
    RC(scratch_t(c, "retry_in", (size_t)std::max<int64_t>(n, 1), &retry_in));
    CK(cudaMemsetAsync(err, 0, sizeof(int), c->stream));
    int *rowpart;
    RC(scratch_t(c, "rowpart", (size_t)std::max<int64_t>(pr.A->ncols, 1) * 33, &rowpart));
    CK(launch_rowpart(pr.A->ncols, pr.A->col_ptr, pr.A->row_idx, pr.A->nrows, rowpart, c->stream));
    base.rowpart = rowpart;
    // interleaved (row, value) copy of A for the private family's 8-byte gathers
    int2 *apair;
    RC(scratch_t(c, "apair", (size_t)std::max<int64_t>(pr.A->nnz, 1), &apair));
    CK(launch_pack_pairs(pr.A->nnz, pr.A->row_idx, pr.A->val, apair, c->stream));
    base.apair = apair;
    // locality order of the work lists (MCLX_ORDER=0 turns it off)
    int32_t *colbin = nullptr;
    uint32_t *okey = nullptr;
    int64_t *ohist = nullptr, *ooffs = nullptr;
    void *otmp = nullptr;
    if (c->order_lists) {
        const int64_t nbk = (int64_t)kAllBins << kOrderBits;
        RC(scratch_t(c, "colbin", (size_t)std::max<int64_t>(n, 1), &colbin));
        RC(scratch_t(c, "order_key", (size_t)std::max<int64_t>(n, 1), &okey));
        RC(scratch_t(c, "order_hist", (size_t)nbk, &ohist));
        RC(scratch_t(c, "order_offs", (size_t)nbk + 1, &ooffs));
        RC(scratch(c, "order_scan_tmp", scan_tmp_bytes(nbk), &otmp));
        CK(launch_minhash_key(n, pr.B->col_ptr, pr.B->row_idx, pr.cb, okey, c->stream));
    }


    // split columns (kFused only): big columns as row-range parts, see run_split
    // (the row-range parts address A with 32-bit positions)
    const bool use_split = c->split && mode == kFused && pr.A->ncols > 0 &&
                           pr.A->nnz < ((int64_t)1 << 32) && (!candm || base.pp.kmax <= kCandMax);
    int32_t *split_list = nullptr, *split_P = nullptr;
    int *split_count = nullptr, *col_flag = nullptr;
    if (use_split) {
        RC(scratch_t(c, "split_list", (size_t)std::max<int64_t>(n, 1), &split_list));
        RC(scratch_t(c, "split_P", (size_t)std::max<int64_t>(n, 1), &split_P));
        split_count = counts + 2 * NB1 + 4;
        RC(scratch_t(c, "col_flag", (size_t)std::max<int64_t>(n, 1), &col_flag));
    }

    // Rounds: 0 sizes by the caller's estimate / exact sizes; 1 re-runs overflowed
    // columns with 4x the estimate; 2 with the exact upper bound min(f_j, m), which
    // cannot overflow (load <= 1/2 < the 7/8 fill limit).  Retried columns run in the
    // CTA-shared-table family: a private-family column can also overflow when its output
    // rows crowd into one warp's row range (inputs whose labels carry locality), and a
    // shared table has no such skew.
    int64_t ncls = n;
    const int32_t *cls_list = nullptr;
    const int nrounds = 3;
    int herr = 0;
    for (int round = 0; round < nrounds; round++) {
        // everything but the error flag (bins, counters, retry, ESC, split counts; stats)
        CK(cudaMemsetAsync(counts, 0, sizeof(int) * (2 * NB1 + 1), c->stream));
        CK(cudaMemsetAsync(esc_count, 0, ints_bytes - sizeof(int) * (2 * NB1 + 2) + ulls_bytes,
                           c->stream));
        ClassifyArgs ca;
        memset(&ca, 0, sizeof ca);
        ca.n = ncls;
        ca.cols = cls_list;
        ca.flops = f;
        ca.bcp = pr.B->col_ptr;
        ca.cb = pr.cb;
        ca.est = round < 2 ? est : nullptr;
        ca.exact = round == 0 ? exact : nullptr;
        ca.m = pr.A->nrows;
        ca.alpha = round == 0 ? c->alpha : 4.0f * c->alpha;
        ca.max_load = round == 2 ? 0.5f : c->max_load;
        ca.force_bin = force_bin < 0 ? -1 : force_bin % kFamily;
        // the private family addresses A with 32-bit offsets
        const bool big_a = pr.A->nnz >= ((int64_t)1 << 32);
        ca.force_family = force_bin >= 0 ? force_bin / kFamily : (round > 0 || big_a) ? 1 : c->family;
        ca.list_stride = std::max<int64_t>(n, 1);
        ca.bin_count = counts;
        ca.lists = lists;
        ca.gcap_col = gcap_col;
        ca.bin_flops = bflops;
        ca.bin_nnzb = bnnzb;
        ca.colbin = colbin;
        ca.fp64_terms = c->fp64_terms;
        if (use_esc && round == 0) {
            ca.esc_max = kEscCap;
            ca.esc_cf = c->esc_cf;
            ca.esc_count = esc_count;
            ca.esc_list = esc_list;
            ca.esc_flops = esc_flops;
        }
        if (use_split && round < 2) {
            // the exact round stays in the global bin, which cannot overflow
            ca.split_max = INT64_MAX;  // the global-table variant takes any size
            ca.split_min = c->split_min_need;
            ca.split_part_need = c->split_part_need;
            ca.dense_min_P = c->dense_min_P;
            ca.split_big = c->split_big;
            ca.split_count = split_count;
            ca.split_list = split_list;
            ca.split_P = split_P;
            CK(cudaMemsetAsync(col_flag, 0, sizeof(int) * std::max<int64_t>(n, 1), c->stream));
        }
        CK(launch_classify(ca, c->stream));
        if (colbin)
            CK(launch_order_lists(ncls, cls_list, colbin, okey, ohist, ooffs, otmp, lists,
                                  ca.list_stride, c->stream));
        int hc[2 * kAllBins + 6];
        RC(readback(c, counts, sizeof(int) * kInts, hc));  // sync 1 of the round
        const int nesc = ca.esc_max > 0 ? hc[2 * NB1 + 2] : 0;
        const int nsplit = ca.split_max > 0 ? hc[2 * NB1 + 4] : 0;
        if (nsplit > 0) {
            BinArgs a = base;
            a.acp = pr.A->col_ptr;
            a.arow = pr.A->row_idx;
            a.aval = pr.A->val;
            a.m = pr.A->nrows;
            a.bcp = pr.B->col_ptr;
            a.brow = pr.B->row_idx;
            a.bval = pr.B->val;
            a.cb = pr.cb;
            a.flops = f;
            a.retry_list = retry_list;
            a.retry_count = retry_count;
            a.err_flag = err;
            a.col_flag = col_flag;
            CK(cudaEventRecord(c->bev[2 * kNumBins], c->stream));
            int64_t nitems = 0;
            RC(run_split(c, pr, nsplit, split_list, split_P, a, bout + kNumBins, &nitems, st));
            CK(cudaEventRecord(c->bev[2 * kNumBins + 1], c->stream));
            if (st) {
                float ms = 0.f;
                CK(cudaEventSynchronize(c->bev[2 * kNumBins + 1]));
                CK(cudaEventElapsedTime(&ms, c->bev[2 * kNumBins], c->bev[2 * kNumBins + 1]));
                st->bin_ms[kNumBins] += ms;
                st->split_ms += ms;
                if (round == 0) st->split_cols += nsplit;
                st->split_items += nitems;
            }
        }
        if (nesc > 0) {  // low-cf columns: expand, sort, compress (one CTA per column)
            BinArgs a = base;
            a.acp = pr.A->col_ptr;
            a.arow = pr.A->row_idx;
            a.aval = pr.A->val;
            a.m = pr.A->nrows;
            a.bcp = pr.B->col_ptr;
            a.brow = pr.B->row_idx;
            a.bval = pr.B->val;
            a.cb = pr.cb;
            a.flops = f;
            a.list = esc_list;
            a.count = esc_count;
            a.counter = esc_counter;
            a.err_flag = err;
            a.bin_out = esc_out;
            const int grid = (int)std::min<int64_t>(nesc, (int64_t)std::max(1, esc_occupancy(mode)) * c->sms);
            CK(cudaEventRecord(c->bev[2 * kAllBins], c->stream));
            CK(launch_esc(mode, a, grid, c->stream));
            CK(cudaEventRecord(c->bev[2 * kAllBins + 1], c->stream));
        }
        bool launched[kAllBins] = {};
        for (int bi = kAllBins - 1; bi >= 0; bi--) {
            // heaviest bins first: global, then big shared-memory tables, both families
            const int b = (bi % 2 == 0) ? bi / 2 : kFamily + bi / 2;
            if (hc[b] == 0) continue;
            BinArgs a = base;
            a.acp = pr.A->col_ptr;
            a.arow = pr.A->row_idx;
            a.aval = pr.A->val;
            a.m = pr.A->nrows;
            a.bcp = pr.B->col_ptr;
            a.brow = pr.B->row_idx;
            a.bval = pr.B->val;
            a.cb = pr.cb;
            a.flops = f;
            a.list = lists + (int64_t)b * std::max<int64_t>(n, 1);
            a.count = counts + b;
            a.counter = counters + b;
            a.retry_list = retry_list;
            a.retry_count = retry_count;
            a.err_flag = err;
            a.bin_out = bout + b;
            const int occ = std::max(1, c->occ[mode][b]);
            if (b % kFamily == kNumBins) {
                // fp64 global-memory tables, allocated per chunk of the bin's list so that
                // the live tables stay within c->gbin_budget bytes (R-MAT hubs: C4)
                int32_t *gcap;
                int64_t *gcap64, *goff;
                int *gcount;
                void *tmp;
                RC(scratch_t(c, "gcap", (size_t)hc[b], &gcap));
                RC(scratch_t(c, "gcap64", (size_t)hc[b], &gcap64));
                RC(scratch_t(c, "goff", (size_t)hc[b] + 1, &goff));
                RC(scratch_t(c, "gcount", 2, &gcount));
                RC(scratch(c, "scan_tmp", scan_tmp_bytes(hc[b]), &tmp));
                {   // largest columns first (LPT): homogeneous chunks, hubs start first
                    std::vector<int32_t> hl((size_t)hc[b]);
                    std::vector<int64_t> hfl((size_t)hc[b]);
                    int64_t *gf;
                    RC(scratch_t(c, "gbin_flops", (size_t)hc[b], &gf));
                    CK(launch_gather_i64(hc[b], a.list, f, gf, c->stream));
                    RC(readback(c, a.list, sizeof(int32_t) * hc[b], hl.data()));
                    RC(readback(c, gf, sizeof(int64_t) * hc[b], hfl.data()));
                    std::vector<int> ord((size_t)hc[b]);
                    for (int i = 0; i < hc[b]; i++) ord[i] = i;
                    std::stable_sort(ord.begin(), ord.end(),
                                     [&](int x, int y) { return hfl[x] > hfl[y]; });
                    std::vector<int32_t> sl((size_t)hc[b]);
                    for (int i = 0; i < hc[b]; i++) sl[i] = hl[ord[i]];
                    RC(upload(c, sl.data(), sizeof(int32_t) * hc[b], const_cast<int32_t *>(a.list)));
                }
                CK(launch_global_layout(hc[b], a.list, gcap_col, gcap, gcap64, c->stream));
                CK(launch_scan_i64(gcap64, goff, hc[b], tmp, c->stream));
                std::vector<int64_t> hoff((size_t)hc[b] + 1);
                RC(readback(c, goff, sizeof(int64_t) * (hc[b] + 1), hoff.data()));
                const int64_t slots_budget = std::max<int64_t>(c->gbin_budget / 12, 1 << 20);
                CK(cudaEventRecord(c->bev[2 * b], c->stream));
                for (int i0 = 0; i0 < hc[b];) {
                    int i1 = i0 + 1;
                    while (i1 < hc[b] && hoff[i1 + 1] - hoff[i0] <= slots_budget) i1++;
                    const int64_t chunk = hoff[i1] - hoff[i0];
                    int *gkeys;
                    double *gvals;
                    RC(scratch_t(c, "gkeys", (size_t)chunk, &gkeys));
                    RC(scratch_t(c, "gvals", (size_t)chunk, &gvals));
                    const int cnt_chunk = i1 - i0;
                    RC(upload(c, &cnt_chunk, sizeof(int), gcount));
                    CK(cudaMemsetAsync(gcount + 1, 0, sizeof(int), c->stream));
                    BinArgs ag = a;
                    ag.list = a.list + i0;
                    ag.count = gcount;
                    ag.counter = gcount + 1;
                    ag.goff = goff + i0;
                    ag.gcap = gcap + i0;
                    ag.gkeys = gkeys - hoff[i0];   // goff[idx] - hoff[i0] indexes the chunk
                    ag.gvals = gvals - hoff[i0];
                    const int grid = (int)std::min<int64_t>(cnt_chunk, (int64_t)occ * c->sms);
                    CK(launch_bin(mode, b, ag, grid, c->stream));
                    if (i1 < hc[b]) CK(cudaStreamSynchronize(c->stream));  // scratch reuse
                    i0 = i1;
                }
                CK(cudaEventRecord(c->bev[2 * b + 1], c->stream));
                launched[b] = true;
                continue;
            }
            const int grid = (int)std::min<int64_t>(hc[b], (int64_t)occ * c->sms);
            CK(cudaEventRecord(c->bev[2 * b], c->stream));
            CK(launch_bin(mode, b, a, grid, c->stream));
            CK(cudaEventRecord(c->bev[2 * b + 1], c->stream));
            launched[b] = true;
        }
        // sync 2 of the round: retries, the error flag and (with stats) the bin counters
        std::vector<unsigned char> hm(ints_bytes + ulls_bytes);
        RC(readback(c, meta, st ? ints_bytes + ulls_bytes : ints_bytes, hm.data()));
        const int *hi = reinterpret_cast<const int *>(hm.data());
        const unsigned long long *hf = reinterpret_cast<const unsigned long long *>(hm.data() + ints_bytes);
        const int nretry = hi[2 * NB1];
        herr = hi[2 * NB1 + 1];
        if (st) {
            for (int b = 0; b < NB1; b++) {
                if (round == 0) {
                    st->bin_cols[b % kFamily] += hc[b];
                    st->bin_flops[b % kFamily] += (int64_t)hf[b];
                    st->bin_nnzb[b % kFamily] += (int64_t)hf[NB1 + b];
                }
                st->bin_out[b % kFamily] += (int64_t)hf[2 * NB1 + b];
                if (!launched[b]) continue;
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, c->bev[2 * b], c->bev[2 * b + 1]));
                st->bin_ms[b % kFamily] += ms;
            }
            if (round == 0) st->bin_cols[kNumBins] += nsplit;  // split columns: with the global bin
            if (nesc > 0) {
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, c->bev[2 * kAllBins], c->bev[2 * kAllBins + 1]));
                st->esc_cols += nesc;
                st->esc_flops += (int64_t)hf[3 * NB1];
                st->esc_out += (int64_t)hf[3 * NB1 + 1];
                st->esc_ms += ms;
            }
        }
        if (nretry == 0) break;
        if (round == nrounds - 1)
            return fail(c, MCL_ERR_INTERNAL, "hash table overflow after exact re-binning");
        if (st) st->retries += nretry;
        CK(cudaMemcpyAsync(retry_in, retry_list, sizeof(int32_t) * nretry, cudaMemcpyDeviceToDevice,
                           c->stream));
        ncls = nretry;
        cls_list = retry_in;
    }
    if (herr) return fail(c, MCL_ERR_INTERNAL, "device consistency check failed (code %d)", herr);
    return MCL_OK;
}

int validate_product(mcl_ctx *c, const mcl_csc_t *A, const mcl_csc_t *B, int64_t b, int64_t e) {
    RC(check_csc(c, A, "A"));
    RC(check_csc(c, B, "B"));
    if (A->ncols != B->nrows)
        return fail(c, MCL_ERR_DIM, "A.ncols (%lld) != B.nrows (%lld)", (long long)A->ncols,
                    (long long)B->nrows);
    if (b < 0 || e > B->ncols || b > e) return fail(c, MCL_ERR_DIM, "bad column range [%lld,%lld)",
                                                     (long long)b, (long long)e);
    return MCL_OK;
}

// Exact symbolic sizes of a product's output columns (sized by a Cohen estimate).
int symbolic_sizes(mcl_ctx *c, const Prod &pr, const int64_t *f, const float *est, int force_bin,
                   int64_t *nnz_out, mcl_stats_t *st) {
    CK(cudaMemsetAsync(nnz_out, 0, sizeof(int64_t) * std::max<int64_t>(pr.n, 1), c->stream));
    BinArgs base;
    memset(&base, 0, sizeof base);
    base.sym_nnz = nnz_out;
    return run_bins(c, kSym, pr, f, est, nullptr, force_bin, base, st);
}

int spgemm_impl(mcl_ctx *c, const mcl_csc_t *A, const mcl_csc_t *B, int64_t cb, int64_t ce,
                const mcl_params_t *pin, mcl_csc_t *C, mcl_stats_t *st) {
    mcl_params_t p;
    if (pin) p = *pin;
    else mcl_params_default(&p);
    RC(check_params(c, &p));
    RC(validate_product(c, A, B, cb, ce));
    const int64_t n = ce - cb;
    Prod pr{A, B, cb, n};
    init_stats(st);
    const int64_t launches0 = g_launches;
    CK(cudaEventRecord(c->ev[0], c->stream));
    int64_t *f, *nnzc;
    float *est;
    void *tmp;
    unsigned long long *tot;
    RC(scratch_t(c, "flops", (size_t)std::max<int64_t>(n, 1), &f));
    RC(scratch_t(c, "est", (size_t)std::max<int64_t>(n, 1), &est));
    RC(scratch_t(c, "nnz_sym", (size_t)std::max<int64_t>(n, 1), &nnzc));
    RC(scratch_t(c, "tot", 4, &tot));
    RC(scratch(c, "scan_tmp", scan_tmp_bytes(n + 1), &tmp));
    CK(launch_flops(n, A->col_ptr, B->col_ptr, B->row_idx, cb, f, c->stream));
    CK(cudaEventRecord(c->ev[1], c->stream));
    RC(cohen(c, pr, p.est_keys, p.seed, est, nullptr));
    CK(cudaEventRecord(c->ev[2], c->stream));
    // Output sizing.  Capacity mode (default when it fits c->cap_budget): every column gets
    // an upper-bound slot of min(f_j, m) entries, the numeric pass records the true counts
    // and a scan + copy compacts the result -- no symbolic hashing pass.  Otherwise the
    // exact symbolic pass sizes the CSC first.
    int64_t *capcp = nullptr, *ccnt = nullptr;
    int32_t *crow = nullptr;
    float *cval = nullptr;
    bool capacity = false;
    if (!getenv("MCLX_EXACT_SYMBOLIC")) {
        RC(scratch_t(c, "cap_cp", (size_t)n + 1, &capcp));
        RC(scratch_t(c, "cap_cnt", (size_t)std::max<int64_t>(n, 1), &ccnt));
        CK(launch_kcap(n, f, A->nrows, INT32_MAX, ccnt, c->stream));
        CK(launch_scan_i64(ccnt, capcp, n, tmp, c->stream));
        int64_t tcap = 0;
        RC(readback(c, capcp + n, sizeof(int64_t), &tcap));
        if (tcap * 8 <= c->cap_budget) {
            capacity = true;
            RC(scratch_t(c, "cap_row", (size_t)std::max<int64_t>(tcap, 1), &crow));
            RC(scratch_t(c, "cap_val", (size_t)std::max<int64_t>(tcap, 1), &cval));
        }
    }
    if (!capacity) RC(symbolic_sizes(c, pr, f, est, p.force_bin, nnzc, nullptr));
    CK(cudaEventRecord(c->ev[3], c->stream));
    C->col_ptr = nullptr;
    mcl_csc_t out;
    zero_csc(&out);
    out.col_ptr = (int64_t *)dalloc(c, (size_t)(n + 1) * sizeof(int64_t));
    if (!out.col_ptr) return fail(c, MCL_ERR_OOM, "cannot allocate col_ptr");
    int rc = MCL_OK;
    do {
        cudaError_t e;
        int64_t nnz = 0;
        out.nrows = A->nrows;
        out.ncols = n;
        out.row0 = A->row0;
        out.col0 = B->col0 + cb;
        out.n_global = A->n_global ? A->n_global : A->nrows;
        BinArgs base;
        memset(&base, 0, sizeof base);
        if (capacity) {
            base.c_cp = capcp;
            base.c_row = crow;
            base.c_val = cval;
            base.c_cnt = ccnt;
            if ((rc = run_bins(c, kNum, pr, f, est, nullptr, p.force_bin, base, st)) != MCL_OK) break;
            e = launch_scan_i64(ccnt, out.col_ptr, n, tmp, c->stream);
            if (e != cudaSuccess) { rc = fail(c, MCL_ERR_CUDA, "scan: %s", cudaGetErrorString(e)); break; }
            if ((rc = readback(c, out.col_ptr + n, sizeof(int64_t), &nnz)) != MCL_OK) break;
            if ((rc = alloc_rows_vals(c, &out, nnz)) != MCL_OK) break;
            e = launch_copy_cols(n, ccnt, capcp, crow, cval, out.col_ptr, out.row_idx, out.val, c->stream);
            if (e != cudaSuccess) { rc = fail(c, MCL_ERR_CUDA, "copy: %s", cudaGetErrorString(e)); break; }
        } else {
            e = launch_scan_i64(nnzc, out.col_ptr, n, tmp, c->stream);
            if (e != cudaSuccess) { rc = fail(c, MCL_ERR_CUDA, "scan: %s", cudaGetErrorString(e)); break; }
            if ((rc = readback(c, out.col_ptr + n, sizeof(int64_t), &nnz)) != MCL_OK) break;
            if ((rc = alloc_rows_vals(c, &out, nnz)) != MCL_OK) break;
            base.c_cp = out.col_ptr;
            base.c_row = out.row_idx;
            base.c_val = out.val;
            if ((rc = run_bins(c, kNum, pr, f, nullptr, nnzc, p.force_bin, base, st)) != MCL_OK) break;
        }
        CK(cudaEventRecord(c->ev[4], c->stream));
        e = launch_reduce_i64(f, n, tot, c->stream);
        if (e != cudaSuccess) { rc = fail(c, MCL_ERR_CUDA, "reduce: %s", cudaGetErrorString(e)); break; }
        double est_tot = 0;
        double *dsum = (double *)(tot + 1);
        e = launch_reduce_f32(est, n, dsum, c->stream);
        if (e != cudaSuccess) { rc = fail(c, MCL_ERR_CUDA, "reduce: %s", cudaGetErrorString(e)); break; }
        unsigned long long hv[2];
        if ((rc = readback(c, tot, 2 * sizeof(unsigned long long), hv)) != MCL_OK) break;
        memcpy(&est_tot, &hv[1], sizeof(double));
        if (st) {
            st->flops = (int64_t)hv[0];
            st->nnz_in = A->nnz;
            st->nnz_unpruned = nnz;
            st->nnz_out = nnz;
            st->est_nnz = est_tot;
            st->cf = nnz > 0 ? (double)hv[0] / (double)nnz : 0.0;
            st->estimator_used = capacity ? 3 : 1;
            st->ms[0] = elapsed(c, 0, 1);
            st->ms[1] = elapsed(c, 1, 2);
            st->ms[2] = elapsed(c, 2, 3);
            st->ms[3] = elapsed(c, 3, 4);
            st->ms[6] = elapsed(c, 0, 4);
            st->peak_bytes = (int64_t)c->peak;
            st->launches = g_launches - launches0;
        }
        *C = out;
        return MCL_OK;
    } while (0);
    dfree(c, out.col_ptr, 0);
    dfree(c, out.row_idx, 0);
    dfree(c, out.val, 0);
    zero_csc(C);
    return rc;
}

// Scan per-column counts into a fresh CSC and copy the staged columns into it.
int assemble(mcl_ctx *c, int64_t nrows, int64_t n, const int64_t *cnt, const int64_t *soff,
             const int32_t *srow, const float *sval, mcl_csc_t *out, int64_t *nnz_out) {
    void *tmp;
    RC(scratch(c, "scan_tmp", scan_tmp_bytes(n + 1), &tmp));
    zero_csc(out);
    out->col_ptr = (int64_t *)dalloc(c, (size_t)(n + 1) * sizeof(int64_t));
    if (!out->col_ptr) return fail(c, MCL_ERR_OOM, "cannot allocate col_ptr");
    CK(launch_scan_i64(cnt, out->col_ptr, n, tmp, c->stream));
    int64_t nnz = 0;
    RC(readback(c, out->col_ptr + n, sizeof(int64_t), &nnz));
    int rc = alloc_rows_vals(c, out, nnz);
    if (rc != MCL_OK) {
        dfree(c, out->col_ptr, 0);
        dfree(c, out->row_idx, 0);
        dfree(c, out->val, 0);
        zero_csc(out);
        return rc;
    }
    out->nrows = nrows;
    out->ncols = n;
    out->n_global = nrows;
    CK(launch_copy_cols(n, cnt, soff, srow, sval, out->col_ptr, out->row_idx, out->val, c->stream));
    *nnz_out = nnz;
    return MCL_OK;
}

// Phase planner (§II: HipMCL forms the product "in phases" of column batches;
// P:575-579 / P:594-595 §V: the estimate sizes them; reading Q15): cut the columns [0, n)
// into h batches of near-equal estimated bytes (bytes_dev: int64 [n], device) so that one
// batch fits `budget` bytes; h = ceil(total / budget), or c->force_phases.  bounds receives
// h + 1 column boundaries.  Two small read-backs (the total, the h - 1 cuts).
int plan_phases(mcl_ctx *c, const int64_t *bytes_dev, int64_t n,
                const std::function<double(double)> &budget_of, std::vector<int64_t> &bounds,
                int64_t *total_out) {
    bounds.assign(1, 0);
    if (n <= 0) {
        bounds.push_back(0);
        if (total_out) *total_out = 0;
        return MCL_OK;
    }
    int64_t *prefix, *cut;
    void *tmp;
    RC(scratch_t(c, "phase_prefix", (size_t)n + 1, &prefix));
    RC(scratch(c, "phase_scan_tmp", scan_tmp_bytes(n + 1), &tmp));
    CK(launch_scan_i64(bytes_dev, prefix, n, tmp, c->stream));
    int64_t total = 0;
    RC(readback(c, prefix + n, sizeof(int64_t), &total));
    if (total_out) *total_out = total;
    int64_t h = c->force_phases > 0
                    ? c->force_phases
                    : std::max<int64_t>(1, (int64_t)std::ceil((double)total / budget_of((double)total)));
    h = std::min<int64_t>(h, std::min<int64_t>(n, 4096));
    if (h > 1) {
        RC(scratch_t(c, "phase_cut", (size_t)h, &cut));
        CK(launch_phase_cuts(prefix, n, (int)h, cut, c->stream));
        std::vector<int64_t> hc((size_t)h - 1);
        RC(readback(c, cut, sizeof(int64_t) * (h - 1), hc.data()));
        for (int64_t v : hc)
            if (v > bounds.back() && v < n) bounds.push_back(v);
    }
    bounds.push_back(n);
    return MCL_OK;
}

// bytes a phase may use: MCLX_PHASE_BUDGET_MB, else mem_safety x the device's free memory.
// need (bytes the caller is about to compare with the budget; < 0 unknown): cudaMemGetInfo is
// a driver round trip of ~5 ms on these boxes (50+ ms at times) during which the GPU sits idle,
// so the free memory last seen is reused while the need stays within half of its budget.
double phase_budget(mcl_ctx *c, double mem_safety, double need = -1.0) {
    if (c->phase_budget > 0) return (double)c->phase_budget;
    if (need >= 0.0 && c->free_seen > 0 && need <= 0.5 * mem_safety * (double)c->free_seen)
        return std::max(1.0, mem_safety * (double)c->free_seen);
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
        cudaGetLastError();
        return 1e18;
    }
    c->free_seen = fr;
    return std::max(1.0, mem_safety * (double)fr);
}

// out = [pieces[0] | pieces[1] | ...] (column concatenation of the phase outputs; the
// pieces share nrows / row0 / n_global).  Pieces are not freed here.
int concat_cols(mcl_ctx *c, const std::vector<mcl_csc_t> &pieces, mcl_csc_t *out) {
    zero_csc(out);
    int64_t n = 0, nnz = 0;
    for (auto &q : pieces) {
        n += q.ncols;
        nnz += q.nnz;
    }
    out->col_ptr = (int64_t *)dalloc(c, (size_t)(n + 1) * sizeof(int64_t));
    if (!out->col_ptr) return fail(c, MCL_ERR_OOM, "cannot allocate col_ptr");
    int rc = alloc_rows_vals(c, out, nnz);
    if (rc != MCL_OK) {
        free_csc(c, out);
        return rc;
    }
    int64_t coff = 0, off = 0;
    for (auto &q : pieces) {
        cudaError_t e = launch_offset_colptr(q.ncols + 1, q.col_ptr, off, out->col_ptr + coff, c->stream);
        if (e == cudaSuccess && q.nnz) {
            e = cudaMemcpyAsync(out->row_idx + off, q.row_idx, sizeof(int32_t) * q.nnz,
                                cudaMemcpyDeviceToDevice, c->stream);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(out->val + off, q.val, sizeof(float) * q.nnz,
                                    cudaMemcpyDeviceToDevice, c->stream);
        }
        if (e != cudaSuccess) {
            free_csc(c, out);
            return fail(c, MCL_ERR_CUDA, "concat: %s", cudaGetErrorString(e));
        }
        coff += q.ncols;
        off += q.nnz;
    }
    if (!pieces.empty()) {
        out->nrows = pieces[0].nrows;
        out->row0 = pieces[0].row0;
        out->col0 = pieces[0].col0;
        out->n_global = pieces[0].n_global;
    }
    out->ncols = n;
    out->nnz = nnz;
    return MCL_OK;
}

// accumulate the statistics of one phase into the call's
void add_stats(mcl_stats_t *st, const mcl_stats_t &q) {
    st->flops += q.flops;
    st->nnz_out += q.nnz_out;
    st->retries += q.retries;
    st->chaos = std::max(st->chaos, q.chaos);
    if (q.est_nnz >= 0) st->est_nnz = (st->est_nnz < 0 ? 0 : st->est_nnz) + q.est_nnz;
    for (int b = 0; b <= kNumBins; b++) {
        st->bin_cols[b] += q.bin_cols[b];
        st->bin_flops[b] += q.bin_flops[b];
        st->bin_ms[b] += q.bin_ms[b];
        st->bin_nnzb[b] += q.bin_nnzb[b];
        st->bin_out[b] += q.bin_out[b];
    }
    for (int i = 0; i < 8; i++)
        if (q.ms[i] >= 0) st->ms[i] = (st->ms[i] < 0 ? 0.f : st->ms[i]) + q.ms[i];
    st->split_cols += q.split_cols;
    st->split_items += q.split_items;
    st->split_ms += q.split_ms;
    for (int v = 0; v < 3; v++) {
        st->split_vcols[v] += q.split_vcols[v];
        st->split_vms[v] += q.split_vms[v];
    }
    st->esc_cols += q.esc_cols;
    st->esc_flops += q.esc_flops;
    st->esc_out += q.esc_out;
    st->esc_ms += q.esc_ms;
    st->peak_bytes = std::max(st->peak_bytes, q.peak_bytes);
    st->launches += q.launches;
    st->estimator_used = q.estimator_used;
}

int merge_impl(mcl_ctx_t c, int32_t L, const mcl_csc_t *lists, mcl_csc_t *out) {
    const int64_t m = lists[0].nrows, n = lists[0].ncols;
    int64_t tot = 0;
    for (int l = 0; l < L; l++) {
        RC(check_csc(c, &lists[l], "list"));
        if (lists[l].nrows != m || lists[l].ncols != n)
            return fail(c, MCL_ERR_DIM, "merge: list %d has a different shape", l);
        tot += lists[l].nnz;
    }
    // X = [P_0 | ... | P_{L-1}] (m x L*n) and E = stacked identities (L*n x n): X*E = sum_l P_l
    int64_t *xcp, *ecp;
    int32_t *xrow, *erow;
    float *xval, *eval;
    RC(scratch_t(c, "merge_xcp", (size_t)(L * n + 1), &xcp));
    RC(scratch_t(c, "merge_xrow", (size_t)std::max<int64_t>(tot, 1), &xrow));
    RC(scratch_t(c, "merge_xval", (size_t)std::max<int64_t>(tot, 1), &xval));
    RC(scratch_t(c, "merge_ecp", (size_t)(n + 1), &ecp));
    RC(scratch_t(c, "merge_erow", (size_t)std::max<int64_t>(L * n, 1), &erow));
    RC(scratch_t(c, "merge_eval", (size_t)std::max<int64_t>(L * n, 1), &eval));
    int64_t off = 0;
    for (int l = 0; l < L; l++) {
        CK(launch_offset_colptr(n + 1, lists[l].col_ptr, off, xcp + (int64_t)l * n, c->stream));
        if (lists[l].nnz) {
            CK(cudaMemcpyAsync(xrow + off, lists[l].row_idx, sizeof(int32_t) * lists[l].nnz,
                               cudaMemcpyDeviceToDevice, c->stream));
            CK(cudaMemcpyAsync(xval + off, lists[l].val, sizeof(float) * lists[l].nnz,
                               cudaMemcpyDeviceToDevice, c->stream));
        }
        off += lists[l].nnz;
    }
    CK(launch_stack_identity(n, L, ecp, erow, eval, c->stream));
    mcl_csc_t X, E;
    zero_csc(&X);
    zero_csc(&E);
    X.nrows = m;
    X.ncols = (int64_t)L * n;
    X.nnz = tot;
    X.row0 = lists[0].row0;
    X.n_global = lists[0].n_global;
    X.col_ptr = xcp;
    X.row_idx = xrow;
    X.val = xval;
    E.nrows = (int64_t)L * n;
    E.ncols = n;
    E.nnz = (int64_t)L * n;
    E.col_ptr = ecp;
    E.row_idx = erow;
    E.val = eval;
    mcl_params_t p;
    mcl_params_default(&p);
    p.estimator = 1;
    RC(spgemm_impl(c, &X, &E, 0, n, &p, out, nullptr));
    out->row0 = lists[0].row0;
    out->col0 = lists[0].col0;
    out->n_global = lists[0].n_global;
    return MCL_OK;
}



#define NC(call)                                                                              \
    do {                                                                                      \
        ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess)                                                                \
            return fail(c, MCL_ERR_NCCL, "%s:%d %s: %s", __FILE__, __LINE__, #call,         \
                        ncclGetErrorString(r_));                                              \
    } while (0)

// Stripe / panel boundaries of a 1D cut of [0, n) into `parts` near-equal ranges.  With
// s = lcm(pr, pc) inner panels every panel lies inside one row stripe and one column
// stripe (the boundaries coincide exactly, q*n/s = c*n/pc for q = c*s/pc).
int64_t cut(int64_t n, int parts, int k) { return (int64_t)((__int128)k * n / parts); }
int gcd_i(int a, int b) { return b ? gcd_i(b, a % b) : a; }

// Alg. 2 lines 5-8: after pushing list i (1-based), merge nmerges + 1 lists,
// nmerges = the number of times i halves while even
int alg2_nmerges(int64_t i) {
    int nm = 0;
    while (i % 2 == 0 && i != 0) {
        nm++;
        i /= 2;
    }
    return nm;
}

// Candidate mode of iterate_range_impl: column statistics of the unpruned product (device
// arrays of the range's n columns: entries, entries >= theta, their fp64 mass).
struct CandOut {
    int64_t *nnz, *m;
    double *s;
    // filled by iterate_range_impl: the candidates stay in its staging slots -- column j's at
    // [start[j], start[j] + count[j]) of (row, val) -- plus their total and the unpruned total
    const int64_t *start = nullptr, *count = nullptr;
    const int32_t *row = nullptr;
    const float *val = nullptr;
    int64_t total = 0, unpruned = 0;
};

// Distributed prune / select / recover / inflate of a block column set whose columns are
// split over the ranks of `comm` (the column communicator; nullptr = whole columns).
// pre: C holds only each row block's top-max(S, R) candidates (iterate_range_impl's
// candidate mode) and pre the statistics of the unpruned block columns.  Exact for every
// branch: the kept set is the column's top-K (K <= max(S, R)) or its entries >= theta when
// there are at most S of them, and both lie among the row blocks' top-max(S, R).
int dist_prune(mcl_ctx *c, const mcl_csc_t *C, ncclComm_t comm, const PruneParams &pp,
               mcl_csc_t *out, float *chaos_out, const CandOut *pre = nullptr,
               const int64_t *ccnt = nullptr) {
    const int64_t n = C->ncols;
    const int64_t n1 = std::max<int64_t>(n, 1);
    const int grid = (int)std::min<int64_t>(n1, (int64_t)c->sms * 8);
    int64_t *nnz, *m, *K, *kcnt, *scnt;
    double *sm, *sums;
    int8_t *mode;
    int32_t *rem, *done, *rowcut;
    uint32_t *vpre, *rpre;
    unsigned *hist;
    float *cmax;
    void *tmp;
    RC(scratch_t(c, "dp_nnz", 3 * n1, &nnz));  // nnz | m | kcnt
    m = nnz + n1;
    kcnt = nnz + 2 * n1;
    RC(scratch_t(c, "dp_K", n1, &K));
    RC(scratch_t(c, "dp_sm", n1, &sm));
    RC(scratch_t(c, "dp_sums", 4 * n1, &sums));
    RC(scratch_t(c, "dp_mode", n1, &mode));
    RC(scratch_t(c, "dp_i32", 3 * n1, &rem));
    done = rem + n1;
    rowcut = rem + 2 * n1;
    RC(scratch_t(c, "dp_pre", 2 * n1, &vpre));
    rpre = vpre + n1;
    int64_t *selflag, *selpos;
    int32_t *sel;
    unsigned long long *undone;
    RC(scratch_t(c, "dp_selflag", 2 * n1 + 1, &selflag));
    selpos = selflag + n1;
    RC(scratch_t(c, "dp_sel", n1, &sel));
    RC(scratch_t(c, "dp_undone", 2, &undone));
    RC(scratch_t(c, "dp_scnt", n1, &scnt));  // (not "scnt": the candidates' counts may live there)
    RC(scratch_t(c, "dp_chaos_max", 4, &cmax));
    RC(scratch(c, "scan_tmp", scan_tmp_bytes(n + 1), &tmp));
    CK(cudaEventRecord(c->pev[0], c->stream));
    if (pre) {  // C holds candidates: the statistics of the unpruned columns come with them
        if (n > 0) {
            CK(cudaMemcpyAsync(nnz, pre->nnz, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, c->stream));
            CK(cudaMemcpyAsync(m, pre->m, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, c->stream));
            CK(cudaMemcpyAsync(sm, pre->s, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
        }
    } else {
        CK(launch_dp_stats(n, C->col_ptr, C->val, pp.theta, nnz, m, sm, grid, c->stream));
    }
    if (comm) {
        NC(ncclGroupStart());
        NC(ncclAllReduce(nnz, nnz, 2 * n1, ncclInt64, ncclSum, comm, c->stream));
        NC(ncclAllReduce(sm, sm, n1, ncclFloat64, ncclSum, comm, c->stream));
        NC(ncclGroupEnd());
    }
    CK(cudaEventRecord(c->pev[1], c->stream));
    CK(launch_dp_branch(n, nnz, m, sm, pp, K, mode, rem, vpre, rowcut, c->stream));
    CK(cudaMemsetAsync(done, 0, sizeof(int32_t) * n1, c->stream));
    CK(cudaMemsetAsync(rpre, 0, sizeof(uint32_t) * n1, c->stream));
    // exact global top-K cut of the select columns (same list, same order on every rank)
    CK(launch_dp_sellist(n, mode, selflag, selpos, sel, tmp, c->stream));
    int64_t nsel = 0;
    if (n > 0) {
        int64_t last[2];
        RC(readback(c, selpos + n - 1, sizeof(int64_t), &last[0]));
        RC(readback(c, selflag + n - 1, sizeof(int64_t), &last[1]));
        nsel = last[0] + last[1];
    }
    // candidate columns hold <= max(S, R) entries per rank, so every global digit count fits
    // 16 bits: two bins per 32-bit word halve the histogram all-reduces
    int nranks = 1;
    if (comm && ncclCommCount(comm, &nranks) != ncclSuccess) nranks = 1 << 20;
    const int packed = pre && (int64_t)pp.kmax * nranks < 65536 ? 1 : 0;
    const int hw = packed ? 128 : 256;
    if (nsel > 0) {
        RC(scratch_t(c, "dp_hist", 256 * (size_t)nsel, &hist));
        const int hgrid = (int)std::min<int64_t>(nsel, (int64_t)c->sms * 8);
        for (int pass = 0; pass < 8; pass++) {
            if (pass == 4) {  // ties at the cut need the row passes only if some column is open
                unsigned long long open = 0;
                CK(launch_dp_undone(nsel, sel, done, undone, c->stream));
                RC(readback(c, undone, sizeof open, &open));
                if (open == 0) break;
            }
            CK(launch_dp_hist(nsel, sel, C->col_ptr, C->row_idx, C->val, C->row0, mode, vpre, rpre,
                              done, pass, hist, hgrid, c->stream, packed, ccnt));
            if (comm) NC(ncclAllReduce(hist, hist, hw * nsel, ncclUint32, ncclSum, comm, c->stream));
            CK(launch_dp_digit(nsel, sel, hist, pass, vpre, rpre, rem, done, rowcut, c->stream, packed));
        }
    }
    CK(cudaEventRecord(c->pev[2], c->stream));
    CK(launch_dp_keepstats(n, C->col_ptr, C->row_idx, C->val, C->row0, mode, vpre, rowcut, pp, kcnt,
                           sums, grid, c->stream, ccnt));
    // the local kept counts lay out the output directly (kcnt is all-reduced below)
    int64_t *lcnt;
    RC(scratch_t(c, "dp_lcnt", n1, &lcnt));
    if (n > 0)
        CK(cudaMemcpyAsync(lcnt, kcnt, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, c->stream));
    if (comm) {
        NC(ncclGroupStart());
        NC(ncclAllReduce(kcnt, kcnt, n1, ncclInt64, ncclSum, comm, c->stream));
        NC(ncclAllReduce(sums, sums, n1, ncclFloat64, ncclSum, comm, c->stream));
        NC(ncclAllReduce(sums + n1, sums + n1, n1, ncclFloat64, ncclMax, comm, c->stream));
        NC(ncclAllReduce(sums + 2 * n1, sums + 2 * n1, 2 * n1, ncclFloat64, ncclSum, comm,
                         c->stream));
        NC(ncclGroupEnd());
    }
    CK(cudaEventRecord(c->pev[3], c->stream));
    // the kept entries go straight to the output CSC (col_ptr = scan of the local counts)
    mcl_csc_t o;
    zero_csc(&o);
    OutGuard guard(c, &o);
    o.col_ptr = (int64_t *)dalloc(c, (size_t)(n + 1) * sizeof(int64_t));
    if (!o.col_ptr) return fail(c, MCL_ERR_OOM, "cannot allocate col_ptr");
    CK(launch_scan_i64(lcnt, o.col_ptr, n, tmp, c->stream));
    int64_t nnz_out = 0;
    RC(readback(c, o.col_ptr + n, sizeof(int64_t), &nnz_out));
    RC(alloc_rows_vals(c, &o, nnz_out));
    CK(cudaMemsetAsync(cmax, 0, sizeof(float), c->stream));
    CK(launch_dp_write(n, C->col_ptr, C->row_idx, C->val, C->row0, mode, vpre, rowcut, pp, sums,
                       kcnt, o.col_ptr, o.row_idx, o.val, scnt, nullptr, cmax, grid, c->stream, ccnt));
    o.nrows = C->nrows;
    o.ncols = n;
    o.row0 = C->row0;
    o.col0 = C->col0;
    o.n_global = C->n_global;
    CK(cudaEventRecord(c->pev[4], c->stream));
    float h = 0.f;
    RC(readback(c, cmax, sizeof(float), &h));
    *chaos_out = h;
    *out = o;
    guard.release();
    return MCL_OK;
}

}  // namespace

// ====================================================================== public API
extern "C" {

int mcl_version(void) { return MCLX_VERSION; }

void mcl_params_default(mcl_params_t *p) {
    if (!p) return;
    memset(p, 0, sizeof *p);
    p->inflation = 2.0;
    p->prune_threshold = 1e-4;
    p->select_k = 1100;
    p->recover_k = 1400;
    p->recover_pct = 0.9;
    p->chaos_eps = 1e-3;
    p->est_keys = 10;
    p->est_cf_threshold = 2.0;
    p->seed = 0x5eed;
    p->mem_safety = 0.9;
    p->estimator = 0;
    p->force_bin = -1;
}

int mcl_ctx_create(mcl_ctx_t *out, int device, void *stream, mcl_alloc_fn alloc,
                   mcl_free_fn free_fn, void *alloc_state) {
    if (!out) return MCL_ERR_INVALID_ARG;
    *out = nullptr;
    if ((alloc == nullptr) != (free_fn == nullptr)) return MCL_ERR_INVALID_ARG;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
        cudaGetLastError();
        return MCL_ERR_CUDA;
    }
    if (!(prop.major == 10 && prop.minor == 0)) return MCL_ERR_UNSUPPORTED_DEVICE;
    if (cudaSetDevice(device) != cudaSuccess) return MCL_ERR_CUDA;
    mcl_ctx *c = new mcl_ctx();
    c->device = device;
    c->stream = (cudaStream_t)stream;
    c->alloc = alloc;
    c->free_fn = free_fn;
    c->state = alloc_state;
    c->sms = prop.multiProcessorCount;
    g_sms = c->sms;
    if (const char *e = getenv("MCLX_ALPHA")) c->alpha = (float)atof(e);
    if (const char *e = getenv("MCLX_MAX_LOAD")) c->max_load = (float)atof(e);
    if (const char *e = getenv("MCLX_ORDER")) c->order_lists = atoi(e) != 0;
    if (const char *e = getenv("MCLX_SPLIT")) c->split = atoi(e) != 0;
    if (const char *e = getenv("MCLX_SPLIT_BUDGET_MB")) c->split_budget = (int64_t)atoll(e) << 20;
    if (const char *e = getenv("MCLX_SPLIT_MIN_NEED")) c->split_min_need = atoll(e);
    if (const char *e = getenv("MCLX_FP64_TERMS")) c->fp64_terms = atoll(e);
    if (const char *e = getenv("MCLX_CAP_BUDGET_MB")) c->cap_budget = (int64_t)atoll(e) << 20;
    if (const char *e = getenv("MCLX_SPLIT_PRIVATE")) c->split_private = atoi(e) != 0;
    if (const char *e = getenv("MCLX_SPLIT_PART_NEED"))
        c->split_part_need = std::max<int64_t>(16, std::min<int64_t>(kPartNeed, atoll(e)));
    if (const char *e = getenv("MCLX_GBIN_BUDGET_MB")) c->gbin_budget = (int64_t)atoll(e) << 20;
    if (const char *e = getenv("MCLX_VALIDATE")) c->validate = atoi(e) != 0;
    if (const char *e = getenv("MCLX_FAMILY")) c->family = atoi(e);
    if (const char *e = getenv("MCLX_SPLIT_CAND")) c->split_cand = atoi(e) != 0;
    if (const char *e = getenv("MCLX_SPLIT_BIG")) c->split_big = atoi(e) != 0;
    if (const char *e = getenv("MCLX_DENSE_MIN_P")) c->dense_min_P = std::max(1, std::min(64, atoi(e)));
    if (const char *e = getenv("MCLX_ESC_CF")) c->esc_cf = atof(e);
    if (const char *e = getenv("MCLX_ESC_ITER_CF")) c->esc_iter_cf = atof(e);
    if (const char *e = getenv("MCLX_PHASES")) c->force_phases = atoi(e);
    if (const char *e = getenv("MCLX_PHASE_BUDGET_MB")) c->phase_budget = (int64_t)atoll(e) << 20;
    if (ensure_pin(c, &c->pin, &c->pin_bytes, kPinBytes) != MCL_OK ||
        ensure_pin(c, &c->pin_up, &c->pin_up_bytes, kPinBytes) != MCL_OK ||
        cudaEventCreateWithFlags(&c->up_ev, cudaEventDisableTiming) != cudaSuccess) {
        mcl_ctx_destroy(c);
        return MCL_ERR_CUDA;
    }
    for (int i = 0; i < 8; i++) cudaEventCreate(&c->ev[i]);
    for (int i = 0; i < 2 * kAllBins + 2; i++) cudaEventCreate(&c->bev[i]);
    for (int i = 0; i < 6; i++) cudaEventCreate(&c->pev[i]);
    for (int i = 0; i < 3; i++) cudaEventCreate(&c->sev[i]);
    for (int i = 0; i < 2; i++) cudaEventCreate(&c->vev[i]);
    for (int m = 0; m < 3; m++)
        for (int b = 0; b < kAllBins; b++) c->occ[m][b] = bin_occupancy(m, b);
    if (cudaGetLastError() != cudaSuccess) {
        mcl_ctx_destroy(c);
        return MCL_ERR_CUDA;
    }
    *out = c;
    return MCL_OK;
}

int mcl_ctx_set_stream(mcl_ctx_t c, void *stream) {
    if (!c) return MCL_ERR_INVALID_ARG;
    c->stream = (cudaStream_t)stream;
    return MCL_OK;
}

int mcl_ctx_destroy(mcl_ctx_t c) {
    if (!c) return MCL_ERR_INVALID_ARG;
    cudaSetDevice(c->device);
    if (c->world) {
        ncclCommDestroy(c->rowc);
        ncclCommDestroy(c->colc);
        ncclCommDestroy(c->world);
    }
    for (auto &kv : c->scratch) dfree(c, kv.second.p, kv.second.bytes);
    cudaStreamSynchronize(c->stream);
    for (int i = 0; i < 8; i++)
        if (c->ev[i]) cudaEventDestroy(c->ev[i]);
    for (int i = 0; i < 2 * kAllBins + 2; i++)
        if (c->bev[i]) cudaEventDestroy(c->bev[i]);
    for (int i = 0; i < 6; i++)
        if (c->pev[i]) cudaEventDestroy(c->pev[i]);
    for (int i = 0; i < 3; i++)
        if (c->sev[i]) cudaEventDestroy(c->sev[i]);
    for (int i = 0; i < 2; i++)
        if (c->vev[i]) cudaEventDestroy(c->vev[i]);
    for (int i = 0; i < 5; i++)
        if (c->qev[i]) cudaEventDestroy(c->qev[i]);
    if (c->cstream) cudaStreamDestroy(c->cstream);
    if (c->pin) cudaFreeHost(c->pin);
    if (c->pin_up) cudaFreeHost(c->pin_up);
    if (c->up_ev) cudaEventDestroy(c->up_ev);
    delete c;
    return MCL_OK;
}

const char *mcl_last_error(mcl_ctx_t c) { return c ? c->err.c_str() : "null context"; }

int mcl_csc_release(mcl_ctx_t c, mcl_csc_t *m) {
    if (!c || !m) return MCL_ERR_INVALID_ARG;
    dfree(c, m->col_ptr, (size_t)(m->ncols + 1) * sizeof(int64_t));
    dfree(c, m->row_idx, (size_t)m->nnz * sizeof(int32_t));
    dfree(c, m->val, (size_t)m->nnz * sizeof(float));
    zero_csc(m);
    return MCL_OK;
}

int mcl_preprocess(mcl_ctx_t c, const mcl_csc_t *G, int add_loops, mcl_csc_t *A_out) {
    if (!c || !A_out) return MCL_ERR_INVALID_ARG;
    zero_csc(A_out);
    cudaSetDevice(c->device);
    RC(check_csc(c, G, "G"));
    if (G->nrows != G->ncols) return fail(c, MCL_ERR_DIM, "G must be square");
    const int64_t n = G->ncols;
    int64_t *cnt;
    void *tmp;
    RC(scratch_t(c, "pre_cnt", (size_t)std::max<int64_t>(n, 1), &cnt));
    RC(scratch(c, "scan_tmp", scan_tmp_bytes(n + 1), &tmp));
    CK(launch_pre_count(n, G->col_ptr, G->row_idx, add_loops, cnt, c->stream));
    mcl_csc_t out;
    zero_csc(&out);
    OutGuard guard(c, &out);
    out.col_ptr = (int64_t *)dalloc(c, (size_t)(n + 1) * sizeof(int64_t));
    if (!out.col_ptr) return fail(c, MCL_ERR_OOM, "col_ptr");
    CK(launch_scan_i64(cnt, out.col_ptr, n, tmp, c->stream));
    int64_t nnz = 0;
    RC(readback(c, out.col_ptr + n, sizeof(int64_t), &nnz));
    RC(alloc_rows_vals(c, &out, nnz));
    out.nrows = n;
    out.ncols = n;
    out.n_global = n;
    CK(launch_pre_fill(n, G->col_ptr, G->row_idx, G->val, add_loops, out.col_ptr, out.row_idx,
                       out.val, c->stream));
    *A_out = out;
    guard.release();
    return MCL_OK;
}

int mcl_flops(mcl_ctx_t c, const mcl_csc_t *A, const mcl_csc_t *B, int64_t *flops_dev,
              int64_t *total) {
    if (!c) return MCL_ERR_INVALID_ARG;
    cudaSetDevice(c->device);
    RC(validate_product(c, A, B, 0, B ? B->ncols : 0));
    const int64_t n = B->ncols;
    int64_t *f = flops_dev;
    if (!f) RC(scratch_t(c, "flops", (size_t)std::max<int64_t>(n, 1), &f));
    CK(launch_flops(n, A->col_ptr, B->col_ptr, B->row_idx, 0, f, c->stream));
    if (total) {
        unsigned long long *tot;
        RC(scratch_t(c, "tot", 4, &tot));
        CK(launch_reduce_i64(f, n, tot, c->stream));
        unsigned long long h = 0;
        RC(readback(c, tot, sizeof h, &h));
        *total = (int64_t)h;
    }
    return MCL_OK;
}

int mcl_estimate(mcl_ctx_t c, const mcl_csc_t *A, const mcl_csc_t *B, int32_t r, uint64_t seed,
                 float *est_dev, float *keys_dev, double *total) {
    if (!c || !est_dev) return c ? fail(c, MCL_ERR_INVALID_ARG, "est_dev is NULL") : MCL_ERR_INVALID_ARG;
    cudaSetDevice(c->device);
    if (r < 2 || r > 16) return fail(c, MCL_ERR_INVALID_ARG, "r must be in [2,16]");
    RC(validate_product(c, A, B, 0, B ? B->ncols : 0));
    Prod pr{A, B, 0, B->ncols};
    RC(cohen(c, pr, r, seed, est_dev, keys_dev));
    if (total) {
        unsigned long long *tot;
        RC(scratch_t(c, "tot", 4, &tot));
        double *d = (double *)tot;
        CK(launch_reduce_f32(est_dev, B->ncols, d, c->stream));
        RC(readback(c, d, sizeof(double), total));
    }
    return MCL_OK;
}

int mcl_symbolic(mcl_ctx_t c, const mcl_csc_t *A, const mcl_csc_t *B, int64_t *nnz_dev,
                 int64_t *total) {
    if (!c || !nnz_dev) return c ? fail(c, MCL_ERR_INVALID_ARG, "nnz_dev is NULL") : MCL_ERR_INVALID_ARG;
    cudaSetDevice(c->device);
    RC(validate_product(c, A, B, 0, B ? B->ncols : 0));
    mcl_params_t p;
    mcl_params_default(&p);
    const int64_t n = B->ncols;
    Prod pr{A, B, 0, n};
    int64_t *f;
    float *est;
    RC(scratch_t(c, "flops", (size_t)std::max<int64_t>(n, 1), &f));
    RC(scratch_t(c, "est", (size_t)std::max<int64_t>(n, 1), &est));
    CK(launch_flops(n, A->col_ptr, B->col_ptr, B->row_idx, 0, f, c->stream));
    RC(cohen(c, pr, p.est_keys, p.seed, est, nullptr));
    RC(symbolic_sizes(c, pr, f, est, -1, nnz_dev, nullptr));
    if (total) {
        unsigned long long *tot;
        RC(scratch_t(c, "tot", 4, &tot));
        CK(launch_reduce_i64(nnz_dev, n, tot, c->stream));
        unsigned long long h = 0;
        RC(readback(c, tot, sizeof h, &h));
        *total = (int64_t)h;
    }
    return MCL_OK;
}

int mcl_spgemm(mcl_ctx_t c, const mcl_csc_t *A, const mcl_csc_t *B, int64_t col_begin,
               int64_t col_end, const mcl_params_t *p, mcl_csc_t *C_out, mcl_stats_t *st) {
    if (!c || !C_out) return MCL_ERR_INVALID_ARG;
    zero_csc(C_out);
    cudaSetDevice(c->device);
    return spgemm_impl(c, A, B, col_begin, col_end, p, C_out, st);
}

int mcl_expand(mcl_ctx_t c, const mcl_csc_t *A, int64_t col_begin, int64_t col_end,
               const mcl_params_t *p, mcl_csc_t *C_out, mcl_stats_t *st) {
    if (!c || !C_out) return MCL_ERR_INVALID_ARG;
    zero_csc(C_out);
    cudaSetDevice(c->device);
    RC(check_csc(c, A, "A"));
    if (A->nrows != A->ncols) return fail(c, MCL_ERR_DIM, "expansion needs a square A");
    return spgemm_impl(c, A, A, col_begin, col_end, p, C_out, st);
}

int mcl_prune_inflate(mcl_ctx_t c, const mcl_csc_t *C, const mcl_params_t *pin, mcl_csc_t *A_next,
                      float *chaos_dev, mcl_stats_t *st) {
    if (!c) return MCL_ERR_INVALID_ARG;
    if (!A_next || !pin) return fail(c, MCL_ERR_INVALID_ARG, "NULL argument");
    zero_csc(A_next);
    cudaSetDevice(c->device);
    RC(check_params(c, pin));
    RC(check_csc(c, C, "C"));
    init_stats(st);
    const int64_t n = C->ncols;
    const PruneParams pp = prune_params(pin);
    const int64_t launches0 = g_launches;
    CK(cudaEventRecord(c->ev[0], c->stream));
    int64_t *kcap, *soff, *cnt;
    float *chaos, *cmax;
    int32_t *srow;
    float *sval;
    void *tmp;
    RC(scratch_t(c, "kcap", (size_t)std::max<int64_t>(n, 1), &kcap));
    RC(scratch_t(c, "soff", (size_t)n + 1, &soff));
    RC(scratch_t(c, "scnt", (size_t)std::max<int64_t>(n, 1), &cnt));
    RC(scratch_t(c, "chaos", (size_t)std::max<int64_t>(n, 1), &chaos));
    RC(scratch_t(c, "chaos_max", 4, &cmax));
    RC(scratch(c, "scan_tmp", scan_tmp_bytes(n + 1), &tmp));
    CK(launch_kcap_cp(n, C->col_ptr, pp.kmax, kcap, c->stream));
    CK(launch_scan_i64(kcap, soff, n, tmp, c->stream));
    int64_t stot = 0;
    RC(readback(c, soff + n, sizeof(int64_t), &stot));
    RC(scratch_t(c, "s_row", (size_t)std::max<int64_t>(stot, 1), &srow));
    RC(scratch_t(c, "s_val", (size_t)std::max<int64_t>(stot, 1), &sval));
    CK(cudaMemsetAsync(cmax, 0, sizeof(float), c->stream));
    const int grid = (int)std::min<int64_t>(std::max<int64_t>(n, 1), (int64_t)c->sms * 8);
    CK(launch_prune(n, C->col_ptr, C->row_idx, C->val, soff, srow, sval, cnt,
                    chaos_dev ? chaos_dev : chaos, cmax, pp, grid, c->stream));
    CK(cudaEventRecord(c->ev[1], c->stream));
    int64_t nnz = 0;
    OutGuard guard(c, A_next);
    RC(assemble(c, C->nrows, n, cnt, soff, srow, sval, A_next, &nnz));
    A_next->row0 = C->row0;
    A_next->col0 = C->col0;
    A_next->n_global = C->n_global ? C->n_global : C->nrows;
    CK(cudaEventRecord(c->ev[2], c->stream));
    float hmax = 0.f;
    RC(readback(c, cmax, sizeof(float), &hmax));
    if (st) {
        st->nnz_in = C->nnz;
        st->nnz_unpruned = C->nnz;
        st->nnz_out = nnz;
        st->chaos = hmax;
        st->ms[4] = elapsed(c, 0, 1);
        st->ms[5] = elapsed(c, 1, 2);
        st->ms[6] = elapsed(c, 0, 2);
        st->peak_bytes = (int64_t)c->peak;
        st->launches = g_launches - launches0;
    }
    guard.release();
    return MCL_OK;
}

int mcl_iterate(mcl_ctx_t c, const mcl_csc_t *A, const mcl_params_t *pin, mcl_csc_t *A_next,
                mcl_stats_t *st) {
    if (!c) return MCL_ERR_INVALID_ARG;
    if (!A) return fail(c, MCL_ERR_INVALID_ARG, "A is NULL");
    return mcl_iterate_range(c, A, 0, A->ncols, pin, A_next, st);
}

constexpr int kNeedPhases = 1;  // iterate_range_impl: the columns do not fit one phase

// one phase of mcl_iterate_range: the fused iteration on output columns [col_begin, col_end)
// of A * B (B = A for the expansion).
// check_budget: return kNeedPhases (nothing allocated) when the staging of the pruned
// columns + A_next, 16 B x sum_j min(max(S,R), f_j, m) + 16 B x n, exceeds the phase budget.
// cand (the 2D SUMMA's row blocks): A_next receives every column's top-max(S, R) entries,
// unscaled, and cand its statistics -- the prune needs the sums over all row blocks.
static int iterate_range_impl(mcl_ctx_t c, const mcl_csc_t *A, const mcl_csc_t *B, int64_t col_begin,
                              int64_t col_end, const mcl_params_t *pin, mcl_csc_t *A_next,
                              mcl_stats_t *st, bool check_budget = false,
                              CandOut *cand = nullptr) {
    if (!c) return MCL_ERR_INVALID_ARG;
    if (!A_next || !pin) return fail(c, MCL_ERR_INVALID_ARG, "NULL argument");
    zero_csc(A_next);
    cudaSetDevice(c->device);
    RC(check_params(c, pin));
    RC(check_csc(c, A, "A"));
    if (B == A) {
        if (A->nrows != A->ncols) return fail(c, MCL_ERR_DIM, "mcl_iterate needs a square A");
    } else {
        RC(check_csc(c, B, "B"));
        if (A->ncols != B->nrows) return fail(c, MCL_ERR_DIM, "inner dimensions differ");
    }
    if (col_begin < 0 || col_end > B->ncols || col_begin > col_end)
        return fail(c, MCL_ERR_DIM, "bad column range [%lld,%lld)", (long long)col_begin,
                    (long long)col_end);
    init_stats(st);
    const int64_t launches0 = g_launches;
    const mcl_params_t &p = *pin;
    const int64_t n = col_end - col_begin;
    Prod pr{A, B, col_begin, n};
    const PruneParams pp = prune_params(pin);
    CK(cudaEventRecord(c->ev[0], c->stream));
    int64_t *f, *kcap, *soff, *cnt, *nnzc = nullptr;
    float *est, *chaos, *cmax;
    int32_t *srow;
    float *sval;
    unsigned long long *tot;
    void *tmp;
    RC(scratch_t(c, "flops", (size_t)std::max<int64_t>(n, 1), &f));
    RC(scratch_t(c, "est", (size_t)std::max<int64_t>(n, 1), &est));
    RC(scratch_t(c, "kcap", (size_t)std::max<int64_t>(n, 1), &kcap));
    RC(scratch_t(c, "soff", (size_t)n + 1, &soff));
    RC(scratch_t(c, "scnt", (size_t)std::max<int64_t>(n, 1), &cnt));
    RC(scratch_t(c, "chaos", (size_t)std::max<int64_t>(n, 1), &chaos));
    RC(scratch_t(c, "chaos_max", 4, &cmax));
    RC(scratch_t(c, "tot", 4, &tot));
    RC(scratch(c, "scan_tmp", scan_tmp_bytes(n + 1), &tmp));

    // a1: flops and the total
    CK(launch_flops(n, A->col_ptr, B->col_ptr, B->row_idx, col_begin, f, c->stream));
    CK(launch_reduce_i64(f, n, tot, c->stream));
    CK(cudaEventRecord(c->ev[1], c->stream));
    // a2: Cohen estimate, then the P:1076-1077 policy
    RC(cohen(c, pr, p.est_keys, p.seed, est, nullptr));
    double *dsum = (double *)(tot + 1);
    CK(launch_reduce_f32(est, n, dsum, c->stream));
    unsigned long long hv[2];
    RC(readback(c, tot, sizeof hv, hv));
    double est_tot;
    memcpy(&est_tot, &hv[1], sizeof(double));
    const int64_t flops = (int64_t)hv[0];
    const double cf_est = est_tot > 0 ? (double)flops / est_tot : 0.0;
    int use_exact = p.estimator == 1 || (p.estimator == 0 && cf_est < p.est_cf_threshold);
    CK(cudaEventRecord(c->ev[2], c->stream));
    // a3: exact symbolic sizes when the policy asks for them
    if (use_exact) {
        RC(scratch_t(c, "nnz_sym", (size_t)std::max<int64_t>(n, 1), &nnzc));
        RC(symbolic_sizes(c, pr, f, est, p.force_bin, nnzc, nullptr));
    }
    CK(cudaEventRecord(c->ev[3], c->stream));
    // staging slots of the pruned columns
    CK(launch_kcap(n, f, A->nrows, pp.kmax, kcap, c->stream));
    CK(launch_scan_i64(kcap, soff, n, tmp, c->stream));
    int64_t stot = 0;
    RC(readback(c, soff + n, sizeof(int64_t), &stot));
    if (check_budget) {
        const double bytes = 16.0 * (double)stot + 16.0 * (double)n;
        // (the free-memory query only for sizable iterations, or an explicit budget)
        if ((bytes > (double)(1 << 30) || c->phase_budget > 0) &&
            bytes > phase_budget(c, pin->mem_safety, bytes))
            return kNeedPhases;
    }
    RC(scratch_t(c, "s_row", (size_t)std::max<int64_t>(stot, 1), &srow));
    RC(scratch_t(c, "s_val", (size_t)std::max<int64_t>(stot, 1), &sval));
    CK(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * std::max<int64_t>(n, 1), c->stream));
    CK(cudaMemsetAsync(chaos, 0, sizeof(float) * std::max<int64_t>(n, 1), c->stream));
    CK(cudaMemsetAsync(cmax, 0, sizeof(float), c->stream));
    // a4-a7: fused numeric SpGEMM + select / prune / recover / inflate / renormalise
    BinArgs base;
    memset(&base, 0, sizeof base);
    base.soff = soff;
    base.s_row = srow;
    base.s_val = sval;
    base.s_cnt = cnt;
    base.chaos = chaos;
    base.chaos_max = cmax;
    base.pp = pp;
    if (cand) {  // columns without products keep zero statistics
        base.cand_k = pp.kmax;
        base.stg_nnz = cand->nnz;
        base.stg_m = cand->m;
        base.stg_s = cand->s;
        const size_t n1 = (size_t)std::max<int64_t>(n, 1);
        CK(cudaMemsetAsync(cand->nnz, 0, sizeof(int64_t) * n1, c->stream));
        CK(cudaMemsetAsync(cand->m, 0, sizeof(int64_t) * n1, c->stream));
        CK(cudaMemsetAsync(cand->s, 0, sizeof(double) * n1, c->stream));
    }
    if (st) {
        for (int b = 0; b <= kNumBins; b++) st->bin_cols[b] = st->bin_flops[b] = 0;
    }
    RC(run_bins(c, kFused, pr, f, use_exact ? nullptr : est, use_exact ? nnzc : nullptr,
                p.force_bin, base, st, cf_est));
    CK(cudaEventRecord(c->ev[4], c->stream));
    int64_t nnz = 0;
    OutGuard guard(c, A_next);
    if (cand) {
        // the candidates stay in the staging slots (the distributed prune reads them there);
        // their total and the unpruned total from the statistics, one read-back
        CK(launch_reduce_i64(cnt, n, tot + 2, c->stream));
        CK(launch_reduce_i64(cand->nnz, n, tot + 3, c->stream));
        unsigned long long ht[2] = {0, 0};
        RC(readback(c, tot + 2, sizeof ht, ht));
        cand->start = soff;
        cand->count = cnt;
        cand->row = srow;
        cand->val = sval;
        cand->total = nnz = (int64_t)ht[0];
        cand->unpruned = (int64_t)ht[1];
        CK(cudaEventRecord(c->ev[5], c->stream));
    } else {
        // a8: assemble A_next
        RC(assemble(c, A->nrows, n, cnt, soff, srow, sval, A_next, &nnz));
        A_next->row0 = A->row0;
        A_next->col0 = B->col0 + col_begin;
        A_next->n_global = A->n_global ? A->n_global : A->nrows;
        CK(cudaEventRecord(c->ev[5], c->stream));
    }
    float hmax = 0.f;
    RC(readback(c, cmax, sizeof(float), &hmax));
    if (st) {
        st->flops = flops;
        st->nnz_in = A->nnz;
        st->nnz_out = nnz;
        st->est_nnz = est_tot;
        st->cf = cf_est;
        st->chaos = hmax;
        st->estimator_used = use_exact ? 1 : 2;
        st->ms[0] = elapsed(c, 0, 1);
        st->ms[1] = elapsed(c, 1, 2);
        st->ms[2] = elapsed(c, 2, 3);
        st->ms[3] = elapsed(c, 3, 4);
        st->ms[5] = elapsed(c, 4, 5);
        st->ms[6] = elapsed(c, 0, 5);
        st->peak_bytes = (int64_t)c->peak;
        st->launches = g_launches - launches0;
    }
    guard.release();
    return MCL_OK;
}

int mcl_iterate_range(mcl_ctx_t c, const mcl_csc_t *A, int64_t col_begin, int64_t col_end,
                      const mcl_params_t *pin, mcl_csc_t *A_next, mcl_stats_t *st) {
    if (!c) return MCL_ERR_INVALID_ARG;
    if (!A_next || !pin) return fail(c, MCL_ERR_INVALID_ARG, "NULL argument");
    zero_csc(A_next);
    cudaSetDevice(c->device);
    RC(check_params(c, pin));
    RC(check_csc(c, A, "A"));
    if (A->nrows != A->ncols) return fail(c, MCL_ERR_DIM, "mcl_iterate needs a square A");
    if (col_begin < 0 || col_end > A->ncols || col_begin > col_end)
        return fail(c, MCL_ERR_DIM, "bad column range [%lld,%lld)", (long long)col_begin,
                    (long long)col_end);
    // Phases (Q15).  The fused iteration never holds the unpruned product; what
    // grows with the columns is the staging of the pruned columns and A_next: 16 B x
    // min(max(S, R), f_j, m) per column (+ its col_ptr).  Columns are cut into batches of
    // near-equal bytes within mem_safety x free HBM, each batch runs as one fused iteration
    // and the batches' outputs are concatenated.
    const int64_t n = col_end - col_begin;
    if (c->force_phases <= 1) {  // one phase unless it would not fit (checked inside)
        const int rc = iterate_range_impl(c, A, A, col_begin, col_end, pin, A_next, st, true);
        if (rc != kNeedPhases) {
            if (rc == MCL_OK && st) st->phases = 1;
            return rc;
        }
    }
    const PruneParams pp = prune_params(pin);
    int64_t *f, *bytes;
    RC(scratch_t(c, "phase_flops", (size_t)std::max<int64_t>(n, 1), &f));
    RC(scratch_t(c, "phase_bytes", (size_t)std::max<int64_t>(n, 1), &bytes));
    CK(launch_flops(n, A->col_ptr, A->col_ptr, A->row_idx, col_begin, f, c->stream));
    CK(launch_kcap(n, f, A->nrows, pp.kmax, bytes, c->stream));
    CK(launch_affine_i64(n, bytes, 16, 16, bytes, false, c->stream));
    std::vector<int64_t> bounds;
    RC(plan_phases(c, bytes, n, [&](double need) { return phase_budget(c, pin->mem_safety, need); },
                   bounds, nullptr));
    const int h = (int)bounds.size() - 1;
    if (h <= 1) {
        const int rc = iterate_range_impl(c, A, A, col_begin, col_end, pin, A_next, st);
        if (rc == MCL_OK && st) st->phases = 1;
        return rc;
    }
    init_stats(st);
    std::vector<mcl_csc_t> pieces;
    int rc = MCL_OK;
    for (int q = 0; q < h && rc == MCL_OK; q++) {
        mcl_csc_t piece;
        mcl_stats_t sq;
        rc = iterate_range_impl(c, A, A, col_begin + bounds[q], col_begin + bounds[q + 1], pin, &piece,
                                st ? &sq : nullptr);
        if (rc == MCL_OK) {
            pieces.push_back(piece);
            if (st) add_stats(st, sq);
        }
    }
    if (rc == MCL_OK) rc = concat_cols(c, pieces, A_next);
    for (auto &q : pieces) free_csc(c, &q);
    if (rc != MCL_OK) return rc;
    if (st) {
        st->nnz_in = A->nnz;
        st->nnz_out = A_next->nnz;
        st->phases = h;
        st->peak_bytes = (int64_t)c->peak;
    }
    return MCL_OK;
}

int mcl_clusters(mcl_ctx_t c, const mcl_csc_t *A, int32_t *labels_dev, int64_t *ncl) {
    if (!c) return MCL_ERR_INVALID_ARG;
    if (!labels_dev) return fail(c, MCL_ERR_INVALID_ARG, "labels_dev is NULL");
    cudaSetDevice(c->device);
    RC(check_csc(c, A, "A"));
    if (A->nrows != A->ncols) return fail(c, MCL_ERR_DIM, "clusters need a square A");
    const int64_t n = A->ncols;
    int32_t *parent;
    int64_t *flag, *rank;
    void *tmp;
    RC(scratch_t(c, "cc_parent", (size_t)std::max<int64_t>(n, 1), &parent));
    RC(scratch_t(c, "cc_flag", (size_t)std::max<int64_t>(n, 1), &flag));
    RC(scratch_t(c, "cc_rank", (size_t)n + 1, &rank));
    RC(scratch(c, "scan_tmp", scan_tmp_bytes(n + 1), &tmp));
    CK(launch_cc(n, A->col_ptr, A->row_idx, parent, flag, rank, tmp, labels_dev, c->stream));
    int64_t k = 0;
    RC(readback(c, rank + n, sizeof(int64_t), &k));
    if (ncl) *ncl = k;
    return MCL_OK;
}

int mcl_summa_schedule(int pr, int pc, int rank, int64_t n, int stage_mult, int64_t *out,
                       int64_t cap) {
    if (pr < 1 || pc < 1 || rank < 0 || rank >= pr * pc || n < 0 || stage_mult < 1 || !out)
        return MCL_ERR_INVALID_ARG;
    const int s = pr / gcd_i(pr, pc) * pc * stage_mult;
    if (cap < 4 + 5 * (int64_t)s) return MCL_ERR_INVALID_ARG;
    const int gi = rank / pc, gj = rank % pc;
    out[0] = cut(n, pr, gi);
    out[1] = cut(n, pr, gi + 1);
    out[2] = cut(n, pc, gj);
    out[3] = cut(n, pc, gj + 1);
    for (int q = 0; q < s; q++) {
        int64_t *o = out + 4 + 5 * q;
        o[0] = cut(n, s, q);
        o[1] = cut(n, s, q + 1);
        o[2] = (int64_t)q * pc / s;  // the A-panel's owner: (gi, o[2]), broadcast along my row
        o[3] = (int64_t)q * pr / s;  // the B-panel's owner: (o[3], gj), along my column
        o[4] = alg2_nmerges(q + 1);
    }
    return s;
}

int mcl_host_csc_release(mcl_csc_t *m) {
    if (!m) return MCL_ERR_INVALID_ARG;
    if (m->col_ptr) cudaFreeHost(m->col_ptr);
    if (m->row_idx) cudaFreeHost(m->row_idx);
    if (m->val) cudaFreeHost(m->val);
    zero_csc(m);
    return MCL_OK;
}

// Host-memory-backed iteration: the Pipelined Sparse SUMMA of P:337-363 §III on one GPU, for
// an iterate that does not fit the device.  See include/mclx.h.
int mcl_iterate_hostmem(mcl_ctx_t c, const mcl_csc_t *Ah, const mcl_params_t *pin, int32_t stages,
                        int32_t phases, mcl_csc_t *out, mcl_stats_t *st) {
    if (!c) return MCL_ERR_INVALID_ARG;
    if (!Ah || !pin || !out) return fail(c, MCL_ERR_INVALID_ARG, "NULL argument");
    zero_csc(out);
    cudaSetDevice(c->device);
    RC(check_params(c, pin));
    if (Ah->nrows != Ah->ncols || Ah->nrows < 0 || Ah->nnz < 0 || !Ah->col_ptr ||
        (Ah->nnz > 0 && (!Ah->row_idx || !Ah->val)))
        return fail(c, MCL_ERR_DIM, "A must be a square host CSC");
    init_stats(st);
    const int64_t launches0 = g_launches;
    const int64_t n = Ah->ncols, nnz = Ah->nnz;
    const PruneParams pp = prune_params(pin);
    // sizes: an A-panel holds nnz / s entries (two of them live), a phase's B columns nnz / h
    // plus its partial products; both cut so they stay well inside mem_safety x free HBM
    const double budget = phase_budget(c, pin->mem_safety);
    const int64_t s = stages > 0 ? stages
                                 : std::max<int64_t>(1, (int64_t)std::ceil(12.0 * (double)nnz / (0.1 * budget)));
    const int64_t h = phases > 0 ? phases
                                 : std::max<int64_t>(1, (int64_t)std::ceil(12.0 * (double)nnz / (0.1 * budget)));
    if (s > n && n > 0) return fail(c, MCL_ERR_INVALID_ARG, "more stages than columns");
    cudaStream_t cs;
    CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaEvent_t ready[2], freed[2], start, stop;
    for (int i = 0; i < 2; i++) {
        cudaEventCreateWithFlags(&ready[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&freed[i], cudaEventDisableTiming);
    }
    cudaEventCreate(&start);
    cudaEventCreate(&stop);
    struct Cleanup {
        cudaStream_t cs;
        cudaEvent_t *ev;
        ~Cleanup() {
            cudaStreamSynchronize(cs);
            cudaStreamDestroy(cs);
            for (int i = 0; i < 6; i++) cudaEventDestroy(ev[i]);
        }
    } ;
    cudaEvent_t evs[6] = {ready[0], ready[1], freed[0], freed[1], start, stop};
    Cleanup cleanup{cs, evs};
    CK(cudaEventRecord(start, c->stream));
    // the phases: column batches of near-equal nnz(B_*j), cut on the device from col_ptr
    int64_t *dcp;
    RC(scratch_t(c, "hm_colptr", (size_t)n + 1, &dcp));
    CK(cudaMemcpyAsync(dcp, Ah->col_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, c->stream));
    std::vector<int64_t> bounds{0};
    if (h > 1 && n > 0) {
        int64_t *cut;
        RC(scratch_t(c, "hm_cut", (size_t)h, &cut));
        CK(launch_phase_cuts(dcp, n, (int)h, cut, c->stream));
        std::vector<int64_t> hc((size_t)h - 1);
        RC(readback(c, cut, sizeof(int64_t) * (h - 1), hc.data()));
        for (int64_t v : hc)
            if (v > bounds.back() && v < n) bounds.push_back(v);
    }
    bounds.push_back(n);
    const int nph = (int)bounds.size() - 1;
    // the A-panels (columns K_q of A, contiguous in CSC): double-buffered on the copy stream
    int64_t max_k = 1, max_pa = 1;
    for (int64_t q = 0; q < s; q++) {
        const int64_t k0 = cut(n, (int)s, (int)q), k1 = cut(n, (int)s, (int)q + 1);
        max_k = std::max(max_k, k1 - k0);
        max_pa = std::max(max_pa, Ah->col_ptr[k1] - Ah->col_ptr[k0]);
    }
    struct Buf2 {
        int64_t *cp, *cpraw;
        int32_t *row;
        float *val;
    } pa[2];
    for (int i = 0; i < 2; i++) {
        const std::string t = std::to_string(i);
        RC(scratch_t(c, ("hm_pa_cp" + t).c_str(), (size_t)max_k + 1, &pa[i].cp));
        RC(scratch_t(c, ("hm_pa_cpraw" + t).c_str(), (size_t)max_k + 1, &pa[i].cpraw));
        RC(scratch_t(c, ("hm_pa_row" + t).c_str(), (size_t)max_pa, &pa[i].row));
        RC(scratch_t(c, ("hm_pa_val" + t).c_str(), (size_t)max_pa, &pa[i].val));
    }
    std::vector<mcl_csc_t> hpieces;  // pruned phases, host (pinned)
    auto drop_host = [&]() {
        for (auto &x : hpieces) mcl_host_csc_release(&x);
        hpieces.clear();
    };
    int64_t flops = 0, nnz_unpruned = 0, peak_partial = 0, h2d = 0;
    float chaos = 0.f;
    int rc = MCL_OK;
    int64_t issued = 0;  // A-panel copies issued so far (buffer = issued & 1)
    auto issue_panel = [&](int64_t q) -> int {
        const int64_t k0 = cut(n, (int)s, (int)q), k1 = cut(n, (int)s, (int)q + 1);
        const int64_t a0 = Ah->col_ptr[k0], a1 = Ah->col_ptr[k1];
        Buf2 &B = pa[issued & 1];
        if (issued >= 2) CK(cudaStreamWaitEvent(cs, freed[issued & 1], 0));  // product done with it
        CK(cudaMemcpyAsync(B.cpraw, Ah->col_ptr + k0, sizeof(int64_t) * (k1 - k0 + 1),
                           cudaMemcpyHostToDevice, cs));
        CK(launch_rebase_colptr(k1 - k0 + 1, B.cpraw, B.cp, cs));
        if (a1 > a0) {
            CK(cudaMemcpyAsync(B.row, Ah->row_idx + a0, sizeof(int32_t) * (a1 - a0),
                               cudaMemcpyHostToDevice, cs));
            CK(cudaMemcpyAsync(B.val, Ah->val + a0, sizeof(float) * (a1 - a0), cudaMemcpyHostToDevice, cs));
        }
        CK(cudaEventRecord(ready[issued & 1], cs));
        h2d += (k1 - k0 + 1) * 8 + (a1 - a0) * 8;
        issued++;
        return MCL_OK;
    };
    for (int ph = 0; ph < nph && rc == MCL_OK; ph++) {
        const int64_t c0 = bounds[ph], c1 = bounds[ph + 1], nb = c1 - c0;
        const int64_t b0 = Ah->col_ptr[c0], b1 = Ah->col_ptr[c1];
        // the phase's columns B = A[:, c0:c1) (copied once), sliced by rows per stage below
        int64_t *bcp, *bcpraw, *first, *bcnt, *pbcp;
        int32_t *brow, *pbrow;
        float *bval, *pbval;
        void *tmp;
        RC(scratch_t(c, "hm_b_cp", (size_t)nb + 1, &bcp));
        RC(scratch_t(c, "hm_b_cpraw", (size_t)nb + 1, &bcpraw));
        RC(scratch_t(c, "hm_b_row", (size_t)std::max<int64_t>(b1 - b0, 1), &brow));
        RC(scratch_t(c, "hm_b_val", (size_t)std::max<int64_t>(b1 - b0, 1), &bval));
        RC(scratch_t(c, "hm_first", (size_t)std::max<int64_t>(nb, 1), &first));
        RC(scratch_t(c, "hm_bcnt", (size_t)std::max<int64_t>(nb, 1), &bcnt));
        RC(scratch_t(c, "hm_pb_cp", (size_t)nb + 1, &pbcp));
        RC(scratch_t(c, "hm_pb_row", (size_t)std::max<int64_t>(b1 - b0, 1), &pbrow));
        RC(scratch_t(c, "hm_pb_val", (size_t)std::max<int64_t>(b1 - b0, 1), &pbval));
        RC(scratch(c, "scan_tmp", scan_tmp_bytes(nb + 1), &tmp));
        CK(cudaMemcpyAsync(bcpraw, Ah->col_ptr + c0, sizeof(int64_t) * (nb + 1), cudaMemcpyHostToDevice,
                           c->stream));
        CK(launch_rebase_colptr(nb + 1, bcpraw, bcp, c->stream));
        if (b1 > b0) {
            CK(cudaMemcpyAsync(brow, Ah->row_idx + b0, sizeof(int32_t) * (b1 - b0), cudaMemcpyHostToDevice,
                               c->stream));
            CK(cudaMemcpyAsync(bval, Ah->val + b0, sizeof(float) * (b1 - b0), cudaMemcpyHostToDevice,
                               c->stream));
        }
        h2d += (nb + 1) * 8 + (b1 - b0) * 8;
        std::vector<mcl_csc_t> stack;
        int64_t live = 0;
        if (ph == 0) RC(issue_panel(0));
        for (int64_t q = 0; q < s && rc == MCL_OK; q++) {
            // the next A-panel streams in while this stage multiplies
            const int64_t qn = q + 1 < s ? q + 1 : (ph + 1 < nph ? 0 : -1);
            const int cur = (int)((issued - 1) & 1);
            if (qn >= 0 && (rc = issue_panel(qn)) != MCL_OK) break;
            const int64_t k0 = cut(n, (int)s, (int)q), k1 = cut(n, (int)s, (int)q + 1);
            CK(cudaStreamWaitEvent(c->stream, ready[cur], 0));
            // rows K_q of the phase's columns
            CK(launch_rowslice_count(nb, bcp, brow, k0, k1, first, bcnt, c->stream));
            CK(launch_scan_i64(bcnt, pbcp, nb, tmp, c->stream));
            int64_t nbq = 0;
            RC(readback(c, pbcp + nb, sizeof(int64_t), &nbq));
            CK(launch_rowslice_copy(nb, first, pbcp, brow, bval, k0, pbrow, pbval, c->stream));
            mcl_csc_t Pa, Pb, Pq;
            zero_csc(&Pa);
            zero_csc(&Pb);
            Pa.nrows = n;
            Pa.ncols = k1 - k0;
            Pa.nnz = Ah->col_ptr[k1] - Ah->col_ptr[k0];
            Pa.col0 = k0;
            Pa.n_global = n;
            Pa.col_ptr = pa[cur].cp;
            Pa.row_idx = pa[cur].row;
            Pa.val = pa[cur].val;
            Pb.nrows = k1 - k0;
            Pb.ncols = nb;
            Pb.nnz = nbq;
            Pb.row0 = k0;
            Pb.col0 = c0;
            Pb.n_global = n;
            Pb.col_ptr = pbcp;
            Pb.row_idx = pbrow;
            Pb.val = pbval;
            mcl_stats_t sst;
            if ((rc = spgemm_impl(c, &Pa, &Pb, 0, nb, pin, &Pq, &sst)) != MCL_OK) break;
            CK(cudaEventRecord(freed[cur], c->stream));
            flops += sst.flops;
            Pq.col0 = c0;
            stack.push_back(Pq);
            live += Pq.nnz;
            peak_partial = std::max(peak_partial, live);
            // Alg. 2: merge nmerges+1 lists at even stage counts
            const int nmerges = alg2_nmerges(q + 1);
            if (nmerges > 0) {
                std::vector<mcl_csc_t> L(stack.end() - (nmerges + 1), stack.end());
                mcl_csc_t merged;
                if ((rc = merge_impl(c, (int32_t)L.size(), L.data(), &merged)) != MCL_OK) break;
                for (auto &x : L) {
                    live -= x.nnz;
                    free_csc(c, &x);
                }
                stack.resize(stack.size() - L.size());
                stack.push_back(merged);
                live += merged.nnz;
                peak_partial = std::max(peak_partial, live);
            }
        }
        if (rc == MCL_OK && stack.size() > 1) {  // Q16
            mcl_csc_t merged;
            rc = merge_impl(c, (int32_t)stack.size(), stack.data(), &merged);
            if (rc == MCL_OK) {
                for (auto &x : stack) free_csc(c, &x);
                stack.assign(1, merged);
            }
        }
        if (rc != MCL_OK) {
            for (auto &x : stack) free_csc(c, &x);
            break;
        }
        // prune / inflate the phase on the device, then its pruned columns to host memory
        mcl_csc_t Cb = stack[0], piece;
        float ch = 0.f;
        rc = dist_prune(c, &Cb, nullptr, pp, &piece, &ch);
        nnz_unpruned += Cb.nnz;
        free_csc(c, &Cb);
        if (rc != MCL_OK) break;
        chaos = std::max(chaos, ch);
        mcl_csc_t hp;
        zero_csc(&hp);
        hp.nrows = n;
        hp.ncols = nb;
        hp.nnz = piece.nnz;
        hp.col0 = c0;
        hp.n_global = n;
        cudaError_t e = cudaMallocHost(&hp.col_ptr, sizeof(int64_t) * (nb + 1));
        if (e == cudaSuccess) e = cudaMallocHost(&hp.row_idx, sizeof(int32_t) * std::max<int64_t>(piece.nnz, 1));
        if (e == cudaSuccess) e = cudaMallocHost(&hp.val, sizeof(float) * std::max<int64_t>(piece.nnz, 1));
        if (e == cudaSuccess) e = cudaMemcpyAsync(hp.col_ptr, piece.col_ptr, sizeof(int64_t) * (nb + 1),
                                                  cudaMemcpyDeviceToHost, c->stream);
        if (e == cudaSuccess && piece.nnz)
            e = cudaMemcpyAsync(hp.row_idx, piece.row_idx, sizeof(int32_t) * piece.nnz, cudaMemcpyDeviceToHost,
                                c->stream);
        if (e == cudaSuccess && piece.nnz)
            e = cudaMemcpyAsync(hp.val, piece.val, sizeof(float) * piece.nnz, cudaMemcpyDeviceToHost, c->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
        free_csc(c, &piece);
        hpieces.push_back(hp);
        if (e != cudaSuccess) {
            cudaGetLastError();
            rc = fail(c, MCL_ERR_CUDA, "hostmem phase output: %s", cudaGetErrorString(e));
        }
    }
    if (rc != MCL_OK) {
        drop_host();
        return rc;
    }
    // the phases, concatenated in host memory (each phase's col_ptr is 0-based)
    int64_t tot = 0;
    for (auto &x : hpieces) tot += x.nnz;
    mcl_csc_t o;
    zero_csc(&o);
    cudaError_t e = cudaMallocHost(&o.col_ptr, sizeof(int64_t) * (n + 1));
    if (e == cudaSuccess) e = cudaMallocHost(&o.row_idx, sizeof(int32_t) * std::max<int64_t>(tot, 1));
    if (e == cudaSuccess) e = cudaMallocHost(&o.val, sizeof(float) * std::max<int64_t>(tot, 1));
    if (e != cudaSuccess) {
        cudaGetLastError();
        mcl_host_csc_release(&o);
        drop_host();
        return fail(c, MCL_ERR_OOM, "cannot allocate the host output");
    }
    int64_t coff = 0, off = 0;
    o.col_ptr[0] = 0;
    for (auto &x : hpieces) {
        for (int64_t j = 1; j <= x.ncols; j++) o.col_ptr[coff + j] = x.col_ptr[j] + off;
        memcpy(o.row_idx + off, x.row_idx, sizeof(int32_t) * x.nnz);
        memcpy(o.val + off, x.val, sizeof(float) * x.nnz);
        coff += x.ncols;
        off += x.nnz;
    }
    drop_host();
    o.nrows = n;
    o.ncols = n;
    o.nnz = tot;
    o.n_global = n;
    *out = o;
    CK(cudaEventRecord(stop, c->stream));
    if (st) {
        CK(cudaEventSynchronize(stop));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, start, stop);
        st->ms[6] = ms;
        st->flops = flops;
        st->nnz_in = nnz;
        st->nnz_unpruned = nnz_unpruned;
        st->nnz_out = tot;
        st->chaos = chaos;
        st->phases = nph;
        st->stages = (int32_t)s;
        st->peak_partial = peak_partial;
        st->comm_bytes = h2d;  // host -> device bytes of the panels and phase columns
        st->peak_bytes = (int64_t)c->peak;
        st->launches = g_launches - launches0;
        st->estimator_used = 1;
    }
    return MCL_OK;
}

int mcl_merge(mcl_ctx_t c, int32_t L, const mcl_csc_t *lists, mcl_csc_t *out) {
    if (!c) return MCL_ERR_INVALID_ARG;
    if (!out || !lists || L < 1) return fail(c, MCL_ERR_INVALID_ARG, "bad merge arguments");
    zero_csc(out);
    cudaSetDevice(c->device);
    return merge_impl(c, L, lists, out);
}

int mcl_block(mcl_ctx_t c, const mcl_csc_t *A, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
              mcl_csc_t *out) {
    if (!c) return MCL_ERR_INVALID_ARG;
    if (!out) return fail(c, MCL_ERR_INVALID_ARG, "out is NULL");
    zero_csc(out);
    cudaSetDevice(c->device);
    RC(check_csc(c, A, "A"));
    if (r0 < 0 || r1 > A->nrows || r0 > r1 || c0 < 0 || c1 > A->ncols || c0 > c1)
        return fail(c, MCL_ERR_DIM, "block out of range");
    const int64_t nc = c1 - c0;
    int64_t *first, *cnt;
    void *tmp;
    RC(scratch_t(c, "blk_first", (size_t)std::max<int64_t>(nc, 1), &first));
    RC(scratch_t(c, "blk_cnt", (size_t)std::max<int64_t>(nc, 1), &cnt));
    RC(scratch(c, "scan_tmp", scan_tmp_bytes(nc + 1), &tmp));
    mcl_csc_t o;
    zero_csc(&o);
    OutGuard guard(c, &o);
    o.col_ptr = (int64_t *)dalloc(c, sizeof(int64_t) * (nc + 1));
    if (!o.col_ptr) return fail(c, MCL_ERR_OOM, "col_ptr");
    CK(launch_rowslice_count(nc, A->col_ptr + c0, A->row_idx, r0, r1, first, cnt, c->stream));
    CK(launch_scan_i64(cnt, o.col_ptr, nc, tmp, c->stream));
    int64_t nnz = 0;
    RC(readback(c, o.col_ptr + nc, sizeof(int64_t), &nnz));
    RC(alloc_rows_vals(c, &o, nnz));
    CK(launch_rowslice_copy(nc, first, o.col_ptr, A->row_idx, A->val, r0, o.row_idx, o.val,
                            c->stream));
    o.nrows = r1 - r0;
    o.ncols = nc;
    o.row0 = A->row0 + r0;
    o.col0 = A->col0 + c0;
    o.n_global = A->n_global ? A->n_global : A->nrows;
    *out = o;
    guard.release();
    return MCL_OK;
}

int mcl_prof_read(uint64_t out[12], int reset) {
    if (!out) return MCL_ERR_INVALID_ARG;
    unsigned long long v[12];
    prof_read(v, reset);
    for (int i = 0; i < 12; i++) out[i] = v[i];
    return MCL_OK;
}

int mcl_nccl_unique_id(unsigned char out[128]) {
    if (!out) return MCL_ERR_INVALID_ARG;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return MCL_ERR_NCCL;
    memcpy(out, id.internal, 128);
    return MCL_OK;
}

int mcl_ctx_set_grid(mcl_ctx_t c, int pr, int pc, int rank, const unsigned char id[128]) {
    if (!c) return MCL_ERR_INVALID_ARG;
    if (pr < 1 || pc < 1 || rank < 0 || rank >= pr * pc || !id)
        return fail(c, MCL_ERR_INVALID_ARG, "bad grid %dx%d rank %d", pr, pc, rank);
    cudaSetDevice(c->device);
    if (c->world) {
        ncclCommDestroy(c->rowc);
        ncclCommDestroy(c->colc);
        ncclCommDestroy(c->world);
        c->world = c->rowc = c->colc = nullptr;
    }
    ncclUniqueId uid;
    memcpy(uid.internal, id, 128);
    NC(ncclCommInitRank(&c->world, pr * pc, uid, rank));
    const int gi = rank / pc, gj = rank % pc;
    NC(ncclCommSplit(c->world, gi, gj, &c->rowc, nullptr));
    NC(ncclCommSplit(c->world, gj, gi, &c->colc, nullptr));
    if (!c->cstream) {
        CK(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
        for (int i = 0; i < 5; i++) CK(cudaEventCreateWithFlags(&c->qev[i], cudaEventDisableTiming));
    }
    c->pr = pr;
    c->pc = pc;
    c->rank = rank;
    return MCL_OK;
}

int mcl_summa_iterate(mcl_ctx_t c, const mcl_csc_t *A, const mcl_params_t *pin, mcl_csc_t *A_next,
                      mcl_stats_t *st) {
    if (!c) return MCL_ERR_INVALID_ARG;
    if (!A_next || !pin) return fail(c, MCL_ERR_INVALID_ARG, "NULL argument");
    zero_csc(A_next);
    cudaSetDevice(c->device);
    if (!c->world) return fail(c, MCL_ERR_INVALID_ARG, "mcl_ctx_set_grid has not been called");
    RC(check_params(c, pin));
    RC(check_csc(c, A, "A"));
    init_stats(st);
    const int64_t launches0 = g_launches;
    const int pr = c->pr, pc = c->pc, gi = c->rank / pc, gj = c->rank % pc;
    const int64_t n = A->n_global;
    if (A->row0 != cut(n, pr, gi) || A->nrows != cut(n, pr, gi + 1) - cut(n, pr, gi) ||
        A->col0 != cut(n, pc, gj) || A->ncols != cut(n, pc, gj + 1) - cut(n, pc, gj))
        return fail(c, MCL_ERR_DIM, "block (%d,%d) does not match the %dx%d grid of n=%lld", gi, gj,
                    pr, pc, (long long)n);
    if (pr == 1 && !getenv("MCLX_SUMMA_STAGED") && !getenv("MCLX_SUMMA_ACCUM")) {
        // 1 x pc grid: every column of C = A*A lives on one rank.  The stage broadcasts of
        // the A-panels (the pc column stripes) are issued together, and instead of
        // materialising one partial product per stage and merging them (Alg. 2), all stages
        // accumulate in the fused kernel's hash table; the prune is then local.
        const int P = pc;
        int64_t *szd;
        RC(scratch_t(c, "summa_sz", (size_t)P, &szd));
        const int64_t my = A->nnz;
        RC(upload(c, &my, sizeof(int64_t), szd + c->rank));
        NC(ncclAllGather(szd + c->rank, szd, 1, ncclInt64, c->world, c->stream));
        std::vector<int64_t> sz(P), off(P + 1, 0);
        RC(readback(c, szd, sizeof(int64_t) * P, sz.data()));
        for (int r = 0; r < P; r++) off[r + 1] = off[r] + sz[r];
        const int64_t tot = off[P];
        int64_t *fcp, *cps;
        int32_t *frow;
        float *fval;
        RC(scratch_t(c, "summa_fcp", (size_t)n + 1, &fcp));
        RC(scratch_t(c, "summa_cps", (size_t)n + P, &cps));
        RC(scratch_t(c, "summa_frow", (size_t)std::max<int64_t>(tot, 1), &frow));
        RC(scratch_t(c, "summa_fval", (size_t)std::max<int64_t>(tot, 1), &fval));
        NC(ncclGroupStart());
        for (int r = 0; r < P; r++) {
            const int64_t c0 = cut(n, P, r), nc = cut(n, P, r + 1) - c0;
            const bool me = r == c->rank;
            NC(ncclBroadcast(me ? (const void *)A->col_ptr : (const void *)(cps + c0 + r), cps + c0 + r,
                             nc + 1, ncclInt64, r, c->world, c->stream));
            if (sz[r]) {
                NC(ncclBroadcast(me ? (const void *)A->row_idx : (const void *)(frow + off[r]),
                                 frow + off[r], sz[r], ncclInt32, r, c->world, c->stream));
                NC(ncclBroadcast(me ? (const void *)A->val : (const void *)(fval + off[r]),
                                 fval + off[r], sz[r], ncclFloat32, r, c->world, c->stream));
            }
        }
        NC(ncclGroupEnd());
        for (int r = 0; r < P; r++) {
            const int64_t c0 = cut(n, P, r), nc = cut(n, P, r + 1) - c0;
            CK(launch_offset_colptr(nc + 1, cps + c0 + r, off[r], fcp + c0, c->stream));
        }
        // Cohen's first layer (min of the row keys over each column of A) is the
        // one estimator pass over all of A: each rank computes it for its own column block
        // and the blocks are broadcast, instead of every rank redoing all of A
        if (pin->estimator != 1) {
            const int rk = pin->est_keys;
            float *X, *Mf;
            RC(scratch_t(c, "cohen_X", (size_t)std::max<int64_t>(n, 1) * rk, &X));
            RC(scratch_t(c, "cohen_Mfull", (size_t)std::max<int64_t>(n, 1) * rk, &Mf));
            CK(launch_cohen_keys(n, 0, rk, pin->seed, X, nullptr, c->stream));
            const int64_t my0 = cut(n, P, c->rank);
            CK(launch_cohen_min(A->ncols, A->col_ptr, A->row_idx, 0, X, rk, Mf + my0 * rk, nullptr,
                                c->stream));
            NC(ncclGroupStart());
            for (int r = 0; r < P; r++) {
                const int64_t c0 = cut(n, P, r), nc = cut(n, P, r + 1) - c0;
                if (nc) NC(ncclBroadcast(Mf + c0 * rk, Mf + c0 * rk, nc * rk, ncclFloat32, r, c->world,
                                         c->stream));
            }
            NC(ncclGroupEnd());
            c->cohen_M_pre = Mf;
            c->cohen_M_r = rk;
        }
        mcl_csc_t Af;
        zero_csc(&Af);
        Af.nrows = n;
        Af.ncols = n;
        Af.nnz = tot;
        Af.n_global = n;
        Af.col_ptr = fcp;
        Af.row_idx = frow;
        Af.val = fval;
        const int rc_it = mcl_iterate_range(c, &Af, A->col0, A->col0 + A->ncols, pin, A_next, st);
        c->cohen_M_pre = nullptr;  // consumed by that call (or dropped on its failure)
        RC(rc_it);
        OutGuard guard(c, A_next);
        float chaos = st ? st->chaos : 0.f;
        float *cm;
        RC(scratch_t(c, "chaos_max", 4, &cm));
        RC(upload(c, &chaos, sizeof(float), cm));
        NC(ncclAllReduce(cm, cm, 1, ncclFloat32, ncclMax, c->world, c->stream));
        RC(readback(c, cm, sizeof(float), &chaos));
        if (st) {
            st->chaos = chaos;
            st->comm_bytes = (tot - my) * 8 + (n - A->ncols) * 8;
            st->phases = 1;
        }
        guard.release();
        return MCL_OK;
    }
    // inner panels: s = lcm(pr, pc) (Q17), times MCLX_SUMMA_STAGES (a multiplier that keeps
    // every panel inside one row and one column stripe; tests use it to run Alg. 2's merges
    // on a 1 x 1 grid)
    int smul = 1;
    if (const char *e = getenv("MCLX_SUMMA_STAGES")) smul = std::max(1, atoi(e));
    const int s = pr / gcd_i(pr, pc) * pc * smul;
    const int64_t nj = A->ncols, mi = A->nrows;
    const PruneParams pp = prune_params(pin);
    CK(cudaEventRecord(c->sev[0], c->stream));

    // ---- sizes of the panels this rank owns, all-gathered once (P:239-243 stage k)
    int64_t *hdr, *first, *cnt;
    RC(scratch_t(c, "summa_hdr", (size_t)2 * s * pr * pc, &hdr));
    RC(scratch_t(c, "summa_first", (size_t)std::max<int64_t>(nj, 1), &first));
    RC(scratch_t(c, "summa_cnt", (size_t)std::max<int64_t>(nj, 1), &cnt));
    void *tmp;
    RC(scratch(c, "scan_tmp", scan_tmp_bytes(nj + 1), &tmp));
    int64_t *bcp_own;
    RC(scratch_t(c, "summa_bcp_own", (size_t)s * (nj + 1), &bcp_own));
    std::vector<int64_t> mine(2 * s, 0), a0s((size_t)s, 0);
    for (int q = 0; q < s; q++) {
        const int64_t k0 = cut(n, s, q), k1 = cut(n, s, q + 1);
        if ((int64_t)q * pc / s == gj) {  // A-panel owner: columns K_q of my block
            int64_t ab[2];
            RC(readback(c, A->col_ptr + (k0 - A->col0), sizeof(int64_t), &ab[0]));
            RC(readback(c, A->col_ptr + (k1 - A->col0), sizeof(int64_t), &ab[1]));
            mine[2 * q] = ab[1] - ab[0];
            a0s[q] = ab[0];
        }
        if ((int64_t)q * pr / s == gi) {  // B-panel owner: rows K_q of my block
            CK(launch_rowslice_count(nj, A->col_ptr, A->row_idx, k0 - A->row0, k1 - A->row0, first,
                                     cnt, c->stream));
            CK(launch_scan_i64(cnt, bcp_own + (int64_t)q * (nj + 1), nj, tmp, c->stream));
            RC(readback(c, bcp_own + (int64_t)q * (nj + 1) + nj, sizeof(int64_t), &mine[2 * q + 1]));
        }
    }
    RC(upload(c, mine.data(), sizeof(int64_t) * 2 * s, hdr + (int64_t)2 * s * c->rank));
    NC(ncclAllGather(hdr + (int64_t)2 * s * c->rank, hdr, 2 * s, ncclInt64, c->world, c->stream));
    std::vector<int64_t> table((size_t)2 * s * pr * pc);
    RC(readback(c, hdr, sizeof(int64_t) * table.size(), table.data()));

    // ---- every stage's panels, broadcast once on the comm stream and kept resident.  Rank
    // (i, j) then holds A[rows_i, :] and A[:, cols_j] (nnz(A) (1/pr + 1/pc) entries), all the
    // operands of every phase, so a phase re-runs its stage products without re-broadcasting
    // (P:317-319 notes that cost for HipMCL's phases).  The compute stream waits for stage q's
    // panels only when it first needs them, so the broadcasts overlap the estimation and the
    // first phase's products.
    struct Panels {
        int64_t *acp, *bcp, *first, *cnt;
        int32_t *arow, *brow;
        float *aval, *bval;
        int64_t nnzA, nnzB, k0, kq;
    };
    std::vector<Panels> pan((size_t)s);
    std::vector<cudaEvent_t> ready((size_t)s, nullptr);
    struct EvGuard {
        std::vector<cudaEvent_t> &v;
        ~EvGuard() {
            for (auto e : v)
                if (e) cudaEventDestroy(e);
        }
    } evg{ready};
    for (int q = 0; q < s; q++) {
        Panels &P = pan[q];
        const int ca = (int)((int64_t)q * pc / s), rb = (int)((int64_t)q * pr / s);
        P.k0 = cut(n, s, q);
        P.kq = cut(n, s, q + 1) - P.k0;
        P.nnzA = table[(size_t)2 * s * (gi * pc + ca) + 2 * q];
        P.nnzB = table[(size_t)2 * s * (rb * pc + gj) + 2 * q + 1];
        const std::string t = std::to_string(q);
        RC(scratch_t(c, ("pa_cp" + t).c_str(), (size_t)P.kq + 1, &P.acp));
        RC(scratch_t(c, ("pa_row" + t).c_str(), (size_t)std::max<int64_t>(P.nnzA, 1), &P.arow));
        RC(scratch_t(c, ("pa_val" + t).c_str(), (size_t)std::max<int64_t>(P.nnzA, 1), &P.aval));
        RC(scratch_t(c, ("pb_cp" + t).c_str(), (size_t)nj + 1, &P.bcp));
        RC(scratch_t(c, ("pb_row" + t).c_str(), (size_t)std::max<int64_t>(P.nnzB, 1), &P.brow));
        RC(scratch_t(c, ("pb_val" + t).c_str(), (size_t)std::max<int64_t>(P.nnzB, 1), &P.bval));
        RC(scratch_t(c, ("pb_first" + t).c_str(), (size_t)std::max<int64_t>(nj, 1), &P.first));
        RC(scratch_t(c, ("pb_cnt" + t).c_str(), (size_t)std::max<int64_t>(nj, 1), &P.cnt));
        CK(cudaEventCreateWithFlags(&ready[q], cudaEventDisableTiming));
    }
    cudaStream_t cs = c->cstream;
    CK(cudaEventRecord(c->qev[4], c->stream));  // A, bcp_own ready
    CK(cudaStreamWaitEvent(cs, c->qev[4], 0));
    int64_t comm_bytes = 0;
    for (int q = 0; q < s; q++) {
        Panels &P = pan[q];
        const int ca = (int)((int64_t)q * pc / s), rb = (int)((int64_t)q * pr / s);
        if (ca == gj) {
            CK(launch_rebase_colptr(P.kq + 1, A->col_ptr + (P.k0 - A->col0), P.acp, cs));
            if (P.nnzA) {
                CK(cudaMemcpyAsync(P.arow, A->row_idx + a0s[q], sizeof(int32_t) * P.nnzA,
                                   cudaMemcpyDeviceToDevice, cs));
                CK(cudaMemcpyAsync(P.aval, A->val + a0s[q], sizeof(float) * P.nnzA,
                                   cudaMemcpyDeviceToDevice, cs));
            }
        } else {
            comm_bytes += (P.kq + 1) * 8 + P.nnzA * 8;
        }
        if (rb == gi) {
            const int64_t *ocp = bcp_own + (int64_t)q * (nj + 1);
            CK(launch_rowslice_count(nj, A->col_ptr, A->row_idx, P.k0 - A->row0, P.k0 + P.kq - A->row0,
                                     P.first, P.cnt, cs));
            CK(cudaMemcpyAsync(P.bcp, ocp, sizeof(int64_t) * (nj + 1), cudaMemcpyDeviceToDevice, cs));
            CK(launch_rowslice_copy(nj, P.first, P.bcp, A->row_idx, A->val, P.k0 - A->row0, P.brow,
                                    P.bval, cs));
        } else {
            comm_bytes += (nj + 1) * 8 + P.nnzB * 8;
        }
        NC(ncclGroupStart());
        NC(ncclBroadcast(P.acp, P.acp, P.kq + 1, ncclInt64, ca, c->rowc, cs));
        if (P.nnzA) {
            NC(ncclBroadcast(P.arow, P.arow, P.nnzA, ncclInt32, ca, c->rowc, cs));
            NC(ncclBroadcast(P.aval, P.aval, P.nnzA, ncclFloat32, ca, c->rowc, cs));
        }
        NC(ncclBroadcast(P.bcp, P.bcp, nj + 1, ncclInt64, rb, c->colc, cs));
        if (P.nnzB) {
            NC(ncclBroadcast(P.brow, P.brow, P.nnzB, ncclInt32, rb, c->colc, cs));
            NC(ncclBroadcast(P.bval, P.bval, P.nnzB, ncclFloat32, rb, c->colc, cs));
        }
        NC(ncclGroupEnd());
        CK(cudaEventRecord(ready[q], cs));
    }
    auto panel_a = [&](int q) {
        mcl_csc_t Pa;
        zero_csc(&Pa);
        Pa.nrows = mi;
        Pa.ncols = pan[q].kq;
        Pa.nnz = pan[q].nnzA;
        Pa.row0 = A->row0;
        Pa.col0 = pan[q].k0;
        Pa.n_global = n;
        Pa.col_ptr = pan[q].acp;
        Pa.row_idx = pan[q].arow;
        Pa.val = pan[q].aval;
        return Pa;
    };
    auto panel_b = [&](int q) {
        mcl_csc_t Pb;
        zero_csc(&Pb);
        Pb.nrows = pan[q].kq;
        Pb.ncols = nj;
        Pb.nnz = pan[q].nnzB;
        Pb.row0 = pan[q].k0;
        Pb.col0 = A->col0;
        Pb.n_global = n;
        Pb.col_ptr = pan[q].bcp;
        Pb.row_idx = pan[q].brow;
        Pb.val = pan[q].bval;
        return Pb;
    };

    // ---- phases (Q15) and the products.  Two forms:
    //  * accumulating (default for pr > 1): C_ij = sum_q A_iq B_qj = A[rows_i, :] A[:, cols_j].
    //    The A-panels are the column ranges of the row stripe and the B-panels the row ranges
    //    of the column stripe, so stacking them gives both stripes and ONE binned hash SpGEMM
    //    forms C_ij: every stage's products land in the same hash tables, the per-stage
    //    partials and Alg. 2's merges are never materialised.  Phases are sized by the
    //    product's upper-bound slots, 16 B x min(f_j, m_i).
    //  * staged (MCLX_SUMMA_STAGED=1): one product per stage and the Alg. 2 binary merge
    //    (P:509-529), phases sized by Cohen's estimate of every stage product:
    //    8 B x 1.3 x sum_q est_q(j) x 2 (partials + the merge's copy) + 16 B.
    // Either way the byte estimates are all-reduced (max) over the column communicator, whose
    // ranks split the same columns and must run the same batches for the distributed prune.
    const bool staged = getenv("MCLX_SUMMA_STAGED") != nullptr;
    std::vector<int64_t> bounds;
    int64_t est_bytes = 0;
    int h = 1;
    std::vector<mcl_csc_t> pieces;
    std::vector<mcl_csc_t> stack;
    int64_t peak_partial = 0, flops = 0, nnz_unpruned = 0;
    float chaos = 0.f, prod_ms = 0.f, prune_ms = 0.f;  // accumulating form: ms[4], ms[7]
    float bin_ms[kNumBins + 1] = {};
    int64_t bin_flops[kNumBins + 1] = {}, bin_cols[kNumBins + 1] = {}, bin_nnzb[kNumBins + 1] = {},
            bin_out[kNumBins + 1] = {};
    int rc = MCL_OK;
    auto drop = [&](std::vector<mcl_csc_t> &v) {
        for (auto &x : v) free_csc(c, &x);
        v.clear();
    };
    mcl_csc_t Ai, Bj;
    zero_csc(&Ai);
    zero_csc(&Bj);
    if (staged) {
        int64_t *pbytes;
        float *pest;
        RC(scratch_t(c, "summa_phase_bytes", (size_t)std::max<int64_t>(nj, 1), &pbytes));
        RC(scratch_t(c, "summa_phase_est", (size_t)std::max<int64_t>(nj, 1), &pest));
        CK(cudaMemsetAsync(pbytes, 0, sizeof(int64_t) * std::max<int64_t>(nj, 1), c->stream));
        for (int q = 0; q < s; q++) {
            CK(cudaStreamWaitEvent(c->stream, ready[q], 0));
            mcl_csc_t Pa = panel_a(q), Pb = panel_b(q);
            RC(cohen(c, Prod{&Pa, &Pb, 0, nj}, pin->est_keys, pin->seed, pest, nullptr));
            CK(launch_affine_est(nj, pest, 8.0 * 1.3 * 2.0, q == 0 ? 16 : 0, pbytes, c->stream));
        }
        if (pr > 1 && nj > 0) NC(ncclAllReduce(pbytes, pbytes, nj, ncclInt64, ncclMax, c->colc, c->stream));
        RC(plan_phases(c, pbytes, nj, [&](double need) { return phase_budget(c, pin->mem_safety, need); },
                       bounds, &est_bytes));
        h = (int)bounds.size() - 1;
        // per phase: stage products on the phase's columns, Alg. 2 binary merge, distributed
        // prune / inflate
        for (int ph = 0; ph < h && rc == MCL_OK; ph++) {
            const int64_t c0 = bounds[ph], c1 = bounds[ph + 1];
            int64_t live_partial = 0;
            for (int q = 0; q < s && rc == MCL_OK; q++) {
                mcl_csc_t Pa = panel_a(q), Pb = panel_b(q), Pq;
                mcl_stats_t sst;
                if ((rc = spgemm_impl(c, &Pa, &Pb, c0, c1, pin, &Pq, &sst)) != MCL_OK) break;
                flops += sst.flops;
                for (int b = 0; b <= kNumBins; b++) {
                    bin_ms[b] += sst.bin_ms[b];
                    bin_flops[b] += sst.bin_flops[b];
                    bin_cols[b] += sst.bin_cols[b];
                    bin_nnzb[b] += sst.bin_nnzb[b];
                    bin_out[b] += sst.bin_out[b];
                }
                Pq.row0 = A->row0;
                Pq.col0 = A->col0 + c0;
                Pq.n_global = n;
                stack.push_back(Pq);
                live_partial += Pq.nnz;
                peak_partial = std::max(peak_partial, live_partial);
                // Alg. 2 lines 5-14: merge nmerges+1 lists when the stage count is even
                const int nmerges = alg2_nmerges(q + 1);
                if (nmerges > 0) {
                    std::vector<mcl_csc_t> L(stack.end() - (nmerges + 1), stack.end());
                    mcl_csc_t merged;
                    if ((rc = merge_impl(c, (int32_t)L.size(), L.data(), &merged)) != MCL_OK) break;
                    for (auto &x : L) {
                        live_partial -= x.nnz;
                        free_csc(c, &x);
                    }
                    stack.resize(stack.size() - L.size());
                    stack.push_back(merged);
                    live_partial += merged.nnz;
                    peak_partial = std::max(peak_partial, live_partial);
                }
            }
            if (rc == MCL_OK && stack.size() > 1) {  // Q16: stage counts that are not powers of two
                mcl_csc_t merged;
                rc = merge_impl(c, (int32_t)stack.size(), stack.data(), &merged);
                if (rc == MCL_OK) {
                    drop(stack);
                    stack.push_back(merged);
                }
            }
            if (rc != MCL_OK) break;
            mcl_csc_t Cb = stack[0], piece;
            stack.clear();
            float ch = 0.f;
            rc = dist_prune(c, &Cb, pr > 1 ? c->colc : nullptr, pp, &piece, &ch);
            nnz_unpruned += Cb.nnz;
            free_csc(c, &Cb);
            if (rc != MCL_OK) break;
            pieces.push_back(piece);
            chaos = std::max(chaos, ch);
        }
    } else {
        if (s > kMaxStages) return fail(c, MCL_ERR_NOT_IMPLEMENTED, "more than %d inner panels", kMaxStages);
        // Cohen's first layer over A[rows_i, :] is split across the row
        // communicator: rank (i, j) takes its own block's columns cols_j (while the panels
        // are in flight), the pc pieces are broadcast on the comm stream after the panels
        float *Mf = nullptr;
        const int rk = pin->est_keys;
        if (pin->estimator != 1) {
            float *X;
            RC(scratch_t(c, "cohen_X", (size_t)std::max<int64_t>(mi, 1) * rk, &X));
            RC(scratch_t(c, "cohen_Mfull", (size_t)std::max<int64_t>(n, 1) * rk, &Mf));
            CK(launch_cohen_keys(mi, A->row0, rk, pin->seed, X, nullptr, c->stream));
            CK(launch_cohen_min(nj, A->col_ptr, A->row_idx, 0, X, rk, Mf + A->col0 * rk, nullptr,
                                c->stream));
            cudaEvent_t mev[2];
            for (auto &e : mev) {
                CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                ready.push_back(e);  // destroyed with the panels' events
            }
            CK(cudaEventRecord(mev[0], c->stream));
            CK(cudaStreamWaitEvent(cs, mev[0], 0));
            NC(ncclGroupStart());
            for (int r = 0; r < pc; r++) {
                const int64_t k0 = cut(n, pc, r), nk = cut(n, pc, r + 1) - k0;
                if (nk) NC(ncclBroadcast(Mf + k0 * rk, Mf + k0 * rk, nk * rk, ncclFloat32, r, c->rowc, cs));
            }
            NC(ncclGroupEnd());
            CK(cudaEventRecord(mev[1], cs));
            CK(cudaStreamWaitEvent(c->stream, mev[1], 0));
        }
        int64_t nnzAi = 0, nnzBj = 0;
        for (int q = 0; q < s; q++) {
            CK(cudaStreamWaitEvent(c->stream, ready[q], 0));
            nnzAi += pan[q].nnzA;
            nnzBj += pan[q].nnzB;
        }
        int64_t *aicp, *bjcp, *bjcnt;
        int32_t *airow, *bjrow;
        float *aival, *bjval;
        RC(scratch_t(c, "summa_aicp", (size_t)n + 1, &aicp));
        RC(scratch_t(c, "summa_airow", (size_t)std::max<int64_t>(nnzAi, 1), &airow));
        RC(scratch_t(c, "summa_aival", (size_t)std::max<int64_t>(nnzAi, 1), &aival));
        RC(scratch_t(c, "summa_bjcp", (size_t)nj + 1, &bjcp));
        RC(scratch_t(c, "summa_bjcnt", (size_t)std::max<int64_t>(nj, 1), &bjcnt));
        RC(scratch_t(c, "summa_bjrow", (size_t)std::max<int64_t>(nnzBj, 1), &bjrow));
        RC(scratch_t(c, "summa_bjval", (size_t)std::max<int64_t>(nnzBj, 1), &bjval));
        int64_t off = 0;
        for (int q = 0; q < s; q++) {  // A[rows_i, :]: the A-panels side by side
            CK(launch_offset_colptr(pan[q].kq + 1, pan[q].acp, off, aicp + pan[q].k0, c->stream));
            if (pan[q].nnzA) {
                CK(cudaMemcpyAsync(airow + off, pan[q].arow, sizeof(int32_t) * pan[q].nnzA,
                                   cudaMemcpyDeviceToDevice, c->stream));
                CK(cudaMemcpyAsync(aival + off, pan[q].aval, sizeof(float) * pan[q].nnzA,
                                   cudaMemcpyDeviceToDevice, c->stream));
            }
            off += pan[q].nnzA;
        }
        VStack v;  // A[:, cols_j]: the B-panels stacked by rows
        memset(&v, 0, sizeof v);
        v.s = s;
        for (int q = 0; q < s; q++) {
            v.cp[q] = pan[q].bcp;
            v.row[q] = pan[q].brow;
            v.val[q] = pan[q].bval;
            v.k0[q] = pan[q].k0;
        }
        CK(launch_vstack(nj, v, bjcnt, nullptr, nullptr, nullptr, true, c->stream));
        CK(launch_scan_i64(bjcnt, bjcp, nj, tmp, c->stream));
        CK(launch_vstack(nj, v, nullptr, bjcp, bjrow, bjval, false, c->stream));
        Ai.nrows = mi;
        Ai.ncols = n;
        Ai.nnz = nnzAi;
        Ai.row0 = A->row0;
        Ai.n_global = n;
        Ai.col_ptr = aicp;
        Ai.row_idx = airow;
        Ai.val = aival;
        Bj.nrows = n;
        Bj.ncols = nj;
        Bj.nnz = nnzBj;
        Bj.col0 = A->col0;
        Bj.n_global = n;
        Bj.col_ptr = bjcp;
        Bj.row_idx = bjrow;
        Bj.val = bjval;
        // fused (default): the product runs in candidate mode -- every output column's
        // top-max(S, R) entries and the statistics of all its entries, from the same kernels as
        // the 1-GPU fused iteration (hub columns as row-range parts) -- so the unpruned C_ij is
        // never written; MCLX_SUMMA_UNFUSED=1 forms C_ij unpruned (spgemm) instead
        const bool fused = getenv("MCLX_SUMMA_UNFUSED") == nullptr;
        int64_t *pbytes, *pf;
        RC(scratch_t(c, "summa_phase_bytes", (size_t)std::max<int64_t>(nj, 1), &pbytes));
        RC(scratch_t(c, "summa_phase_flops", (size_t)std::max<int64_t>(nj, 1), &pf));
        CK(launch_flops(nj, Ai.col_ptr, Bj.col_ptr, Bj.row_idx, 0, pf, c->stream));
        CK(launch_kcap(nj, pf, mi, fused ? pp.kmax : INT32_MAX, pbytes, c->stream));
        CK(launch_affine_i64(nj, pbytes, 16, fused ? 40 : 16, pbytes, false, c->stream));
        if (pr > 1 && nj > 0) NC(ncclAllReduce(pbytes, pbytes, nj, ncclInt64, ncclMax, c->colc, c->stream));
        RC(plan_phases(c, pbytes, nj,
                       [&](double need) {
                           return std::min(0.5 * phase_budget(c, pin->mem_safety, 2.0 * need),
                                           2.0 * (double)c->cap_budget);
                       },
                       bounds, &est_bytes));
        h = (int)bounds.size() - 1;
        CK(cudaEventRecord(c->sev[1], c->stream));  // set-up done
        for (int ph = 0; ph < h && rc == MCL_OK; ph++) {
            const int64_t c0 = bounds[ph], c1 = bounds[ph + 1];
            mcl_csc_t Cb, piece;
            mcl_stats_t sst;
            CandOut co{nullptr, nullptr, nullptr};
            if (fused) {
                const size_t nc1 = (size_t)std::max<int64_t>(c1 - c0, 1);
                RC(scratch_t(c, "cand_nnz", nc1, &co.nnz));
                RC(scratch_t(c, "cand_m", nc1, &co.m));
                RC(scratch_t(c, "cand_s", nc1, &co.s));
                if (Mf) {  // consumed by the phase's estimate
                    c->cohen_M_pre = Mf;
                    c->cohen_M_r = rk;
                }
                rc = iterate_range_impl(c, &Ai, &Bj, c0, c1, pin, &Cb, &sst, false, &co);
                c->cohen_M_pre = nullptr;
            } else {
                rc = spgemm_impl(c, &Ai, &Bj, c0, c1, pin, &Cb, &sst);
            }
            if (rc != MCL_OK) break;
            flops += sst.flops;
            prod_ms += sst.ms[6];
            for (int b = 0; b <= kNumBins; b++) {
                bin_ms[b] += sst.bin_ms[b];
                bin_flops[b] += sst.bin_flops[b];
                bin_cols[b] += sst.bin_cols[b];
                bin_nnzb[b] += sst.bin_nnzb[b];
                bin_out[b] += sst.bin_out[b];
            }
            if (fused) {  // the candidates, read in place from the product's staging slots
                Cb.nrows = mi;
                Cb.ncols = c1 - c0;
                Cb.nnz = co.total;
                Cb.col_ptr = const_cast<int64_t *>(co.start);
                Cb.row_idx = const_cast<int32_t *>(co.row);
                Cb.val = const_cast<float *>(co.val);
            }
            Cb.row0 = A->row0;
            Cb.col0 = A->col0 + c0;
            Cb.n_global = n;
            peak_partial = std::max(peak_partial, Cb.nnz);
            const int64_t unpruned = fused ? co.unpruned : Cb.nnz;
            float ch = 0.f;
            rc = dist_prune(c, &Cb, pr > 1 ? c->colc : nullptr, pp, &piece, &ch, fused ? &co : nullptr,
                            fused ? co.count : nullptr);
            nnz_unpruned += unpruned;
            if (!fused) free_csc(c, &Cb);  // (the candidates are the context's scratch)
            if (rc != MCL_OK) break;
            if (st) {
                float dm = 0.f;
                CK(cudaEventSynchronize(c->pev[4]));
                if (cudaEventElapsedTime(&dm, c->pev[0], c->pev[4]) == cudaSuccess) prune_ms += dm;
                else cudaGetLastError();
            }
            pieces.push_back(piece);
            chaos = std::max(chaos, ch);
        }
    }
    if (rc != MCL_OK) {
        drop(stack);
        drop(pieces);
        return rc;
    }
    OutGuard guard(c, A_next);
    if (h == 1) {
        *A_next = pieces[0];
        pieces.clear();
    } else {
        rc = concat_cols(c, pieces, A_next);
        drop(pieces);
        if (rc != MCL_OK) return rc;
    }
    CK(cudaEventRecord(c->sev[2], c->stream));
    float *cm;
    RC(scratch_t(c, "chaos_max", 4, &cm));
    RC(upload(c, &chaos, sizeof(float), cm));
    NC(ncclAllReduce(cm, cm, 1, ncclFloat32, ncclMax, c->world, c->stream));
    RC(readback(c, cm, sizeof(float), &chaos));
    if (st) {
        st->nnz_in = A->nnz;
        st->nnz_unpruned = nnz_unpruned;
        st->nnz_out = A_next->nnz;
        st->chaos = chaos;
        st->phases = h;
        st->stages = s;
        st->est_nnz = staged ? (double)est_bytes / (8.0 * 1.3 * 2.0) : -1.0;
        st->estimator_used = 1;
        float tot = -1.f;
        cudaEventSynchronize(c->sev[2]);
        if (cudaEventElapsedTime(&tot, c->sev[0], c->sev[2]) != cudaSuccess) cudaGetLastError();
        st->ms[6] = tot;
        float pm[4];
        for (int q = 0; q < 4; q++) {  // the last phase's distributed prune
            pm[q] = 0.f;
            if (cudaEventElapsedTime(&pm[q], c->pev[q], c->pev[q + 1]) != cudaSuccess) {
                cudaGetLastError();
                pm[q] = -1.f;
            }
        }
        st->ms[0] = pm[0];  // prune: local stats + all-reduce
        st->ms[1] = pm[1];  // prune: top-k cut (radix histograms + all-reduces)
        st->ms[2] = pm[2];  // prune: kept sums + all-reduce
        st->ms[5] = pm[3];  // prune: write + assemble
        st->ms[3] = st->ms[4] = st->ms[7] = -1.f;
        if (!staged) {
            if (cudaEventElapsedTime(&st->ms[3], c->sev[0], c->sev[1]) != cudaSuccess) {
                cudaGetLastError();
                st->ms[3] = -1.f;
            }
            st->ms[4] = prod_ms;
            st->ms[7] = prune_ms;
        }
        st->comm_bytes = comm_bytes;
        st->peak_partial = peak_partial;
        st->flops = flops;
        for (int b = 0; b <= kNumBins; b++) {
            st->bin_ms[b] = bin_ms[b];
            st->bin_flops[b] = bin_flops[b];
            st->bin_cols[b] = bin_cols[b];
            st->bin_nnzb[b] = bin_nnzb[b];
            st->bin_out[b] = bin_out[b];
        }
        st->peak_bytes = (int64_t)c->peak;
        st->launches = g_launches - launches0;
    }
    guard.release();
    return MCL_OK;
}

}  // extern "C"
