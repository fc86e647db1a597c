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
// ACCUMULATION, private family (atomic-free values).  The CTA of a bin has W = NT/32
// warps; each warp owns a private slice (cap/W slots) of the column's table and 1/W of the
// row space: the 32-way row-partition index of A (rowpart[k][i] = first position in A_*k
// with row >= ceil(i m/32), built once per call) gives every warp its sub-segment of each
// A_*k.  A warp walks the column's segments on its own (32 segment descriptors loaded by
// its lanes, one per lane, and broadcast with shuffles -- no CTA barrier) in batches of
// kItems sub-segments side by side, 32 rows of each; the gathers of batch i+1 are issued
// before batch i is inserted.  One warp-uniform probe loop resolves all items of a batch
// (warp_insert_n): empty slots are claimed with an integer CAS (only new keys), values are
// added item by item with a plain LDS/FADD/STS (the rows of one item are distinct).
// Measured on B200 (tools/ubench.cu): shared float atomicAdd is a CAS loop
// (ATOMS.CAST.SPIN) at ~2.5 lane-ops/cycle/SM, MATCH.ANY ~0.5, plain RMW ~4.5, so neither
// value atomics nor warp-synchronous matching is used.  Slices are ordered by row range,
// so the compacted table is grouped by row range for the epilogue.
//
// CTA-shared family (short segments, R-MAT-like): one table per CTA, groups of g lanes per
// segment with 16-byte gathers, warps take segments dynamically, slots resolved first and
// float atomicAdds issued with the warp reconverged (insert4b).
//
// kPart: one row-range part of a split column (see run_split in capi.cu), accumulated by
// either family over the part's rowparts and written, rows sorted, to a staging slot.
#include <type_traits>

#include "kernels.h"

namespace mclx {

// Development counters (compiled in with -DMCLX_PROF; read with mcl_prof_read):
// [0] insert calls (warp) [1] probe-loop passes (warp) [2] valid lanes (products)
// [3] accumulate cycles (per warp, summed) [4] epilogue cycles (per CTA) [5] columns
__device__ unsigned long long g_prof[12];
#ifdef MCLX_PROF
#define PROF_ADD(i, v) atomicAdd(&g_prof[i], (unsigned long long)(v))
#else
#define PROF_ADD(i, v) ((void)0)
#endif

#ifndef MCLX_KITEMS
#define MCLX_KITEMS 4
#endif
constexpr int kItems = MCLX_KITEMS;  // sub-segment chunks whose gathers a warp keeps in flight


// Double hashing for the private slices: an odd step from a second hash of the row, so a
// power-of-two slice is walked in a full cycle and keys that share a home slot part ways
// after one probe (linear probing's primary clusters make the warp-uniform probe loop wait
// for the longest run among ~100 lane-items).  Slices are powers of two (CAP / W, or the
// global bin's 64 W 2^k).
__device__ __forceinline__ uint32_t probe_step(int row, uint32_t scap) {
    return (((uint32_t)row * 0x85EBCA6Bu) >> 15 | 1u) & (scap - 1);
}

// Open addressing, four keys per lane at a time (CTA-shared family).  Double hashing
// (probe_step; the CTA-shared tables are powers of two); an empty home slot is claimed by
// integer CAS in the first pass; the table's fill count is updated once per call by one lane
// (a warp-aggregated claim count), not by an atomic per claim inside the probe loop, so the
// warp-uniform loop walks only real collisions.  The float atomicAdds (a CAS loop on
// sm_100) then run with the warp reconverged.  Returns false (warp-uniform) on overflow:
// fill past `limit` (7/8 cap: an under-estimated column fails fast and is re-run in a bigger
// bin), or a walk longer than cap.  `fresh` counts keys this lane created.
template <int MODE, typename V>
__device__ __forceinline__ bool insert4b(int *keys, V *vals, uint32_t cap, const int (&row)[4],
                                         const V (&v)[4], const bool (&valid)[4], int *fill,
                                         int limit, int &fresh) {
    const unsigned FULL = 0xffffffffu;
    volatile int *vk = keys;
    uint32_t s[4];
    int k[4];
    bool need[4];
    int claims = 0;
    bool any = false;
#pragma unroll
    for (int j = 0; j < 4; j++) {
        s[j] = hash_slot(row[j], cap);
        k[j] = valid[j] ? vk[s[j]] : row[j];
    }
#pragma unroll
    for (int j = 0; j < 4; j++) {
        if (valid[j] && k[j] == kEmptyKey) {
            const int old = atomicCAS(&keys[s[j]], kEmptyKey, row[j]);
            claims += old == kEmptyKey;
            k[j] = old == kEmptyKey ? row[j] : old;
        }
        need[j] = k[j] != row[j];
        any |= need[j];
    }
    uint32_t walk = 0;
    while (__any_sync(FULL, any)) {
        any = false;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            if (need[j]) {
                if (k[j] == kEmptyKey) {
                    const int old = atomicCAS(&keys[s[j]], kEmptyKey, row[j]);
                    if (old == kEmptyKey) {
                        claims++;
                        need[j] = false;
                    } else {
                        k[j] = old;
                        need[j] = old != row[j];
                    }
                } else {
                    s[j] = (s[j] + probe_step(row[j], cap)) & (cap - 1);
                    k[j] = vk[s[j]];
                    need[j] = k[j] != row[j];
                }
            }
            any |= need[j];
        }
        if (++walk > cap) break;  // warp-uniform: a (nearly) full table -> overflow below
    }
    fresh += claims;
    int tot = __reduce_add_sync(FULL, claims);
    if (lane_id() == 0) tot = atomicAdd(fill, tot) + tot;
    tot = __shfl_sync(FULL, tot, 0);
    const bool ok = tot <= limit && walk <= cap;
    if (MODE != kSym && ok) {
#pragma unroll
        for (int j = 0; j < 4; j++)
            if (valid[j]) atomicAdd(&vals[s[j]], v[j]);
    }
    return ok;
}

constexpr int kLongSeg = 128;  // CTA-shared family: segments walked by a whole warp

__device__ __forceinline__ int group_size_for(int64_t avg) {
    return avg >= 24 ? 32 : avg >= 12 ? 16 : avg >= 6 ? 8 : 4;
}

// Insert kItems (row, v) per lane into this warp's private slice (keys, vals)[0, scap):
// open addressing with double hashing (probe_step), empty slots claimed with an integer atomicCAS (lanes
// of the warp may race for one slot), `fill` (warp-uniform) counts claimed slots and
// passing `limit` (7/8 of the slice) reports overflow so the column is re-run in a bigger
// bin.  All 32 lanes must call.  (item u: lanes hold distinct rows of one sub-segment;
// the same row may appear in several items).  All slots are probed first and one
// warp-uniform loop resolves misses / claims for every item, so a call that needs a claim
// pays the vote + fill count once for all items, not once per item.  The value updates
// then run item by item with a warp barrier between them: that is what keeps two lanes
// holding the same row in different items from losing an update.
template <int MODE, typename V, int NI>
__device__ __forceinline__ bool warp_insert_n(int *keys, V *vals, uint32_t scap, const bool (&valid)[NI],
                                              const int (&row)[NI], const V (&v)[NI], int &fill,
                                              int limit, unsigned &passes) {
    const unsigned FULL = 0xffffffffu;
    volatile int *vk = keys;
    uint32_t s[NI];
    int k[NI];
    bool need[NI];
#pragma unroll
    for (int u = 0; u < NI; u++) {
        s[u] = hash_slot(row[u], scap);
        k[u] = valid[u] ? vk[s[u]] : row[u];
    }
    bool any = false;
#pragma unroll
    for (int u = 0; u < NI; u++) {
        need[u] = k[u] != row[u];
        any |= need[u];
    }
    while (__any_sync(FULL, any)) {
        passes++;
        int claims = 0;
        any = false;
#pragma unroll
        for (int u = 0; u < NI; u++) {
            if (need[u]) {
                if (k[u] == kEmptyKey) {
                    const int old = atomicCAS(&keys[s[u]], kEmptyKey, row[u]);
                    if (old == kEmptyKey) {
                        claims++;
                        need[u] = false;
                    } else {
                        k[u] = old;  // taken by another lane / item: re-examine
                        need[u] = old != row[u];
                    }
                } else {
                    s[u] = (s[u] + probe_step(row[u], scap)) & (scap - 1);
                    k[u] = vk[s[u]];
                    need[u] = k[u] != row[u];
                }
            }
            any |= need[u];
        }
        fill += __reduce_add_sync(FULL, claims);
        if (fill > limit) return false;
    }
    if (MODE != kSym) {
        __syncwarp();
#pragma unroll
        for (int u = 0; u < NI; u++) {
            if (valid[u]) vals[s[u]] += v[u];
            __syncwarp();
        }
    }
    return true;
}



// Resident CTAs per SM that a private-family bin's table allows (table + ~3 KB static
// shared memory out of 228 KB, at most 2048 threads): the launch bound then gives the
// compiler 65536 / (that x NT) registers -- occupancy is set by the table anyway -- so the
// software-pipelined gathers stay in registers.
template <int CAP, int NT, int MODE, bool GLOBAL, bool ATOMIC>
constexpr int bin_min_blocks() {
    if (ATOMIC) return 1024 / NT > 32 ? 32 : 1024 / NT;
    if (GLOBAL) return 2048 / NT / 2;
    const int tbl = CAP * (MODE == kSym ? 4 : 8) + 3072;
    int b = (228 * 1024) / tbl;
    b = b < 2048 / NT ? b : 2048 / NT;
    b = b < 32 ? b : 32;
    return b < 1 ? 1 : b;
}

template <int CAP, int NT, int MODE, bool GLOBAL, bool ATOMIC>
__global__ void __launch_bounds__(NT, (bin_min_blocks<CAP, NT, MODE, GLOBAL, ATOMIC>())) k_bin(BinArgs a) {
    using V = typename std::conditional<GLOBAL, double, float>::type;
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ unsigned hist[256];
    __shared__ int sint[4];
    __shared__ double sred[NT / 32];
    __shared__ int sscan[NT / 32];
    __shared__ int s_col, s_idx, s_ovf, s_pr;
    __shared__ int swi[2][NT / 32];
    __shared__ double swd[4][NT / 32];
    constexpr int W = NT / 32;         // warps = row-range owners
    constexpr int PSTEP = kParts / W;  // rowpart boundaries per warp
    // the private slices' double-hashing probe walks a full cycle only on a power-of-two
    // slice, and the warps split the 32 rowparts evenly (MCLX_NT* overrides must keep this)
    static_assert(ATOMIC || GLOBAL || (((CAP / W) & (CAP / W - 1)) == 0 && kParts % W == 0),
                  "private-family bins need CAP / W a power of two and W | kParts");

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
            if (MODE == kPart) s_pr = idx < count ? a.item_pr[idx] : 0;
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
        if constexpr (!GLOBAL) {  // 16-byte stores (CAP is a multiple of 4 NT; dsm is aligned)
            int4 *k4 = reinterpret_cast<int4 *>(keys);
            float4 *v4 = reinterpret_cast<float4 *>(vals);
            for (uint32_t i = tid; i < CAP / 4; i += NT) {
                k4[i] = make_int4(kEmptyKey, kEmptyKey, kEmptyKey, kEmptyKey);
                if (MODE != kSym) v4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        } else {
            for (uint32_t i = tid; i < cap; i += NT) {
                keys[i] = kEmptyKey;
                if (MODE != kSym) vals[i] = V(0);
            }
        }
        __syncthreads();

        int fresh = 0;
        bool ok = true;
        if constexpr (ATOMIC) {
            // ---- short segments (R-MAT-like): CTA-shared table, groups of g lanes per
            // segment, integer-CAS claims and float atomicAdd values (insert4b)
            __shared__ int64_t st_start[NT];
            __shared__ int st_k[NT];
            __shared__ float st_b[NT];
            __shared__ int s_fill[1];
            __shared__ int s_next[2];
            if (tid == 0) s_fill[0] = 0;
            __syncthreads();
            // ---- accumulate C_*j = sum_k b_kj A_*k.  Each lane gathers 4 consecutive
            // (row, val) pairs of a segment with one 16-byte load each (segment starts are
            // aligned down to 4 elements and the head / tail masked).
            const int limit = (int)(cap - (cap >> 3));
            const int64_t bj = a.cb + col;
            const int64_t q0 = a.bcp[bj], q1 = a.bcp[bj + 1];
            volatile int *vovf = &s_ovf;
            __shared__ int s_nl, s_ns, s_sumS;
            for (int64_t c0 = q0; c0 < q1; c0 += NT) {
                const int cnt = (int)((q1 - c0) < NT ? (q1 - c0) : NT);
                if (tid == 0) {
                    s_nl = 0;
                    s_ns = 0;
                    s_sumS = 0;
                }
                __syncthreads();
                // descriptors, split in two classes (R-MAT columns mix hub segments of
                // thousands of entries with 1-3 entry ones): long segments listed from the
                // front and walked by whole warps, short ones from the back with a group size
                // from their own mean length; empty (part) segments dropped
                if (tid < cnt) {
                    const int k = __ldg(a.brow + c0 + tid);
                    const int64_t st = __ldg(a.acp + k);
                    int64_t s0 = st;
                    int len;
                    if (MODE == kPart) {
                        // the part's rows: positions [rowpart[k][p0], rowpart[k][p1]) of A_*k
                        const int *pk = a.rowpart + (int64_t)k * (kParts + 1);
                        const int r0 = __ldg(pk + (s_pr & 0xff)), r1 = __ldg(pk + (s_pr >> 8));
                        s0 = st + r0;
                        len = r1 - r0;
                    } else {
                        len = (int)(__ldg(a.acp + k + 1) - st);  // segment length
                    }
                    if (len > 0) {
                        int slot;
                        if (len >= kLongSeg) {
                            slot = atomicAdd(&s_nl, 1);
                        } else {
                            slot = NT - 1 - atomicAdd(&s_ns, 1);
                            atomicAdd(&s_sumS, len);
                        }
                        st_start[slot] = s0;
                        st_k[slot] = len;
                        st_b[slot] = __ldg(a.bval + c0 + tid);
                    }
                }
                if (tid == 0) {
                    s_next[0] = 0;
                    s_next[1] = 0;
                }
                __syncthreads();
                const int nl = s_nl, ns = s_ns;
                const int gS = group_size_for(ns > 0 ? s_sumS / (4 * ns) : 0);
                // one group of g lanes per segment, 4 consecutive entries per lane per step
                // (16-byte gathers from the 4-aligned base, head / tail masked)
                auto walk = [&](int g, int e, bool has) {
                    const int lane_g = lane & (g - 1);
                    int lo = 0, hi = 0;  // valid element window relative to the aligned base
                    float bkj = 0.f;
                    const int *rp = a.arow;
                    const float *vp = a.aval;
                    if (has) {
                        const int64_t t0 = st_start[e];
                        const int64_t ab = t0 & ~(int64_t)3;
                        rp = a.arow + ab;
                        vp = a.aval + ab;
                        lo = (int)(t0 - ab);
                        hi = lo + st_k[e];
                        bkj = st_b[e];
                    }
                    const int lg = 31 - __clz(4 * g);  // g is a power of two: no division
                    const unsigned nstep = (unsigned)((hi + 4 * g - 1) >> lg);
                    const unsigned maxs = __reduce_max_sync(0xffffffffu, nstep);
                    for (unsigned si = 0; si < maxs; si++) {
                        const int i0 = 4 * ((int)si * g + lane_g);
                        int4 r4 = make_int4(-1, -1, -1, -1);
                        float4 v4 = make_float4(0.f, 0.f, 0.f, 0.f);
                        if (i0 < hi) {
                            r4 = __ldg(reinterpret_cast<const int4 *>(rp + i0));
                            if (MODE != kSym) v4 = __ldg(reinterpret_cast<const float4 *>(vp + i0));
                        }
                        const int rr[4] = {r4.x, r4.y, r4.z, r4.w};
                        V pv[4];
                        bool vld[4];
    #pragma unroll
                        for (int j = 0; j < 4; j++) {
                            vld[j] = i0 + j >= lo && i0 + j < hi;
                            pv[j] = GLOBAL ? (V)(&v4.x)[j] * (V)bkj : (V)((&v4.x)[j] * bkj);
                        }
                        if (!insert4b<MODE, V>(keys, vals, cap, rr, pv, vld, &s_fill[0], limit, fresh)) {
                            ok = false;
                            *vovf = 1;
                        }
                        if (!__all_sync(0xffffffffu, ok)) break;
                    }
                    ok = __all_sync(0xffffffffu, ok);
                };
                // segments are handed out dynamically, so warps that drew short segments take
                // more instead of idling at the batch barrier: long ones one per warp (g = 32),
                // then short ones 32/gS per warp
                for (;;) {
                    int e0 = 0;
                    if (lane == 0) e0 = atomicAdd(&s_next[0], 1);
                    e0 = __shfl_sync(0xffffffffu, e0, 0);
                    if (e0 >= nl || !ok) break;  // warp-uniform
                    if (*vovf) {
                        ok = false;
                        break;
                    }
                    walk(32, e0, true);
                }
                for (;;) {
                    int e0 = 0;
                    if (lane == 0) e0 = atomicAdd(&s_next[1], 32 / gS);
                    e0 = __shfl_sync(0xffffffffu, e0, 0);
                    if (e0 >= ns || !ok) break;  // warp-uniform
                    if (*vovf) {
                        ok = false;
                        break;
                    }
                    const int es = e0 + lane / gS;
                    walk(gS, NT - 1 - es, es < ns);
                }
                __syncthreads();
            }

        } else {
            // ---- accumulate C_*j = sum_k b_kj A_*k: warp `warp` handles rows of its range
            unsigned prof_passes = 0, prof_calls = 0, prof_valid = 0;
#ifdef MCLX_PROF
            const long long prof_t0 = clock64();
#endif
            const uint32_t scap = cap / W;
            int *wkeys = keys + (size_t)warp * scap;
            V *wvals = vals + (size_t)warp * scap;
            const int limit = (int)(scap - (scap >> 3));
            const int64_t bj = a.cb + col;
            const int64_t q0 = a.bcp[bj], q1 = a.bcp[bj + 1];
            int fill = 0;
            // Software pipeline over batches.  A batch is kItems sub-segments side by side,
            // 32 rows of each (chunk c); a group is 32 consecutive segments of B_*j whose
            // descriptors (this warp's sub-segment: start, length, b_kj) sit one per lane.
            // The gathers of batch i+1 -- and the descriptor loads of the group after the
            // next -- are issued before batch i is inserted, so each warp always has a
            // batch of loads in flight while it works on the hash table.
            // A positions as 32-bit offsets (the host routes A with nnz >= 2^32 to the
            // CTA-shared family): one shuffle per descriptor and one IMAD.WIDE per gather
            auto load_desc = [&](int64_t g, uint32_t &dlo, int &dlen, float &db) {
                dlo = 0;
                dlen = 0;
                db = 0.f;
                if (g + lane < q1) {
                    const int k = __ldg(a.brow + g + lane);
                    const int64_t base = __ldg(a.acp + k);
                    if (MODE == kPart) {
                        // a split part: the warps divide its fine rowparts [4 p0, 4 p1)
                        constexpr int F = kFineParts / kParts;
                        const int pp0 = F * (s_pr & 0xff), pstep = (F * (s_pr >> 8) - pp0) / W;
                        const int *pk = a.rowpart_fine + (int64_t)k * (kFineParts + 1) + pp0 + warp * pstep;
                        const int p0 = __ldg(pk), p1 = __ldg(pk + pstep);
                        dlo = (uint32_t)(base + p0);
                        dlen = p1 - p0;
                    } else if (W == 1) {
                        dlo = (uint32_t)base;
                        dlen = (int)(__ldg(a.acp + k + 1) - base);
                    } else {
                        const int *pk = a.rowpart + (int64_t)k * (kParts + 1) + warp * PSTEP;
                        const int p0 = __ldg(pk), p1 = __ldg(pk + PSTEP);
                        dlo = (uint32_t)(base + p0);
                        dlen = p1 - p0;
                    }
                    db = __ldg(a.bval + g + lane);
                }
            };
            // batch at (group g, first segment eb, chunk c) -> registers; returns the
            // longest sub-segment of the batch (chunks continue while c + 32 < it)
            auto fetch = [&](int64_t g, int eb, int c, uint32_t dlo, int dlen, float db, int (&rr)[kItems],
                             float (&av)[kItems], float (&bb)[kItems]) {
                const int ncnt = (int)((q1 - g) < 32 ? (q1 - g) : 32);
                const int t = c + lane;
                int ml = 0;
    #pragma unroll
                for (int u = 0; u < kItems; u++) {
                    const int e = eb + u;
                    const uint32_t lo = __shfl_sync(0xffffffffu, dlo, e & 31);
                    int len = __shfl_sync(0xffffffffu, dlen, e & 31);
                    bb[u] = __shfl_sync(0xffffffffu, db, e & 31);
                    if (e >= ncnt) len = 0;
                    ml = len > ml ? len : ml;
                    const bool v = t < len;
                    const uint32_t q = lo + (uint32_t)t;
                    // one 8-byte gather of the interleaved (row, value) pair (+4% on C3 over
                    // separate row / value loads)
                    const int2 pv = v ? __ldg(a.apair + q) : make_int2(-1, 0);
                    rr[u] = pv.x;
                    av[u] = __int_as_float(pv.y);
                }
                return ml;
            };
            int64_t g = q0;
            uint32_t clo, nlo;
            int clen, nlen;
            float cdb, ndb;
            load_desc(g, clo, clen, cdb);
            load_desc(g + 32, nlo, nlen, ndb);
            int eb = 0, c = 0;
            int rr[kItems];
            float av[kItems], bb[kItems];
            int ml = g < q1 ? fetch(g, eb, c, clo, clen, cdb, rr, av, bb) : 0;
            // one pipeline step: fetch the next batch into (nr, na, nb), insert the current
            // one from (cr, ca, cb).  The loop below runs it twice per trip with the two
            // register sets swapped, so no batch is copied between them.
            auto step = [&](int (&cr)[kItems], float (&ca)[kItems], float (&cb)[kItems],
                            int (&nr)[kItems], float (&na)[kItems], float (&nb)[kItems]) {
                // position of the next batch
                int neb = eb, nc = c + 32;
                int64_t ng = g;
                if (nc >= ml) {
                    nc = 0;
                    neb = eb + kItems;
                    const int ncnt = (int)((q1 - g) < 32 ? (q1 - g) : 32);
                    if (neb >= ncnt) {
                        neb = 0;
                        ng = g + 32;
                        clo = nlo;
                        clen = nlen;
                        cdb = ndb;
                        load_desc(ng + 32, nlo, nlen, ndb);
                    }
                }
                const int nml = ng < q1 ? fetch(ng, neb, nc, clo, clen, cdb, nr, na, nb) : 0;
                // insert the current batch
                bool vl[kItems];
                V vv[kItems];
    #pragma unroll
                for (int u = 0; u < kItems; u++) {
                    vl[u] = cr[u] >= 0;
                    vv[u] = GLOBAL ? (V)ca[u] * (V)cb[u] : (V)(ca[u] * cb[u]);
                }
#ifdef MCLX_PROF
    #pragma unroll
                for (int u = 0; u < kItems; u++) {
                    prof_calls++;
                    prof_valid += __popc(__ballot_sync(0xffffffffu, vl[u]));
                }
#endif
                if (!warp_insert_n<MODE, V, kItems>(wkeys, wvals, scap, vl, cr, vv, fill, limit,
                                                    prof_passes))
                    ok = false;
                g = ng;
                eb = neb;
                c = nc;
                ml = nml;
            };
            int rr2[kItems];
            float av2[kItems], bb2[kItems];
            while (g < q1 && ok) {
                step(rr, av, bb, rr2, av2, bb2);
                if (!(g < q1 && ok)) break;
                step(rr2, av2, bb2, rr, av, bb);
            }
            fresh = lane == 0 ? fill : 0;
#ifdef MCLX_PROF
            if (lane == 0) {
                PROF_ADD(0, prof_calls);
                PROF_ADD(1, prof_passes);
                PROF_ADD(2, prof_valid);
                PROF_ADD(3, clock64() - prof_t0);
            }
#else
            (void)prof_passes;
            (void)prof_calls;
            (void)prof_valid;
#endif
        }
        if (!ok && lane == 0) s_ovf = 1;
        __syncthreads();
        if (s_ovf) {
            if (tid == 0) {
                if (MODE == kPart) {
                    // the whole split column is re-run (once, whichever part overflowed)
                    a.stg_cnt[idx] = 0;
                    if (atomicExch(&a.col_flag[col], 1) == 0)
                        a.retry_list[atomicAdd(a.retry_count, 1)] = col;
                } else {
                    a.retry_list[atomicAdd(a.retry_count, 1)] = col;
                }
            }
            continue;  // loop head re-syncs before s_col is rewritten
        }

        if (MODE == kSym) {
            const int nnz = block_sum<NT, int>(fresh, sscan);
            if (tid == 0) a.sym_nnz[col] = nnz;
            __syncthreads();
            continue;
        }

#ifdef MCLX_PROF
        const long long prof_e0 = clock64();
        if (tid == 0) PROF_ADD(5, 1);
#endif
        if constexpr (!ATOMIC) {
            // ---- warp-local epilogue: warp `warp` owns slice [warp*scap, +scap) and an
            // ordered row range, so it compacts, selects its part of the kept set, sorts it
            // and writes it at its offset; only the branch decision, the radix-select
            // histograms and the sums are CTA-wide.
            const uint32_t scap = cap / W;
            int *wk = keys + (size_t)warp * scap;
            V *wv = vals + (size_t)warp * scap;
            int cnt_w = warp_compact<V>(wk, wv, (int)scap,
                                        [](int k, V) { return k != kEmptyKey; });
#ifdef MCLX_PROF
            if (tid == 0) PROF_ADD(6, clock64() - prof_e0);  // compaction of the slices
            const long long prof_e1 = clock64();
#endif
            // candidate mode (kFused, cand_k > 0): the kPart candidate epilogue per column
            const bool candm = MODE == kFused && a.cand_k > 0;
            const int64_t sidx = MODE == kPart ? idx : col;
            if ((MODE == kPart || candm) && a.cand_k > 0) {
                // candidates: statistics of all the part's entries, then each warp keeps its
                // slice's share of the part's top-cand_k (segmented radix select)
                const double theta = a.pp.theta;
                int mloc = 0;
                double sloc = 0.0;
                for (int i = lane; i < cnt_w; i += 32) {
                    const double v = (double)(float)wv[i];
                    if (v >= theta) {
                        mloc++;
                        sloc += v;
                    }
                }
                mloc = warp_sum(mloc);
                sloc = warp_sum(sloc);
                if (lane == 0) {
                    swi[0][warp] = cnt_w;
                    swi[1][warp] = mloc;
                    swd[0][warp] = sloc;
                }
                __syncthreads();
                int nnz = 0, m = 0;
                double sm = 0.0;
                for (int w2 = 0; w2 < W; w2++) {
                    nnz += swi[0][w2];
                    m += swi[1][w2];
                    sm += swd[0][w2];
                }
                if (tid == 0) {
                    a.stg_nnz[sidx] = nnz;
                    a.stg_m[sidx] = m;
                    a.stg_s[sidx] = sm;
                }
                if (nnz > a.cand_k) {
                    uint32_t t = 0;
                    int rowcut = 0;
                    radix_select_topk_seg<NT, V>(wk, wv, cnt_w, a.cand_k, t, rowcut, hist, sint);
                    cnt_w = warp_compact<V>(wk, wv, cnt_w, [=](int k, V v) {
                        const uint32_t b = val_bits(v);
                        return b > t || (b == t && k <= rowcut);
                    });
                }
                __syncthreads();  // swi reuse below
            }
            if (MODE == kNum || MODE == kPart || candm) {
                if (lane == 0) swi[0][warp] = cnt_w;
                __syncthreads();
                int off = 0, tot = 0;
                for (int w2 = 0; w2 < W; w2++) {
                    off += w2 < warp ? swi[0][w2] : 0;
                    tot += swi[0][w2];
                }
                int32_t *orow;
                float *oval;
                if (MODE == kNum) {
                    const int64_t dst = a.c_cp[col];
                    if (a.c_cnt) {  // capacity slots: record the count (<= min(f_j, m))
                        if (tid == 0) a.c_cnt[col] = tot;
                    } else if (tid == 0 && a.c_cp[col + 1] - dst != tot) {
                        atomicExch(a.err_flag, 1);
                    }
                    orow = a.c_row + dst;
                    oval = a.c_val + dst;
                } else if (candm) {  // the column's staging slot (tot <= min(cand_k, f_j, m))
                    orow = a.s_row + a.soff[col];
                    oval = a.s_val + a.soff[col];
                    if (tid == 0) {
                        a.s_cnt[col] = tot;
                        atomicAdd(a.bin_out, (unsigned long long)tot);
                    }
                } else {  // split part: its staging slot (tot <= the 7/8 fill limit)
                    orow = a.stg_row + a.stg_off[idx];
                    oval = a.stg_val + a.stg_off[idx];
                    if (tid == 0) a.stg_cnt[idx] = tot;
                }
                warp_sort_write<V>(wk, wv, cnt_w, (int)scap, orow + off, oval + off,
                                   [](V v) { return (float)v; });
                __syncthreads();
                continue;
            }
            const PruneParams &pp = a.pp;
            int mloc = 0;
            double sloc = 0.0;
            for (int i = lane; i < cnt_w; i += 32) {
                const double v = (double)wv[i];
                if (v >= pp.theta) {
                    mloc++;
                    sloc += v;
                }
            }
            mloc = warp_sum(mloc);
            sloc = warp_sum(sloc);
            if (lane == 0) {
                swi[0][warp] = cnt_w;
                swi[1][warp] = mloc;
                swd[0][warp] = sloc;
            }
            __syncthreads();
            int nnz = 0, m = 0;
            double sm = 0.0;
            for (int w2 = 0; w2 < W; w2++) {
                nnz += swi[0][w2];
                m += swi[1][w2];
                sm += swd[0][w2];
            }
            int64_t K;
            const int br = prune_branch(pp, nnz, m, sm, K);
            uint32_t t = 0;
            int rowcut = 0;
            int sel = 0;  // 0: v >= theta, 1: top-K, 2: all
            if (br == 0) {
                sel = 0;
            } else if (K >= nnz) {
                sel = 2;
            } else {
                radix_select_topk_seg<NT, V>(wk, wv, cnt_w, (int)K, t, rowcut, hist, sint);
                sel = 1;
            }
            const double theta = pp.theta;
            const int kept_w = warp_compact<V>(wk, wv, cnt_w, [=](int k, V v) {
                if (sel == 0) return (double)v >= theta;
                if (sel == 2) return true;
                const uint32_t bb = val_bits(v);
                return bb > t || (bb == t && k <= rowcut);
            });
#ifdef MCLX_PROF
            if (tid == 0) PROF_ADD(7, clock64() - prof_e1);  // stats + select + kept
            const long long prof_e2 = clock64();
#endif
            double sv = 0.0, mx = 0.0, sq = 0.0, sr = 0.0;
            for (int i = lane; i < kept_w; i += 32) {
                const double v = (double)wv[i];
                sv += v;
                mx = v > mx ? v : mx;
                sq += v * v;
                sr += pow_r(v, pp);
            }
            sv = warp_sum(sv);
            mx = warp_max(mx);
            sq = warp_sum(sq);
            sr = warp_sum(sr);
            __syncthreads();  // swi / swd reuse
            if (lane == 0) {
                swi[0][warp] = kept_w;
                swd[0][warp] = sv;
                swd[1][warp] = mx;
                swd[2][warp] = sq;
                swd[3][warp] = sr;
            }
            __syncthreads();
            int off = 0, kept = 0;
            sv = 0.0;
            mx = 0.0;
            sq = 0.0;
            sr = 0.0;
            for (int w2 = 0; w2 < W; w2++) {
                off += w2 < warp ? swi[0][w2] : 0;
                kept += swi[0][w2];
                sv += swd[0][w2];
                mx = swd[1][w2] > mx ? swd[1][w2] : mx;
                sq += swd[2][w2];
                sr += swd[3][w2];
            }
            if (tid == 0 && kept != (int)K) atomicExch(a.err_flag, 2);
            const float chaos =
                kept > 0 ? (float)((double)kept * (mx / sv - sq / (sv * sv))) : 0.0f;
            const int64_t dst = a.soff[col] + off;
#ifdef MCLX_PROF
            if (tid == 0) PROF_ADD(8, clock64() - prof_e2);  // sums
            const long long prof_e3 = clock64();
#endif
            warp_sort_write<V>(wk, wv, kept_w, (int)scap, a.s_row + dst, a.s_val + dst,
                               [&](V v) { return (float)(pow_r((double)v, pp) / sr); });
            if (tid == 0) {
                a.s_cnt[col] = kept;
                a.chaos[col] = chaos;
                atomicAdd(a.bin_out, (unsigned long long)kept);
                atomic_max_nonneg_float(a.chaos_max, chaos);
#ifdef MCLX_PROF
                PROF_ADD(4, clock64() - prof_e0);
                PROF_ADD(9, clock64() - prof_e3);  // sort + write
#endif
            }
            __syncthreads();
        } else {
            // ---- compact occupied slots to the front of the table
            const int nnz = compact_inplace<NT, V>(
                keys, vals, (int)cap, [](int k, V) { return k != kEmptyKey; }, sscan);

            if (MODE == kNum) {
                const int64_t dst = a.c_cp[col];
                if (a.c_cnt) {
                    if (tid == 0) a.c_cnt[col] = nnz;
                } else if (tid == 0 && a.c_cp[col + 1] - dst != nnz) {
                    atomicExch(a.err_flag, 1);
                }
                sort_write<NT, V>(keys, vals, nnz, (int)cap, a.c_row + dst, a.c_val + dst,
                                  [](V v) { return (float)v; }, sscan);
                continue;
            }
            const bool candm = MODE == kFused && a.cand_k > 0;
            if (MODE == kPart || candm) {
                // nnz <= the 7/8 fill limit <= stg_cap.  With candidates: statistics of all
                // entries, then only the part's top-cand_k are sorted and staged.  Candidate
                // mode: the same per output column, into the column's slot.
                const int64_t sidx = MODE == kPart ? idx : col;
                int keep = nnz;
                if (a.cand_k > 0) {
                    const double theta = a.pp.theta;
                    int mloc = 0;
                    double sloc = 0.0;
                    for (int i = tid; i < nnz; i += NT) {
                        const double v = (double)(float)vals[i];
                        if (v >= theta) {
                            mloc++;
                            sloc += v;
                        }
                    }
                    const int m = block_sum<NT, int>(mloc, sscan);
                    const double sm = block_sum<NT, double>(sloc, sred);
                    if (tid == 0) {
                        a.stg_nnz[sidx] = nnz;
                        a.stg_m[sidx] = m;
                        a.stg_s[sidx] = sm;
                    }
                    if (nnz > a.cand_k) {
                        uint32_t t = 0;
                        int rowcut = 0;
                        radix_select_topk<NT, V>(keys, vals, nnz, a.cand_k, t, rowcut, hist, sint);
                        keep = compact_inplace<NT, V>(
                            keys, vals, nnz,
                            [=](int k, V v) {
                                const uint32_t b = val_bits(v);
                                return b > t || (b == t && k <= rowcut);
                            },
                            sscan);
                    }
                }
                const int64_t dst = candm ? a.soff[col] : a.stg_off[idx];
                sort_write<NT, V>(keys, vals, keep, (int)cap, (candm ? a.s_row : a.stg_row) + dst,
                                  (candm ? a.s_val : a.stg_val) + dst, [](V v) { return (float)v; },
                                  sscan);
                if (tid == 0) {
                    if (candm) {
                        a.s_cnt[col] = keep;
                        atomicAdd(a.bin_out, (unsigned long long)keep);
                    } else {
                        a.stg_cnt[idx] = keep;
                    }
                }
                continue;
            }

    #ifdef MCLX_PROF
            if (tid == 0) PROF_ADD(6, clock64() - prof_e0);  // compaction of the table
            const long long prof_e1 = clock64();
    #endif
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

    #ifdef MCLX_PROF
            if (tid == 0) PROF_ADD(7, clock64() - prof_e1);  // stats + select + kept compaction
            const long long prof_e2 = clock64();
    #endif
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
    #ifdef MCLX_PROF
            if (tid == 0) PROF_ADD(8, clock64() - prof_e2);  // sums
            const long long prof_e3 = clock64();
    #endif
            sort_write<NT, V>(keys, vals, kept, (int)cap, a.s_row + dst, a.s_val + dst,
                              [&](V v) { return (float)(pow_r((double)v, pp) / sr); }, sscan);
            if (tid == 0) {
                a.s_cnt[col] = kept;
                a.chaos[col] = chaos;
                atomicAdd(a.bin_out, (unsigned long long)kept);
                atomic_max_nonneg_float(a.chaos_max, chaos);
    #ifdef MCLX_PROF
                PROF_ADD(4, clock64() - prof_e0);
                PROF_ADD(9, clock64() - prof_e3);  // sort + write
    #endif
            }
            __syncthreads();
        }
    }
}

void prof_read(unsigned long long out[12], int reset) {
    cudaMemcpyFromSymbol(out, g_prof, sizeof(unsigned long long) * 12);
    if (reset) {
        unsigned long long z[12] = {};
        cudaMemcpyToSymbol(g_prof, z, sizeof z);
    }
}

template <int CAP, int NT, int MODE, bool GLOBAL, bool ATOMIC>
static size_t smem_of() {
    if (GLOBAL) return 0;
    return (size_t)CAP * (MODE == kSym ? 4 : 8);
}

template <int CAP, int NT, int MODE, bool GLOBAL, bool ATOMIC>
static int occ_of() {
    auto fn = k_bin<CAP, NT, MODE, GLOBAL, ATOMIC>;
    size_t sm = smem_of<CAP, NT, MODE, GLOBAL, ATOMIC>();
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, NT, sm);
    return nb;
}

template <int CAP, int NT, int MODE, bool GLOBAL, bool ATOMIC>
static cudaError_t launch_of(const BinArgs &a, int grid, cudaStream_t s) {
    ++g_launches;
    k_bin<CAP, NT, MODE, GLOBAL, ATOMIC><<<grid, NT, smem_of<CAP, NT, MODE, GLOBAL, ATOMIC>(), s>>>(a);
    return cudaGetLastError();
}

// threads of the private-family bins 3-5 (development overrides: -DMCLX_NT3=... etc.)
#ifndef MCLX_NT3
#define MCLX_NT3 128
#endif
#ifndef MCLX_NT4
#define MCLX_NT4 256
#endif
#ifndef MCLX_NT5
#define MCLX_NT5 512
#endif
#define MCLX_BIN_SWITCH(MODE, WHAT, ...)                                          \
    switch (bin) {                                                                \
        case 0: return WHAT<512, 32, MODE, false, false>(__VA_ARGS__);            \
        case 1: return WHAT<1024, 32, MODE, false, false>(__VA_ARGS__);           \
        case 2: return WHAT<2048, 64, MODE, false, false>(__VA_ARGS__);           \
        case 3: return WHAT<4096, MCLX_NT3, MODE, false, false>(__VA_ARGS__);       \
        case 4: return WHAT<8192, MCLX_NT4, MODE, false, false>(__VA_ARGS__);       \
        case 5: return WHAT<16384, MCLX_NT5, MODE, false, false>(__VA_ARGS__);       \
        case 6: return WHAT<0, kGlobalThreads, MODE, true, false>(__VA_ARGS__);   \
        case 7: return WHAT<512, 64, MODE, false, true>(__VA_ARGS__);             \
        case 8: return WHAT<1024, 64, MODE, false, true>(__VA_ARGS__);            \
        case 9: return WHAT<2048, 128, MODE, false, true>(__VA_ARGS__);           \
        case 10: return WHAT<4096, 256, MODE, false, true>(__VA_ARGS__);          \
        case 11: return WHAT<8192, 512, MODE, false, true>(__VA_ARGS__);          \
        case 12: return WHAT<16384, 1024, MODE, false, true>(__VA_ARGS__);        \
        default: return WHAT<0, kGlobalThreads, MODE, true, true>(__VA_ARGS__);   \
    }

cudaError_t launch_bin(int mode, int bin, const BinArgs &a, int grid, cudaStream_t s) {
    if (mode == kSym) { MCLX_BIN_SWITCH(kSym, launch_of, a, grid, s) }
    if (mode == kNum) { MCLX_BIN_SWITCH(kNum, launch_of, a, grid, s) }
    MCLX_BIN_SWITCH(kFused, launch_of, a, grid, s)
}

cudaError_t launch_part(int variant, const BinArgs &a, int grid, cudaStream_t s) {
    if (variant == 0) return launch_of<kPartCap, kPartThreads, kPart, false, true>(a, grid, s);
    if (variant == 1) return launch_of<2 * kPartCap, 2 * kPartThreads, kPart, false, true>(a, grid, s);
    // private row-range slices (bin 4 configuration): parts of >= 8 fine rowparts
    return launch_of<kPartCap, kPartCap / 32, kPart, false, false>(a, grid, s);
}
int part_occupancy(int variant) {
    if (variant == 0) return occ_of<kPartCap, kPartThreads, kPart, false, true>();
    if (variant == 1) return occ_of<2 * kPartCap, 2 * kPartThreads, kPart, false, true>();
    return occ_of<kPartCap, kPartCap / 32, kPart, false, false>();
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
