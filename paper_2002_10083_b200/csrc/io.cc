// io.cc -- the I/O around the kernel (SPEC S:547-559 load_graph / run):
// host-side ingestion of a weighted graph into CSC and the cluster output file.  Plain C++17,
// no CUDA: the arrays it returns are host memory the caller uploads (e.g. CSC.from_host).
//
// Input formats (detected from the first line):
//   * MatrixMarket coordinate, "%%MatrixMarket matrix coordinate real|integer|pattern
//     general|symmetric"; 1-based indices; pattern entries get value 1.0; a symmetric file
//     lists the lower triangle (i >= j; an entry above the diagonal is a "symmetric-marker
//     violation") and is expanded;
//   * labelled TSV edge list "src<TAB or space>dst[<TAB>weight]" (weight 1.0 when absent);
//     labels are mapped to dense ids in order of first appearance (the networks of Table I,
//     P:729-749, are "proteins" and "connections").
// Duplicated (i, j) entries are summed and entries whose sum is exactly 0 dropped.
// symmetrize != 0 then returns max(A, A^T) entrywise (an undirected similarity graph given
// one direction per edge; idempotent on symmetric input).  Errors: a malformed line (with
// its number), a negative weight, a non-square matrix, an index out of bounds.
#include <algorithm>
#include <cerrno>
#include <cstdarg>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "mclx.h"

namespace {

struct Triple {
    int64_t i, j;
    double w;
};

int err_out(char *err, size_t errlen, int code, const char *fmt, ...) __attribute__((format(printf, 4, 5)));
int err_out(char *err, size_t errlen, int code, const char *fmt, ...) {
    if (err && errlen) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(err, errlen, fmt, ap);
        va_end(ap);
    }
    return code;
}

// CSC of n x n from triples: sort by (j, i), sum duplicates, drop exact zeros
void build_csc(int64_t n, std::vector<Triple> &t, std::vector<int64_t> &cp, std::vector<int32_t> &ri,
               std::vector<double> &v) {
    std::sort(t.begin(), t.end(), [](const Triple &a, const Triple &b) {
        return a.j != b.j ? a.j < b.j : a.i < b.i;
    });
    cp.assign((size_t)n + 1, 0);
    ri.clear();
    v.clear();
    for (size_t k = 0; k < t.size();) {
        size_t e = k;
        double s = 0.0;
        while (e < t.size() && t[e].i == t[k].i && t[e].j == t[k].j) s += t[e++].w;
        if (s != 0.0) {
            ri.push_back((int32_t)t[k].i);
            v.push_back(s);
            cp[(size_t)t[k].j + 1]++;
        }
        k = e;
    }
    for (int64_t j = 0; j < n; j++) cp[(size_t)j + 1] += cp[(size_t)j];
}

bool blank_or_comment(const char *s) {
    while (*s == ' ' || *s == '\t' || *s == '\r' || *s == '\n') s++;
    return *s == '\0' || *s == '%' || *s == '#';
}

}  // namespace

extern "C" {

int mcl_graph_read(const char *path, int symmetrize, mcl_graph_t *g, char *err, size_t errlen) {
    if (!path || !g) return err_out(err, errlen, MCL_ERR_INVALID_ARG, "NULL argument");
    memset(g, 0, sizeof *g);
    FILE *f = fopen(path, "r");
    if (!f) return err_out(err, errlen, MCL_ERR_INVALID_ARG, "%s: %s", path, strerror(errno));
    std::vector<Triple> t;
    std::vector<std::string> labels;
    std::unordered_map<std::string, int64_t> ids;
    int64_t n = 0;
    char *line = nullptr;
    size_t cap = 0;
    ssize_t len;
    int64_t lineno = 0;
    int rc = MCL_OK;
    bool mm = false, pattern = false, symmetric = false, have_size = false;
    int64_t declared = 0, entries = 0;
    while ((len = getline(&line, &cap, f)) >= 0) {
        lineno++;
        if (lineno == 1 && strncmp(line, "%%MatrixMarket", 14) == 0) {
            char obj[64] = {}, fmt[64] = {}, field[64] = {}, sym[64] = {};
            if (sscanf(line + 14, "%63s %63s %63s %63s", obj, fmt, field, sym) != 4 ||
                strcmp(obj, "matrix") != 0 || strcmp(fmt, "coordinate") != 0) {
                rc = err_out(err, errlen, MCL_ERR_FORMAT, "%s:1: unsupported MatrixMarket header", path);
                break;
            }
            mm = true;
            pattern = strcmp(field, "pattern") == 0;
            if (!pattern && strcmp(field, "real") != 0 && strcmp(field, "integer") != 0) {
                rc = err_out(err, errlen, MCL_ERR_FORMAT, "%s:1: field '%s' not supported", path, field);
                break;
            }
            symmetric = strcmp(sym, "symmetric") == 0;
            if (!symmetric && strcmp(sym, "general") != 0) {
                rc = err_out(err, errlen, MCL_ERR_FORMAT, "%s:1: symmetry '%s' not supported", path, sym);
                break;
            }
            continue;
        }
        if (blank_or_comment(line)) continue;
        if (mm) {
            if (!have_size) {
                long long r, cc, z;
                if (sscanf(line, "%lld %lld %lld", &r, &cc, &z) != 3 || r < 0 || cc < 0 || z < 0) {
                    rc = err_out(err, errlen, MCL_ERR_FORMAT, "%s:%lld: malformed size line", path,
                                 (long long)lineno);
                    break;
                }
                if (r != cc) {
                    rc = err_out(err, errlen, MCL_ERR_DIM, "%s: %lld x %lld is not square", path, r, cc);
                    break;
                }
                n = r;
                declared = z;
                have_size = true;
                t.reserve((size_t)z * (symmetric ? 2 : 1));
                continue;
            }
            long long i, j;
            double w = 1.0;
            const int k = pattern ? sscanf(line, "%lld %lld", &i, &j) : sscanf(line, "%lld %lld %lf", &i, &j, &w);
            if (k != (pattern ? 2 : 3)) {
                rc = err_out(err, errlen, MCL_ERR_FORMAT, "%s:%lld: malformed entry", path, (long long)lineno);
                break;
            }
            if (i < 1 || j < 1 || i > n || j > n) {
                rc = err_out(err, errlen, MCL_ERR_FORMAT, "%s:%lld: index (%lld, %lld) outside %lld x %lld",
                             path, (long long)lineno, i, j, (long long)n, (long long)n);
                break;
            }
            if (symmetric && i < j) {
                rc = err_out(err, errlen, MCL_ERR_FORMAT,
                             "%s:%lld: entry (%lld, %lld) above the diagonal of a symmetric file", path,
                             (long long)lineno, i, j);
                break;
            }
            if (!(w >= 0.0) || !std::isfinite(w)) {
                rc = err_out(err, errlen, MCL_ERR_FORMAT, "%s:%lld: negative or non-finite weight", path,
                             (long long)lineno);
                break;
            }
            entries++;
            t.push_back({i - 1, j - 1, w});
            if (symmetric && i != j) t.push_back({j - 1, i - 1, w});
        } else {
            char a[4096], b[4096];
            double w = 1.0;
            const int k = sscanf(line, "%4095s %4095s %lf", a, b, &w);
            if (k < 2) {
                rc = err_out(err, errlen, MCL_ERR_FORMAT, "%s:%lld: expected 'src dst [weight]'", path,
                             (long long)lineno);
                break;
            }
            if (!(w >= 0.0) || !std::isfinite(w)) {
                rc = err_out(err, errlen, MCL_ERR_FORMAT, "%s:%lld: negative or non-finite weight", path,
                             (long long)lineno);
                break;
            }
            int64_t id[2];
            const char *s2[2] = {a, b};
            for (int q = 0; q < 2; q++) {
                auto it = ids.find(s2[q]);
                if (it == ids.end()) {
                    id[q] = (int64_t)labels.size();
                    ids.emplace(s2[q], id[q]);
                    labels.emplace_back(s2[q]);
                } else {
                    id[q] = it->second;
                }
            }
            // column = source, row = destination
            t.push_back({id[1], id[0], w});
        }
    }
    free(line);
    fclose(f);
    if (rc != MCL_OK) return rc;
    if (mm && !have_size) return err_out(err, errlen, MCL_ERR_FORMAT, "%s: no size line", path);
    if (mm && entries != declared)
        return err_out(err, errlen, MCL_ERR_FORMAT, "%s: %lld entries, the size line declares %lld",
                       path, (long long)entries, (long long)declared);
    if (!mm) n = (int64_t)labels.size();
    if (n > 0x7ffffffeLL) return err_out(err, errlen, MCL_ERR_DIM, "%s: too many vertices", path);
    std::vector<int64_t> cp;
    std::vector<int32_t> ri;
    std::vector<double> v;
    build_csc(n, t, cp, ri, v);
    if (symmetrize) {  // max(A, A^T): add the mirror of every entry, keep the larger value
        std::vector<Triple> u;
        u.reserve(ri.size() * 2);
        for (int64_t j = 0; j < n; j++)
            for (int64_t q = cp[(size_t)j]; q < cp[(size_t)j + 1]; q++) {
                u.push_back({ri[(size_t)q], j, v[(size_t)q]});
                u.push_back({j, ri[(size_t)q], v[(size_t)q]});
            }
        std::sort(u.begin(), u.end(), [](const Triple &a, const Triple &b) {
            return a.j != b.j ? a.j < b.j : (a.i != b.i ? a.i < b.i : a.w > b.w);
        });
        u.erase(std::unique(u.begin(), u.end(),
                            [](const Triple &a, const Triple &b) { return a.i == b.i && a.j == b.j; }),
                u.end());
        build_csc(n, u, cp, ri, v);
    }
    const int64_t nnz = (int64_t)ri.size();
    g->n = n;
    g->nnz = nnz;
    g->col_ptr = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    g->row_idx = (int32_t *)malloc(sizeof(int32_t) * (size_t)std::max<int64_t>(nnz, 1));
    g->val = (float *)malloc(sizeof(float) * (size_t)std::max<int64_t>(nnz, 1));
    if (!g->col_ptr || !g->row_idx || !g->val) {
        mcl_graph_free(g);
        return err_out(err, errlen, MCL_ERR_OOM, "out of host memory");
    }
    memcpy(g->col_ptr, cp.data(), sizeof(int64_t) * (size_t)(n + 1));
    if (nnz) memcpy(g->row_idx, ri.data(), sizeof(int32_t) * (size_t)nnz);
    for (int64_t q = 0; q < nnz; q++) g->val[q] = (float)v[(size_t)q];
    if (!mm) {
        g->labels = (char **)calloc((size_t)std::max<int64_t>(n, 1), sizeof(char *));
        if (!g->labels) {
            mcl_graph_free(g);
            return err_out(err, errlen, MCL_ERR_OOM, "out of host memory");
        }
        for (int64_t i = 0; i < n; i++) g->labels[i] = strdup(labels[(size_t)i].c_str());
    }
    return MCL_OK;
}

void mcl_graph_free(mcl_graph_t *g) {
    if (!g) return;
    if (g->labels)
        for (int64_t i = 0; i < g->n; i++) free(g->labels[i]);
    free(g->labels);
    free(g->col_ptr);
    free(g->row_idx);
    free(g->val);
    memset(g, 0, sizeof *g);
}

int mcl_clusters_write(const char *path, const int32_t *labels, int64_t n, const mcl_graph_t *g) {
    if (!path || (!labels && n > 0) || n < 0) return MCL_ERR_INVALID_ARG;
    if (g && g->n != n) return MCL_ERR_DIM;
    int64_t k = 0;
    for (int64_t i = 0; i < n; i++) {
        if (labels[i] < 0 || labels[i] >= n) return MCL_ERR_INVALID_ARG;
        k = std::max<int64_t>(k, (int64_t)labels[i] + 1);
    }
    // members of each cluster in ascending vertex order (counting sort by label)
    std::vector<int64_t> start((size_t)k + 1, 0);
    for (int64_t i = 0; i < n; i++) start[(size_t)labels[i] + 1]++;
    for (int64_t c = 0; c < k; c++) start[(size_t)c + 1] += start[(size_t)c];
    std::vector<int64_t> pos(start.begin(), start.end() - 1), mem((size_t)n);
    for (int64_t i = 0; i < n; i++) mem[(size_t)pos[(size_t)labels[i]]++] = i;
    FILE *f = fopen(path, "w");
    if (!f) return MCL_ERR_INVALID_ARG;
    const bool named = g && g->labels;
    for (int64_t c = 0; c < k; c++) {
        for (int64_t q = start[(size_t)c]; q < start[(size_t)c + 1]; q++) {
            if (q > start[(size_t)c]) fputc(' ', f);
            if (named) fputs(g->labels[mem[(size_t)q]], f);
            else fprintf(f, "%lld", (long long)mem[(size_t)q] + 1);  // 1-based (MatrixMarket ids)
        }
        fputc('\n', f);
    }
    return fclose(f) == 0 ? MCL_OK : MCL_ERR_INVALID_ARG;
}

}  // extern "C"
