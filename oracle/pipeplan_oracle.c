/*
 * pipeplan_oracle.c — CPU restatement (C99, fp64) of the reference pipeplan
 * hot path.  TEST INFRASTRUCTURE ONLY (see pipeplan_oracle.h).
 *
 * Every function cites the reference lines it restates (paths relative to
 * /root/reference/proj).  Arithmetic is performed in exactly the reference's
 * order so results are bitwise equal to the compiled reference; this is
 * checked against oracle/_ref through tests/golden/.  Build with
 * -ffp-contract=off (oracle/Makefile) so no FMA contraction changes rounding.
 */
#include "pipeplan_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ errors */

static int fail(char* err, size_t errlen, int code, const char* fmt, ...) {
    if (err && errlen) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(err, errlen, fmt, ap);
        va_end(ap);
    }
    return code;
}

/* ------------------------------------------------------------ mt19937_64
 * std::mt19937_64 (ISO C++ [rand.predef]); the reference seeds it directly
 * (tinynet.cpp:181, :449). */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
    static const uint64_t MAG[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (g->idx >= 312) {
        int i;
        for (i = 0; i < 312 - 156; ++i) {
            uint64_t x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
            g->mt[i] = g->mt[i + 156] ^ (x >> 1) ^ MAG[x & 1ULL];
        }
        for (; i < 311; ++i) {
            uint64_t x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
            g->mt[i] = g->mt[i + (156 - 312)] ^ (x >> 1) ^ MAG[x & 1ULL];
        }
        uint64_t x = (g->mt[311] & UM) | (g->mt[0] & LM);
        g->mt[311] = g->mt[155] ^ (x >> 1) ^ MAG[x & 1ULL];
        g->idx = 0;
    }
    uint64_t x = g->mt[g->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* libstdc++ generate_canonical<double,53>(mt19937_64): one draw, / 2^64,
 * clamped below 1 (bits/random.tcc). */
static double canon(mt64* g) {
    double sum = (double)mt64_next(g);
    double ret = sum / 18446744073709551616.0;
    if (ret >= 1.0) ret = nextafter(1.0, 0.0);
    return ret;
}

/* ------------------------------------------------------------ init / data */

/* init_net, tinynet.cpp:176-196: per layer, weights row-major then biases,
 * each uni(-0.5,0.5) * (1/sqrt(fan_in)). */
void or_init_net(const int* dims, int L, uint64_t seed, double* W, double* b) {
    mt64 g;
    mt64_seed(&g, seed);
    size_t wo = 0, bo = 0;
    for (int l = 0; l < L; ++l) {
        const int fi = dims[l], fo = dims[l + 1];
        const double scale = 1.0 / sqrt((double)fi);
        for (long i = 0; i < (long)fo * fi; ++i) W[wo + i] = (canon(&g) * (0.5 - -0.5) + -0.5) * scale;
        for (int i = 0; i < fo; ++i) b[bo + i] = (canon(&g) * (0.5 - -0.5) + -0.5) * scale;
        wo += (size_t)fo * fi;
        bo += (size_t)fo;
    }
}

/* make_blobs, tinynet.cpp:447-461, with libstdc++ normal_distribution
 * (Marsaglia polar, one cached value). */
void or_make_blobs(int samples, int features, double separation, uint64_t seed, double* X,
                   int* labels) {
    mt64 g;
    mt64_seed(&g, seed);
    int saved_ok = 0;
    double saved = 0.0;
    for (int i = 0; i < samples; ++i) {
        const int cls = i % 2;
        labels[i] = cls;
        const double mean = cls == 0 ? -separation : separation;
        for (int j = 0; j < features; ++j) {
            double ret;
            if (saved_ok) {
                saved_ok = 0;
                ret = saved;
            } else {
                double x, y, r2;
                do {
                    x = 2.0 * canon(&g) - 1.0;
                    y = 2.0 * canon(&g) - 1.0;
                    r2 = x * x + y * y;
                } while (r2 > 1.0 || r2 == 0.0);
                const double mult = sqrt(-2 * log(r2) / r2);
                saved = x * mult;
                saved_ok = 1;
                ret = y * mult;
            }
            ret = ret * 1.0 + 0.0;
            X[(size_t)i * features + j] = mean + ret;
        }
    }
}

/* ------------------------------------------------------------ planner */

/* split_layer, partition.cpp:15-48 */
int or_split_layer(int layer_id, int fan_out, const int* devices, int n, int replicate_narrow,
                   int* lo, int* hi, int* replicated, char* err, size_t errlen) {
    (void)devices;
    if (n < 1) return fail(err, errlen, OR_INVALID, "split_layer: need at least one device");
    if (fan_out < n) {
        if (!replicate_narrow)
            return fail(err, errlen, OR_RUNTIME, "layer %d too narrow to split %d ways (fan_out %d)",
                        layer_id, n, fan_out);
        for (int k = 0; k < n; ++k) {
            lo[k] = 0;
            hi[k] = fan_out;
            replicated[k] = 1;
        }
        return OR_OK;
    }
    const int base = fan_out / n, rem = fan_out % n;
    int at = 0;
    for (int k = 0; k < n; ++k) {
        const int size = base + (k < rem ? 1 : 0);
        lo[k] = at;
        hi[k] = at + size;
        replicated[k] = 0;
        at += size;
    }
    return OR_OK;
}

/* split_microbatches, schedule.cpp:46-55 */
int or_split_microbatches(int b, int m, int* sizes, char* err, size_t errlen) {
    if (b < 1 || m < 1)
        return fail(err, errlen, OR_INVALID, "batch and micro-batch count must be >= 1");
    if (m > b)
        return fail(err, errlen, OR_RUNTIME, "micro-batch smaller than one sample (b=%d, m=%d)", b, m);
    for (int k = 0; k < m; ++k) sizes[k] = b / m;
    for (int k = 0; k < b % m; ++k) sizes[k] += 1;
    return OR_OK;
}

/* validate_model, model.cpp:38-62 (dense chain given by fan_in/fan_out) */
static int validate_chain(const int* fan_in, const int* fan_out, int L, char* err, size_t errlen) {
    if (L < 1) return fail(err, errlen, OR_RUNTIME, "model must have at least one layer");
    for (int i = 0; i < L; ++i) {
        if (fan_in[i] < 1 || fan_out[i] < 1)
            return fail(err, errlen, OR_RUNTIME, "layer %d: fan_in and fan_out must be >= 1", i + 1);
        if (i > 0 && fan_out[i - 1] != fan_in[i])
            return fail(err, errlen, OR_RUNTIME,
                        "dimension mismatch between layers %d and %d: fan_out %d vs fan_in %d", i,
                        i + 1, fan_out[i - 1], fan_in[i]);
    }
    return OR_OK;
}

/* default_costs fwd_flops, model.cpp:124-137 */
static double fwd_cost(const int* fan_in, const int* fan_out, const double* fwd, int l) {
    if (fwd && fwd[l] != 0) return fwd[l];
    const double io = (double)fan_in[l] * fan_out[l];
    return 2.0 * io;
}

/* balanced_spans, partition.cpp:55-82 */
static void balanced_spans(const int* fan_in, const int* fan_out, const double* fwd, int L, int Z,
                           int* cuts) {
    double* prefix = (double*)calloc((size_t)L + 1, sizeof(double));
    for (int l = 1; l <= L; ++l) prefix[l] = prefix[l - 1] + fwd_cost(fan_in, fan_out, fwd, l - 1);
    const double total = prefix[L];
    int prev = 0;
    for (int i = 1; i < Z; ++i) {
        const double target = total * i / Z;
        const int lo = prev + 1;
        const int hi = L - (Z - i);
        int best = lo;
        double best_err = fabs(prefix[lo] - target);
        for (int pos = lo + 1; pos <= hi; ++pos) {
            const double e = fabs(prefix[pos] - target);
            if (e < best_err) {
                best = pos;
                best_err = e;
            }
        }
        cuts[i - 1] = best;
        prev = best;
    }
    free(prefix);
}

/* plan_from_spans, partition.cpp:84-106, emitted in the flat encoding */
static int plan_from_spans(const int* fan_out, int L, const int* cuts, const int* groups,
                           const int* group_sizes, int Z, int n, int replicate_narrow, int* out,
                           int cap, int* out_len, char* err, size_t errlen) {
    int len = 2;
    for (int j = 0; j < Z; ++j) {
        const int first = j == 0 ? 1 : cuts[j - 1] + 1;
        const int last = j < Z - 1 ? cuts[j] : L;
        len += 4 + group_sizes[j] + (last - first + 1) * group_sizes[j] * 5;
    }
    len += Z - 1;
    *out_len = len;
    int* buf = (int*)malloc(sizeof(int) * (size_t)len);
    int w = 0, goff = 0, rc = OR_OK;
    buf[w++] = n;
    buf[w++] = Z;
    for (int j = 0; j < Z && rc == OR_OK; ++j) {
        const int first = j == 0 ? 1 : cuts[j - 1] + 1;
        const int last = j < Z - 1 ? cuts[j] : L;
        const int D = group_sizes[j];
        const int* devs = groups + goff;
        buf[w++] = j + 1;
        buf[w++] = first;
        buf[w++] = last;
        buf[w++] = D;
        for (int d = 0; d < D; ++d) buf[w++] = devs[d];
        int lo[512], hi[512], rep[512];
        for (int l = first; l <= last && rc == OR_OK; ++l) {
            rc = or_split_layer(l, fan_out[l - 1], devs, D, replicate_narrow, lo, hi, rep, err, errlen);
            for (int d = 0; d < D && rc == OR_OK; ++d) {
                buf[w++] = l;
                buf[w++] = devs[d];
                buf[w++] = lo[d];
                buf[w++] = hi[d];
                buf[w++] = rep[d];
            }
        }
        goff += D;
    }
    for (int k = 0; k < Z - 1; ++k) buf[w++] = 0;  /* concat_repartition */
    if (rc == OR_OK) {
        if (out && cap >= len) memcpy(out, buf, sizeof(int) * (size_t)len);
        else if (cap > 0) rc = fail(err, errlen, OR_RUNTIME, "plan buffer too small");
    }
    free(buf);
    return rc;
}

/* build_plan, partition.cpp:110-121 */
int or_build_plan(const int* fan_in, const int* fan_out, const double* fwd_flops, int L, int n,
                  int Z, int replicate_narrow, int* out, int cap, int* out_len, char* err,
                  size_t errlen) {
    int rc = validate_chain(fan_in, fan_out, L, err, errlen);
    if (rc) return rc;
    if (n < 1) return fail(err, errlen, OR_INVALID, "build_plan: n must be >= 1");
    if (Z < 1 || Z > L) return fail(err, errlen, OR_RUNTIME, "Z exceeds layer count (Z=%d, L=%d)", Z, L);
    int* cuts = (int*)malloc(sizeof(int) * (size_t)(Z > 1 ? Z : 1));
    int* groups = (int*)malloc(sizeof(int) * (size_t)Z * n);
    int* sizes = (int*)malloc(sizeof(int) * (size_t)Z);
    balanced_spans(fan_in, fan_out, fwd_flops, L, Z, cuts);
    for (int j = 0; j < Z; ++j) {
        sizes[j] = n;
        for (int d = 0; d < n; ++d) groups[j * n + d] = d + 1;
    }
    rc = plan_from_spans(fan_out, L, cuts, groups, sizes, Z, n, replicate_narrow, out, cap, out_len,
                         err, errlen);
    free(cuts);
    free(groups);
    free(sizes);
    return rc;
}

/* build_staged_plan, partition.cpp:123-138 */
int or_build_staged_plan(const int* fan_in, const int* fan_out, const double* fwd_flops, int L,
                         const int* groups, const int* group_sizes, int Z, int replicate_narrow,
                         int* out, int cap, int* out_len, char* err, size_t errlen) {
    int rc = validate_chain(fan_in, fan_out, L, err, errlen);
    if (rc) return rc;
    if (Z < 1 || Z > L) return fail(err, errlen, OR_RUNTIME, "Z exceeds layer count (Z=%d, L=%d)", Z, L);
    int n = 0, off = 0;
    for (int j = 0; j < Z; ++j) {
        if (group_sizes[j] < 1) return fail(err, errlen, OR_INVALID, "device group must not be empty");
        for (int d = 0; d < group_sizes[j]; ++d) n = groups[off + d] > n ? groups[off + d] : n;
        off += group_sizes[j];
    }
    int* cuts = (int*)malloc(sizeof(int) * (size_t)(Z > 1 ? Z : 1));
    balanced_spans(fan_in, fan_out, fwd_flops, L, Z, cuts);
    rc = plan_from_spans(fan_out, L, cuts, groups, group_sizes, Z, n, replicate_narrow, out, cap,
                         out_len, err, errlen);
    free(cuts);
    return rc;
}

/* ------------------------------------------------------------ flat plan parsing */

typedef struct {
    int first, last, D;
    const int* devs;
    const int* shards; /* [(last-first+1) * D][5] */
} sub_view;

static int parse_plan(const int* p, int len, sub_view* subs, int maxz, int* Z, const int** bounds) {
    if (len < 2) return -1;
    int r = 2;
    *Z = p[1];
    if (*Z < 1 || *Z > maxz) return -1;
    for (int j = 0; j < *Z; ++j) {
        if (r + 4 > len) return -1;
        subs[j].first = p[r + 1];
        subs[j].last = p[r + 2];
        subs[j].D = p[r + 3];
        r += 4;
        if (subs[j].D < 1 || r + subs[j].D > len) return -1;
        subs[j].devs = p + r;
        r += subs[j].D;
        const int nl = subs[j].last - subs[j].first + 1;
        if (nl < 0) return -1;
        subs[j].shards = p + r;
        r += nl * subs[j].D * 5;
        if (r > len) return -1;
    }
    if (r + *Z - 1 != len) return -1;
    *bounds = p + r;
    return 0;
}

/* merge_submodules, partition.cpp:157-175 */
int or_merge_submodules(int* plan, int plan_len, const int* group, int group_len, char* err,
                        size_t errlen) {
    sub_view subs[256];
    int Z;
    const int* bounds;
    if (parse_plan(plan, plan_len, subs, 256, &Z, &bounds) != 0)
        return fail(err, errlen, OR_INVALID, "malformed plan");
    if (group_len < 2) return fail(err, errlen, OR_RUNTIME, "merge group must have length >= 2");
    for (int i = 0; i < group_len; ++i) {
        if (group[i] < 1 || group[i] > Z)
            return fail(err, errlen, OR_RUNTIME, "merge group index %d out of range 1..%d", group[i], Z);
        if (i > 0 && group[i] != group[i - 1] + 1)
            return fail(err, errlen, OR_RUNTIME, "group must be contiguous");
    }
    int* b = plan + (bounds - plan);
    for (int i = 0; i + 1 < group_len; ++i) b[group[i] - 1] = 1;
    return OR_OK;
}

/* validate_plan, partition.cpp:232-294 */
static int validate_plan(const int* p, int len, const int* fan_out, int L, char* err, size_t errlen) {
    sub_view subs[256];
    int Z;
    const int* bounds;
    if (parse_plan(p, len, subs, 256, &Z, &bounds) != 0)
        return fail(err, errlen, OR_RUNTIME, "malformed plan encoding");
    int expect_first = 1;
    for (int j = 0; j < Z; ++j) {
        const sub_view* sm = &subs[j];
        if (sm->first != expect_first || sm->last < sm->first)
            return fail(err, errlen, OR_RUNTIME, "sub-module spans must partition 1..L in order");
        expect_first = sm->last + 1;
        for (int l = sm->first; l <= sm->last; ++l) {
            if (l > L) return fail(err, errlen, OR_RANGE, "vector::_M_range_check");
            const int* sh = sm->shards + (size_t)(l - sm->first) * sm->D * 5;
            if (sh[4]) {
                for (int d = 0; d < sm->D; ++d)
                    if (!sh[d * 5 + 4] || sh[d * 5 + 2] != 0 || sh[d * 5 + 3] != fan_out[l - 1])
                        return fail(err, errlen, OR_RUNTIME, "layer %d: inconsistent replication", l);
            } else {
                int lo = 0;
                for (int d = 0; d < sm->D; ++d) {
                    if (sh[d * 5 + 2] != lo || sh[d * 5 + 3] <= sh[d * 5 + 2])
                        return fail(err, errlen, OR_RUNTIME, "layer %d: shards must tile [0, fan_out) exactly", l);
                    lo = sh[d * 5 + 3];
                }
                if (lo != fan_out[l - 1])
                    return fail(err, errlen, OR_RUNTIME, "layer %d: shards must tile [0, fan_out) exactly", l);
            }
            for (int d = 0; d < sm->D; ++d)
                if (sh[d * 5 + 1] != sm->devs[d])
                    return fail(err, errlen, OR_RUNTIME, "layer %d: shard device order must match sub-module devices", l);
        }
    }
    if (expect_first != L + 1)
        return fail(err, errlen, OR_RUNTIME, "plan does not cover all layers (ends at %d of %d)",
                    expect_first - 1, L);
    return OR_OK;
}

/* ------------------------------------------------------------ dense math
 * Matrices are row-major double, every product an ascending-index running sum
 * from 0.0 (tinynet.hpp:11-14, tinynet.cpp:11-48). */

/* matmul_nt, tinynet.cpp:24-35: c(r x n) = a(r x k) . b(n x k)^T */
static void mm_nt(const double* a, const double* b, double* c, int r, int k, int n) {
    for (int i = 0; i < r; ++i)
        for (int j = 0; j < n; ++j) {
            double acc = 0.0;
            for (int t = 0; t < k; ++t) acc += a[(size_t)i * k + t] * b[(size_t)j * k + t];
            c[(size_t)i * n + j] = acc;
        }
}

/* matmul_tn, tinynet.cpp:37-48: c(ca x cb) = a(rows x ca)^T . b(rows x cb) */
static void mm_tn(const double* a, const double* b, double* c, int rows, int ca, int cb) {
    for (int i = 0; i < ca; ++i)
        for (int j = 0; j < cb; ++j) {
            double acc = 0.0;
            for (int t = 0; t < rows; ++t) acc += a[(size_t)t * ca + i] * b[(size_t)t * cb + j];
            c[(size_t)i * cb + j] = acc;
        }
}

/* matmul restricted to rows [lo,hi) of b and columns [lo,hi) of a
 * (matmul(delta_shard, W_shard), tinynet.cpp:11-22 at train_partitioned.cpp:515):
 * c(r x n) = a(r x K)[:, lo:hi] . b(K x n)[lo:hi, :] */
static void mm_nn_slice(const double* a, int K, const double* b, double* c, int r, int n, int lo,
                        int hi) {
    for (int i = 0; i < r; ++i)
        for (int j = 0; j < n; ++j) {
            double acc = 0.0;
            for (int t = lo; t < hi; ++t) acc += a[(size_t)i * K + t] * b[(size_t)t * n + j];
            c[(size_t)i * n + j] = acc;
        }
}

/* apply_activation, tinynet.cpp:96-118 */
static void activate(double* a, int rows, int cols, int act) {
    if (act == 1) {
        for (size_t i = 0; i < (size_t)rows * cols; ++i) a[i] = a[i] > 0.0 ? a[i] : 0.0;
    } else if (act == 2) {
        for (int i = 0; i < rows; ++i) {
            double* row = a + (size_t)i * cols;
            double mx = row[0];
            for (int j = 1; j < cols; ++j) mx = mx < row[j] ? row[j] : mx; /* std::max */
            double sum = 0.0;
            for (int j = 0; j < cols; ++j) {
                row[j] = exp(row[j] - mx);
                sum += row[j];
            }
            for (int j = 0; j < cols; ++j) row[j] /= sum;
        }
    }
}

/* rows_are_probabilities, tinynet.cpp:133-146 */
static int rows_are_probabilities(const double* m, int rows, int cols) {
    for (int i = 0; i < rows; ++i) {
        double sum = 0.0;
        for (int j = 0; j < cols; ++j) {
            const double x = m[(size_t)i * cols + j];
            if (x < 0.0 || x > 1.0 + 1e-9) return 0;
            sum += x;
        }
        if (fabs(sum - 1.0) > 1e-6) return 0;
    }
    return 1;
}

/* loss_sum, tinynet.cpp:216-241 */
static int loss_sum(const double* out, int rows, int cols, const int* labels, int kind, double* res,
                    char* err, size_t errlen) {
    double sum = 0.0;
    if (kind == 0) {
        for (int i = 0; i < rows; ++i) {
            if (cols != 1 && (labels[i] < 0 || labels[i] >= cols))
                return fail(err, errlen, OR_INVALID, "label out of range for one-hot target");
            for (int j = 0; j < cols; ++j) {
                const double t = cols == 1 ? (double)labels[i] : (j == labels[i] ? 1.0 : 0.0);
                const double d = out[(size_t)i * cols + j] - t;
                sum += 0.5 * d * d;
            }
        }
    } else {
        if (!rows_are_probabilities(out, rows, cols))
            return fail(err, errlen, OR_RUNTIME,
                        "cross_entropy needs probability outputs (softmax last layer required)");
        for (int i = 0; i < rows; ++i) {
            const int lbl = labels[i];
            if (lbl < 0 || lbl >= cols) return fail(err, errlen, OR_INVALID, "label out of range");
            const double p = out[(size_t)i * cols + lbl];
            sum += -log(p > 1e-300 ? p : 1e-300);
        }
    }
    *res = sum;
    return OR_OK;
}

/* predict_classes, tinynet.cpp:354-368 */
static void predict(const double* out, int rows, int cols, int* cls) {
    for (int i = 0; i < rows; ++i) {
        const double* r = out + (size_t)i * cols;
        if (cols == 1) {
            cls[i] = r[0] >= 0.5 ? 1 : 0;
        } else {
            int best = 0;
            for (int j = 1; j < cols; ++j)
                if (r[j] > r[best]) best = j;
            cls[i] = best;
        }
    }
}

/* accuracy, tinynet.cpp:370-385 (multiclass: extension, #(pred==label)/n) */
static int accuracy(const int* pred, const int* labels, int n, int multiclass, double* acc, char* err,
                    size_t errlen) {
    long tp = 0, tn = 0, fp = 0, fn = 0, hit = 0;
    for (int i = 0; i < n; ++i) {
        if (multiclass) {
            hit += pred[i] == labels[i];
            continue;
        }
        if (labels[i] != 0 && labels[i] != 1)
            return fail(err, errlen, OR_INVALID, "accuracy expects binary labels");
        if (pred[i] == 1 && labels[i] == 1) ++tp;
        else if (pred[i] == 0 && labels[i] == 0) ++tn;
        else if (pred[i] == 1 && labels[i] == 0) ++fp;
        else ++fn;
    }
    *acc = multiclass ? (double)hit / (double)n : (double)(tp + tn) / (double)(tp + tn + fp + fn);
    return OR_OK;
}

/* validate_net, tinynet.cpp:150-174 */
static int validate_net(const int* dims, const int* acts, int L, const double* W, const double* b,
                        char* err, size_t errlen) {
    if (L < 1) return fail(err, errlen, OR_INVALID, "net must have at least one layer");
    size_t wo = 0, bo = 0;
    for (int l = 0; l < L; ++l) {
        if (dims[l] < 1 || dims[l + 1] < 1)
            return fail(err, errlen, OR_INVALID, "layer %d: empty weight matrix", l + 1);
        if (acts[l] == 2 && l != L - 1)
            return fail(err, errlen, OR_INVALID, "softmax is only valid on the last layer");
        for (size_t i = 0; i < (size_t)dims[l] * dims[l + 1]; ++i)
            if (!isfinite(W[wo + i])) return fail(err, errlen, OR_INVALID, "non-finite weight");
        for (int i = 0; i < dims[l + 1]; ++i)
            if (!isfinite(b[bo + i])) return fail(err, errlen, OR_INVALID, "non-finite bias");
        wo += (size_t)dims[l] * dims[l + 1];
        bo += dims[l + 1];
    }
    return OR_OK;
}

typedef struct {
    int L;
    const int* dims;
    const int* acts;
    size_t* woff;
    size_t* boff;
} netdesc;

static void net_offsets(netdesc* nd, const int* dims, const int* acts, int L) {
    nd->L = L;
    nd->dims = dims;
    nd->acts = acts;
    nd->woff = (size_t*)malloc(sizeof(size_t) * (L + 1));
    nd->boff = (size_t*)malloc(sizeof(size_t) * (L + 1));
    nd->woff[0] = nd->boff[0] = 0;
    for (int l = 0; l < L; ++l) {
        nd->woff[l + 1] = nd->woff[l] + (size_t)dims[l] * dims[l + 1];
        nd->boff[l + 1] = nd->boff[l] + dims[l + 1];
    }
}

static void net_free(netdesc* nd) {
    free(nd->woff);
    free(nd->boff);
}

/* forward over `rows` samples (tinynet.cpp:198-214); q[l], a[l] for l=1..L,
 * a[0] = X.  Buffers are allocated by the caller. */
static void forward_rows(const netdesc* nd, const double* W, const double* bias, const double* X,
                         int rows, double** q, double** a) {
    const int L = nd->L;
    for (int l = 1; l <= L; ++l) {
        const int fi = nd->dims[l - 1], fo = nd->dims[l];
        const double* in = l == 1 ? X : a[l - 1];
        mm_nt(in, W + nd->woff[l - 1], q[l], rows, fi, fo);
        const double* bl = bias + nd->boff[l - 1];
        for (int i = 0; i < rows; ++i)
            for (int j = 0; j < fo; ++j) q[l][(size_t)i * fo + j] += bl[j];
        memcpy(a[l], q[l], sizeof(double) * (size_t)rows * fo);
        activate(a[l], rows, fo, nd->acts[l - 1]);
    }
}

int or_forward(const int* dims, const int* acts, int L, const double* W, const double* b,
               const double* X, int batch, double* acts_out, char* err, size_t errlen) {
    int rc = validate_net(dims, acts, L, W, b, err, errlen);
    if (rc) return rc;
    netdesc nd;
    net_offsets(&nd, dims, acts, L);
    double** q = (double**)calloc(L + 1, sizeof(double*));
    double** a = (double**)calloc(L + 1, sizeof(double*));
    for (int l = 1; l <= L; ++l) {
        q[l] = (double*)malloc(sizeof(double) * (size_t)batch * dims[l]);
        a[l] = (double*)malloc(sizeof(double) * (size_t)batch * dims[l]);
    }
    forward_rows(&nd, W, b, X, batch, q, a);
    size_t off = 0;
    for (int l = 1; l <= L; ++l) {
        memcpy(acts_out + off, a[l], sizeof(double) * (size_t)batch * dims[l]);
        off += (size_t)batch * dims[l];
        free(q[l]);
        free(a[l]);
    }
    free(q);
    free(a);
    net_free(&nd);
    return OR_OK;
}

/* Output delta, sum convention (tinynet.cpp:258-280; shard form
 * train_partitioned.cpp:432-470): CE p - onehot; MSE out - target, masked by
 * q<=0 when the last layer is relu. */
static void output_delta(const netdesc* nd, const double* out, const double* qL, const int* labels,
                         int rows, int kind, double* delta) {
    const int fo = nd->dims[nd->L];
    memcpy(delta, out, sizeof(double) * (size_t)rows * fo);
    if (kind == 1) {
        for (int i = 0; i < rows; ++i) delta[(size_t)i * fo + labels[i]] -= 1.0;
    } else {
        for (int i = 0; i < rows; ++i)
            for (int j = 0; j < fo; ++j) {
                const double t = fo == 1 ? (double)labels[i] : (j == labels[i] ? 1.0 : 0.0);
                delta[(size_t)i * fo + j] = out[(size_t)i * fo + j] - t;
            }
        if (nd->acts[nd->L - 1] == 1)
            for (size_t i = 0; i < (size_t)rows * fo; ++i)
                if (qL[i] <= 0.0) delta[i] = 0.0;
    }
}

static int check_loss_act(const int* acts, int L, int loss, char* err, size_t errlen) {
    if (loss == 1 && acts[L - 1] != 2)
        return fail(err, errlen, OR_RUNTIME,
                    "cross_entropy needs probability outputs (softmax last layer required)");
    if (loss == 0 && acts[L - 1] == 2)
        return fail(err, errlen, OR_RUNTIME, "softmax output requires the cross_entropy loss");
    return OR_OK;
}

/* One layer group list per layer: contributor shards in device order, or a
 * single full-width group for a replicated layer (train_partitioned.cpp:181-190). */
typedef struct {
    int ngroups;
    int lo[512];
    int hi[512];
} layer_groups;

/* The shared partitioned/sequential trainer.  groups == NULL means the
 * sequential oracle (tinynet.cpp:331-352), which divides each gradient by b
 * before the update instead of accumulating micro-batch sums. */
static int train_core(const int* dims, const int* acts, int L, const double* W0, const double* b0,
                      const double* X, const int* labels, int batch, const layer_groups* groups,
                      const int* mb_sizes, int m, double alpha0, double decay, int loss,
                      int iterations, int multiclass, double* W_out, double* b_out,
                      double* loss_hist, double* acc_hist, char* err, size_t errlen) {
    netdesc nd;
    net_offsets(&nd, dims, acts, L);
    const int I0 = dims[0];
    memcpy(W_out, W0, sizeof(double) * nd.woff[L]);
    memcpy(b_out, b0, sizeof(double) * nd.boff[L]);
    int maxw = 0;
    for (int l = 0; l <= L; ++l) maxw = dims[l] > maxw ? dims[l] : maxw;
    /* per micro-batch stashes */
    double*** q = (double***)calloc(m, sizeof(double**));
    double*** a = (double***)calloc(m, sizeof(double**));
    for (int j = 0; j < m; ++j) {
        q[j] = (double**)calloc(L + 1, sizeof(double*));
        a[j] = (double**)calloc(L + 1, sizeof(double*));
        for (int l = 1; l <= L; ++l) {
            q[j][l] = (double*)malloc(sizeof(double) * (size_t)mb_sizes[j] * dims[l]);
            a[j][l] = (double*)malloc(sizeof(double) * (size_t)mb_sizes[j] * dims[l]);
        }
    }
    double* dWacc = (double*)malloc(sizeof(double) * nd.woff[L]);
    double* dbacc = (double*)malloc(sizeof(double) * nd.boff[L]);
    size_t maxmat = 0;
    for (int l = 1; l <= L; ++l) {
        size_t s = (size_t)dims[l] * dims[l - 1];
        maxmat = s > maxmat ? s : maxmat;
    }
    double* dw = (double*)malloc(sizeof(double) * maxmat);
    double* db = (double*)malloc(sizeof(double) * maxw);
    size_t maxrows = (size_t)batch;
    double* delta = (double*)malloc(sizeof(double) * maxrows * maxw);
    double* post = (double*)malloc(sizeof(double) * maxrows * maxw);
    double* part = (double*)malloc(sizeof(double) * maxrows * maxw);
    int* preds = (int*)malloc(sizeof(int) * batch);
    int rc = OR_OK, acc_rc = OR_OK;
    char acc_err[256] = {0};
    double alpha = alpha0;

    for (int t = 1; t <= iterations && rc == OR_OK; ++t) {
        memset(dWacc, 0, sizeof(double) * nd.woff[L]);
        memset(dbacc, 0, sizeof(double) * nd.boff[L]);
        double batch_loss = 0.0;
        int off = 0;
        /* ---- forward, all micro-batches (train_partitioned.cpp:245-419) */
        for (int j = 0; j < m && rc == OR_OK; ++j) {
            const int rows = mb_sizes[j];
            forward_rows(&nd, W_out, b_out, X + (size_t)off * I0, rows, q[j], a[j]);
            double ls;
            rc = loss_sum(a[j][L], rows, dims[L], labels + off, loss, &ls, err, errlen);
            if (rc) break;
            if (groups == NULL) {
                /* loss_value + divergence check, tinynet.cpp:338-342 */
                const double lv = ls / rows;
                if (!isfinite(lv)) {
                    rc = fail(err, errlen, OR_RUNTIME, "diverged at iteration %d", t);
                    break;
                }
                batch_loss = lv;
            } else {
                batch_loss += ls;
            }
            predict(a[j][L], rows, dims[L], preds + off);
            off += rows;
        }
        if (rc) break;
        if (groups == NULL) {
            loss_hist[t - 1] = batch_loss;
            rc = accuracy(preds, labels, batch, multiclass, &acc_hist[t - 1], err, errlen);
            if (rc) break;
        }
        /* ---- backward, all micro-batches (train_partitioned.cpp:422-630) */
        off = 0;
        for (int j = 0; j < m; ++j) {
            const int rows = mb_sizes[j];
            output_delta(&nd, a[j][L], q[j][L], labels + off, rows, loss, delta);
            for (int l = L; l >= 1; --l) {
                const int fo = dims[l], fi = dims[l - 1];
                const double* in = l == 1 ? X + (size_t)off * I0 : a[j][l - 1];
                /* wgrad + bias grad, :504-512 */
                mm_tn(delta, in, dw, rows, fo, fi);
                for (int c = 0; c < fo; ++c) db[c] = 0.0;
                for (int i = 0; i < rows; ++i)
                    for (int c = 0; c < fo; ++c) db[c] += delta[(size_t)i * fo + c];
                double* accw = dWacc + nd.woff[l - 1];
                double* accb = dbacc + nd.boff[l - 1];
                if (groups == NULL) {
                    /* backward(): divide by b per product (tinynet.cpp:296-298) */
                    for (size_t i = 0; i < (size_t)fo * fi; ++i) accw[i] = dw[i] / batch;
                    for (int c = 0; c < fo; ++c) accb[c] = db[c] / batch;
                } else {
                    for (size_t i = 0; i < (size_t)fo * fi; ++i) accw[i] += dw[i];
                    for (int c = 0; c < fo; ++c) accb[c] += db[c];
                }
                if (l == 1) break;
                /* dgrad partials per contributor shard, summed in ascending
                 * device order (:514-568, :578-626) */
                const double* Wl = W_out + nd.woff[l - 1];
                const layer_groups* g = groups ? &groups[l - 1] : NULL;
                const int ng = g ? g->ngroups : 1;
                for (int k = 0; k < ng; ++k) {
                    const int lo = g ? g->lo[k] : 0, hi = g ? g->hi[k] : fo;
                    mm_nn_slice(delta, fo, Wl, k == 0 ? post : part, rows, fi, lo, hi);
                    if (k > 0)
                        for (size_t i = 0; i < (size_t)rows * fi; ++i) post[i] += part[i];
                }
                if (acts[l - 2] == 1) {
                    const double* ql = q[j][l - 1];
                    for (size_t i = 0; i < (size_t)rows * fi; ++i)
                        if (ql[i] <= 0.0) post[i] = 0.0;
                }
                memcpy(delta, post, sizeof(double) * (size_t)rows * fi);
            }
            off += rows;
        }
        /* ---- update (:632-651; sequential: sgd_step, tinynet.cpp:313-329) */
        for (int l = 1; l <= L && rc == OR_OK; ++l) {
            const size_t nw = (size_t)dims[l] * dims[l - 1];
            double* Wl = W_out + nd.woff[l - 1];
            double* bl = b_out + nd.boff[l - 1];
            const double* accw = dWacc + nd.woff[l - 1];
            const double* accb = dbacc + nd.boff[l - 1];
            if (groups == NULL) {
                for (size_t i = 0; i < nw; ++i)
                    if (!isfinite(accw[i])) rc = fail(err, errlen, OR_RUNTIME, "diverged: non-finite gradient");
                for (int i = 0; i < dims[l] && rc == OR_OK; ++i)
                    if (!isfinite(accb[i])) rc = fail(err, errlen, OR_RUNTIME, "diverged: non-finite gradient");
                if (rc) break;
                for (size_t i = 0; i < nw; ++i) Wl[i] -= alpha * accw[i];
                for (int i = 0; i < dims[l]; ++i) bl[i] -= alpha * accb[i];
            } else {
                for (size_t i = 0; i < nw; ++i) {
                    const double gr = accw[i] / batch;
                    if (!isfinite(gr)) {
                        rc = fail(err, errlen, OR_RUNTIME, "diverged at iteration %d", t);
                        break;
                    }
                }
                if (rc) break;
                for (size_t i = 0; i < nw; ++i) Wl[i] -= alpha * (accw[i] / batch);
                for (int i = 0; i < dims[l]; ++i) bl[i] -= alpha * (accb[i] / batch);
            }
        }
        if (rc) break;
        alpha *= 1.0 - decay;
        if (groups != NULL) {
            loss_hist[t - 1] = batch_loss / batch;
            /* history collector, :663-680: its accuracy error is rethrown only
             * after every worker finished without error (:685-689) */
            if (acc_rc == OR_OK)
                acc_rc = accuracy(preds, labels, batch, multiclass, &acc_hist[t - 1], acc_err,
                                  sizeof(acc_err));
        }
    }
    if (rc == OR_OK && acc_rc != OR_OK) rc = fail(err, errlen, acc_rc, "%s", acc_err);

    for (int j = 0; j < m; ++j) {
        for (int l = 1; l <= L; ++l) {
            free(q[j][l]);
            free(a[j][l]);
        }
        free(q[j]);
        free(a[j]);
    }
    free(q);
    free(a);
    free(dWacc);
    free(dbacc);
    free(dw);
    free(db);
    free(delta);
    free(post);
    free(part);
    free(preds);
    net_free(&nd);
    return rc;
}

int or_train_sequential(const int* dims, const int* acts, int L, const double* W, const double* b,
                        const double* X, const int* labels, int batch, double alpha0, double decay,
                        int loss, int iterations, int multiclass, double* W_out, double* b_out,
                        double* loss_hist, double* acc_hist, char* err, size_t errlen) {
    int rc = validate_net(dims, acts, L, W, b, err, errlen);
    if (rc) return rc;
    if (batch < 1) return fail(err, errlen, OR_INVALID, "batch rows and label count disagree");
    rc = check_loss_act(acts, L, loss, err, errlen);
    if (rc) return rc;
    int one = batch;
    return train_core(dims, acts, L, W, b, X, labels, batch, NULL, &one, 1, alpha0, decay, loss,
                      iterations, multiclass, W_out, b_out, loss_hist, acc_hist, err, errlen);
}

int or_train_partitioned(const int* dims, const int* acts, int L, const double* W,
                         const double* b, const double* X, const int* labels, int batch,
                         const int* plan, int plan_len, int m, int mode, double alpha0,
                         double decay, int loss, int iterations, int multiclass, double* W_out,
                         double* b_out, double* loss_hist, double* acc_hist, char* err,
                         size_t errlen) {
    /* entry validation, train_partitioned.cpp:124-141 */
    int rc = validate_net(dims, acts, L, W, b, err, errlen);
    if (rc) return rc;
    char inner[512];
    rc = validate_plan(plan, plan_len, dims + 1, L, inner, sizeof(inner));
    if (rc) return fail(err, errlen, OR_RUNTIME, "plan/net shape mismatch: %s", inner);
    if (mode == 0) return fail(err, errlen, OR_INVALID, "train_partitioned needs sync or async update mode");
    int* mb = (int*)malloc(sizeof(int) * (m > 0 ? m : 1));
    rc = or_split_microbatches(batch, m, mb, err, errlen);
    if (rc) {
        free(mb);
        return rc;
    }
    rc = check_loss_act(acts, L, loss, err, errlen);
    if (rc) {
        free(mb);
        return rc;
    }
    sub_view subs[256];
    int Z;
    const int* bounds;
    parse_plan(plan, plan_len, subs, 256, &Z, &bounds);
    layer_groups* groups = (layer_groups*)calloc(L, sizeof(layer_groups));
    for (int j = 0; j < Z; ++j) {
        for (int l = subs[j].first; l <= subs[j].last; ++l) {
            const int* sh = subs[j].shards + (size_t)(l - subs[j].first) * subs[j].D * 5;
            layer_groups* g = &groups[l - 1];
            if (sh[4]) {
                g->ngroups = 1;
                g->lo[0] = 0;
                g->hi[0] = dims[l];
            } else {
                g->ngroups = subs[j].D;
                for (int d = 0; d < subs[j].D; ++d) {
                    g->lo[d] = sh[d * 5 + 2];
                    g->hi[d] = sh[d * 5 + 3];
                }
            }
        }
    }
    rc = train_core(dims, acts, L, W, b, X, labels, batch, groups, mb, m, alpha0, decay, loss,
                    iterations, multiclass, W_out, b_out, loss_hist, acc_hist, err, errlen);
    free(groups);
    free(mb);
    return rc;
}
