/*
 * oracle/hs_oracle.c -- the CPU ORACLE for the HybridServe cascade router.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2505_12566_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or constant with csrc/.
 *
 * Plain, slow, obviously-correct C: fp64 arithmetic, plain loops, Neumaier
 * (compensated) summation, qsort as the only library primitive.  Each
 * function cites the passage of /root/reference/PAPER.md ("P:<line>") it
 * follows, and the reading taken where the paper is garbled (DESIGN.md
 * "Readings", mirrored from SURVEY.md 8(c) G1..G18).
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py
 * (closed forms, library special cases, hand-worked cascades, brute force).
 * Nothing here is "parity unpinned".
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* enums: the oracle's own numbering (tests pass plain ints)                 */
/* ------------------------------------------------------------------------- */
enum { ORC_F32 = 0, ORC_BF16 = 1 };
enum { ORC_MAXPROB = 0, ORC_MAXPROB_SQ = 1, ORC_ENTROPY = 2 };
enum { ORC_SEQ_NONE = 0, ORC_SEQ_MIN = 1, ORC_SEQ_MEAN = 2 };

/* Exact widening of one stored logit to double (bf16 = top 16 bits of an
 * IEEE binary32; every bf16 and every fp32 value is exactly a double). */
static double load_logit(const void* base, int dtype, int64_t idx) {
    float f;
    if (dtype == ORC_BF16) {
        uint32_t u = ((uint32_t)((const uint16_t*)base)[idx]) << 16;
        memcpy(&f, &u, sizeof f);
    } else {
        f = ((const float*)base)[idx];
    }
    return (double)f;
}

/* Neumaier compensated summation (plain definition of a sum, with the
 * rounding error carried so that the fp64 result is ~exact). */
typedef struct { double s, c; } nsum_t;
static void nsum_add(nsum_t* a, double v) {
    double t = a->s + v;
    if (fabs(a->s) >= fabs(v)) a->c += (a->s - t) + v;
    else                       a->c += (v - t) + a->s;
    a->s = t;
}
static double nsum_get(const nsum_t* a) { return a->s + a->c; }

/* ------------------------------------------------------------------------- */
/* D1. Row confidence statistics.                                            */
/*   P:384-391 (f_theta maps a prediction vector of logits to a score),      */
/*   P:373-375 (Temperature Scaling: theta is a temperature, z = x / T),     */
/*   P:413-416 (classification: max of the softmax, squared -- reading G1).  */
/* Returns 0 on success, 1 if the row is not a valid prediction vector      */
/* (a NaN or +inf entry, or every entry -inf; S:122 requires finite input;  */
/* -inf is accepted as a masked class with p = 0 and entropy term 0).       */
/* ------------------------------------------------------------------------- */
int hso_row_stats(const double* x, int64_t C, double T,
                  double* p_max, double* entropy, int64_t* argmax) {
    /* step 2: reject non-finite rows */
    int64_t n_finite = 0;
    for (int64_t j = 0; j < C; ++j) {
        if (isnan(x[j]) || (isinf(x[j]) && x[j] > 0)) return 1;
        if (!isinf(x[j])) ++n_finite;
    }
    if (n_finite == 0) return 1;
    /* step 3: mx = max_j x_j, j* = lowest index attaining it (reading G12) */
    double mx = x[0];
    int64_t jstar = 0;
    for (int64_t j = 1; j < C; ++j)
        if (x[j] > mx) { mx = x[j]; jstar = j; }
    /* step 4-5: a_j = (x_j - mx) / T; s = sum exp(a_j); w = sum exp(a_j) a_j */
    nsum_t s = {0, 0}, w = {0, 0};
    for (int64_t j = 0; j < C; ++j) {
        if (isinf(x[j])) continue;                 /* masked class: p_j = 0 */
        double a = (x[j] - mx) / T;
        double e = exp(a);
        nsum_add(&s, e);
        nsum_add(&w, e * a);
    }
    double S = nsum_get(&s), W = nsum_get(&w);
    /* step 6: p_max = exp(0)/s = 1/s ; H = -sum p_j ln p_j = ln s - w/s */
    *p_max = 1.0 / S;
    *entropy = log(S) - W / S;
    *argmax = jstar;
    return 0;
}

/* ------------------------------------------------------------------------- */
/* D1' (NEXT-2). Top-K restricted confidence for generation models.         */
/*   "We assign P = TopK(P) to enhance the prediction, while the  */
/*   rest is the same as classification"; f = TopK(softmax(theta(P))^2).    */
/*   Reading: restrict the row to its K largest  */
/*   logits, softmax over the restricted set at temperature T, then the same */
/*   confidence as D1 (p_max, p_max^2 or exp(-H) of the restricted           */
/*   distribution).  The K largest VALUES are a unique multiset, so ties at  */
/*   the K-th place do not matter.  K >= C is the full softmax.  Validity    */
/*   and the argmax are those of the full row (argmax invariance).    */
/* ------------------------------------------------------------------------- */
static int cmp_desc(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return (x < y) - (x > y);
}

int hso_row_stats_topk(const double* x, int64_t C, double T, int64_t K,
                       double* p_max, double* entropy, int64_t* argmax) {
    double p, H;
    int64_t am;
    if (hso_row_stats(x, C, T, &p, &H, &am) != 0) return 1;   /* full-row checks */
    if (K <= 0 || K >= C) {
        *p_max = p; *entropy = H; *argmax = am;
        return 0;
    }
    double* v = (double*)malloc(sizeof(double) * (size_t)C);
    memcpy(v, x, sizeof(double) * (size_t)C);
    qsort(v, (size_t)C, sizeof(double), cmp_desc);        /* v[0] >= v[1] >= ... */
    int64_t k_finite = 0;
    while (k_finite < K && !isinf(v[k_finite])) ++k_finite;  /* -inf: masked, p = 0 */
    /* restricted statistics: the K largest values as their own prediction vector */
    nsum_t s = {0, 0}, w = {0, 0};
    for (int64_t j = 0; j < k_finite; ++j) {
        double a = (v[j] - v[0]) / T;
        double e = exp(a);
        nsum_add(&s, e);
        nsum_add(&w, e * a);
    }
    double S = nsum_get(&s), W = nsum_get(&w);
    free(v);
    *p_max = 1.0 / S;
    *entropy = log(S) - W / S;
    *argmax = am;
    return 0;
}

/* step 7: the confidence of one row from its statistics.
 *   MAXPROB    : p_max                      (north_star; reading G1)
 *   MAXPROB_SQ : p_max^2                    (P:415 taken literally, G1)
 *   ENTROPY    : exp(-H) = 1/perplexity     (north_star; reading G3)      */
static double conf_of(int kind, double p_max, double H) {
    if (kind == ORC_MAXPROB_SQ) return p_max * p_max;
    if (kind == ORC_ENTROPY) return exp(-H);
    return p_max;
}

/* ------------------------------------------------------------------------- */
/* D1 + D2 batched: per-sequence confidence.                                 */
/*   P:420-424 (generation: "the minimal confidence is the confidence of     */
/*   complete output" -> MIN over the L token confidences; MEAN is the       */
/*   north_star's alternative), P:427-430 (QA = MIN with L = 2).             */
/* Batch item i reads sequence r = row_index ? row_index[i] : i; its token  */
/* t is the logits row r*L + t at element offset (r*L + t) * stride.        */
/* Outputs per item: conf, argmax[i*L + t], correct (all L tokens equal     */
/* their labels[r*L + t]; reading G13), bad (1 = invalid row seen).         */
/* ------------------------------------------------------------------------- */
typedef struct {
    const void* logits; int dtype; int64_t n_seq; int L; int64_t C; int64_t stride;
    const int64_t* row_index; double T; int kind; int reduce; int64_t top_k;
    double* conf; int32_t* argmax; const int32_t* labels; uint8_t* correct; uint8_t* bad;
    int64_t lo, hi;
} conf_job_t;

static void* conf_worker(void* arg) {
    conf_job_t* J = (conf_job_t*)arg;
    double* row = (double*)malloc(sizeof(double) * (size_t)J->C);
    for (int64_t i = J->lo; i < J->hi; ++i) {
        int64_t r = J->row_index ? J->row_index[i] : i;
        double cmin = INFINITY;
        nsum_t csum = {0, 0};
        int all_correct = 1, any_bad = 0;
        for (int t = 0; t < J->L; ++t) {
            int64_t tok = r * J->L + t;
            for (int64_t j = 0; j < J->C; ++j)
                row[j] = load_logit(J->logits, J->dtype, tok * J->stride + j);
            double p, H; int64_t am;
            if (hso_row_stats_topk(row, J->C, J->T, J->top_k, &p, &H, &am) != 0) {
                any_bad = 1; am = -1; p = NAN; H = NAN;
            }
            double c = conf_of(J->kind, p, H);
            if (c < cmin || isnan(c)) cmin = c;
            nsum_add(&csum, c);
            if (J->argmax) J->argmax[i * J->L + t] = (int32_t)am;
            if (J->labels && am != (int64_t)J->labels[tok]) all_correct = 0;
        }
        double cs;
        if (any_bad)                          cs = NAN;
        else if (J->reduce == ORC_SEQ_MEAN)   cs = nsum_get(&csum) / (double)J->L;
        else                                  cs = cmin;   /* MIN, or NONE with L == 1 */
        J->conf[i] = cs;
        if (J->correct) J->correct[i] = (uint8_t)(J->labels ? all_correct : 0);
        if (J->bad) J->bad[i] = (uint8_t)any_bad;
    }
    free(row);
    return NULL;
}

/* Returns 0, or -1 on an argument error (C < 2, T <= 0 or non-finite,
 * L < 1, NONE with L > 1, stride < C). */
int hso_confidence(const void* logits, int dtype, int64_t n_seq, int L, int64_t C,
                   int64_t stride, const int64_t* row_index, double T, int kind, int reduce,
                   int64_t top_k, double* conf, int32_t* argmax, const int32_t* labels,
                   uint8_t* correct, uint8_t* bad, int nthreads) {
    if (C < 2 || !(T > 0) || isinf(T) || L < 1 || stride < C || n_seq < 0 || top_k < 0) return -1;
    if (reduce == ORC_SEQ_NONE && L != 1) return -1;
    if (nthreads < 1) nthreads = 1;
    if (n_seq < nthreads) nthreads = n_seq > 0 ? (int)n_seq : 1;
    conf_job_t* jobs = (conf_job_t*)calloc((size_t)nthreads, sizeof(conf_job_t));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int w = 0; w < nthreads; ++w) {
        conf_job_t J = {logits, dtype, n_seq, L, C, stride, row_index, T, kind, reduce, top_k,
                        conf, argmax, labels, correct, bad,
                        n_seq * w / nthreads, n_seq * (w + 1) / nthreads};
        jobs[w] = J;
        pthread_create(&th[w], NULL, conf_worker, &jobs[w]);
    }
    for (int w = 0; w < nthreads; ++w) pthread_join(th[w], NULL);
    free(jobs); free(th);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* NEXT-3. Temperature fitting (Eq. 1).                                      */
/*   "learn parameters theta that minimize the NLL between        */
/*   confidence scores and labels Y on the validation dataset" with Temperature */
/*   Scaling: NLL(T) = (1/n) sum_i [ log sum_j exp(x_ij / T) - x_iy / T ]. */
/*   The minimiser over the clamp range T in [e^-4, e^4] has a plain   */
/*   definition; NLL is convex in beta = 1/T (a log-sum-exp of functions linear */
/*   in beta minus a linear term), so dNLL/dbeta = mean_i (E_p[x_i] - x_iy) is */
/*   non-decreasing and the minimiser is where it changes sign (or a clamp     */
/*   end).  This oracle evaluates that derivative in fp64 (Neumaier sums) and */
/*   bisects on beta to 1e-15 relative.  Rows with a non-finite entry are     */
/*   skipped (masked -inf classes are allowed, p = 0).                        */
/* ------------------------------------------------------------------------- */
static void nll_terms(const void* logits, int dtype, int64_t n, int64_t C, int64_t stride,
                      const int32_t* labels, double beta, double* nll, double* grad, int64_t* used) {
    nsum_t L = {0, 0}, G = {0, 0};
    int64_t u = 0;
    double* row = (double*)malloc(sizeof(double) * (size_t)C);
    for (int64_t i = 0; i < n; ++i) {
        int ok = 1, any = 0;
        double mx = -INFINITY;
        for (int64_t j = 0; j < C; ++j) {
            row[j] = load_logit(logits, dtype, i * stride + j);
            if (isnan(row[j]) || (isinf(row[j]) && row[j] > 0)) ok = 0;
            if (!isinf(row[j])) { any = 1; if (row[j] > mx) mx = row[j]; }
        }
        double xy = row[labels[i]];
        if (!ok || !any || isinf(xy)) continue;
        nsum_t s = {0, 0}, sx = {0, 0};
        for (int64_t j = 0; j < C; ++j) {
            if (isinf(row[j])) continue;
            double e = exp(beta * (row[j] - mx));
            nsum_add(&s, e);
            nsum_add(&sx, e * (row[j] - mx));
        }
        double S = nsum_get(&s);
        nsum_add(&L, beta * (mx - xy) + log(S));          /* LSE(beta x) - beta x_y */
        nsum_add(&G, nsum_get(&sx) / S - (xy - mx));       /* E_p[x] - x_y          */
        ++u;
    }
    free(row);
    *nll = u ? nsum_get(&L) / (double)u : NAN;
    *grad = u ? nsum_get(&G) / (double)u : NAN;
    *used = u;
}

/* mean NLL at temperature T (Eq. 1's objective); rows used -> *used */
double hso_nll(const void* logits, int dtype, int64_t n, int64_t C, int64_t stride,
               const int32_t* labels, double T, int64_t* used) {
    double nll, g;
    nll_terms(logits, dtype, n, C, stride, labels, 1.0 / T, &nll, &g, used);
    return nll;
}

/* argmin_{T in [t_lo, t_hi]} NLL(T); returns T (NAN if no usable row) */
double hso_fit_temperature(const void* logits, int dtype, int64_t n, int64_t C, int64_t stride,
                           const int32_t* labels, double t_lo, double t_hi) {
    double b_lo = 1.0 / t_hi, b_hi = 1.0 / t_lo, nll, g;
    int64_t used;
    nll_terms(logits, dtype, n, C, stride, labels, b_lo, &nll, &g, &used);
    if (!used) return NAN;
    if (g >= 0) return t_hi;                     /* increasing over the range */
    nll_terms(logits, dtype, n, C, stride, labels, b_hi, &nll, &g, &used);
    if (g <= 0) return t_lo;                     /* decreasing over the range */
    for (int it = 0; it < 200 && (b_hi - b_lo) > 1e-15 * b_hi; ++it) {
        double b = 0.5 * (b_lo + b_hi);
        nll_terms(logits, dtype, n, C, stride, labels, b, &nll, &g, &used);
        if (g > 0) b_hi = b; else b_lo = b;
    }
    return 2.0 / (b_lo + b_hi);
}

/* ------------------------------------------------------------------------- */
/* D3 + D4. Threshold test and stable split of one stage's batch.            */
/*   "requests with scores below a threshold at a model in the    */
/*   dataflow are passed to larger models" -> defer iff c < t, accept iff    */
/*   c >= t (tie accepts, G5); the last model accepts everything (t_K = 0,   */
/*   Table III P:816/826/835, G6).  Lists hold batch positions in            */
/*   increasing order (stable).                                              */
/* ------------------------------------------------------------------------- */
void hso_route(const double* conf, int64_t n, double t, int is_last,
               int64_t* acc, int64_t* n_acc, int64_t* dfr, int64_t* n_dfr) {
    int64_t na = 0, nd = 0;
    for (int64_t i = 0; i < n; ++i) {
        int accept = is_last ? 1 : (conf[i] >= t);
        if (accept) acc[na++] = i;
        else        dfr[nd++] = i;
    }
    *n_acc = na;
    *n_dfr = nd;
}

/* D4 per request: stage(r) = first k with c_k(r) >= t_k, else the last.
 * conf[k * n + r] is stage k's confidence for request r (k = 0..K-1). */
void hso_cascade(int K, int64_t n, const double* conf, const double* t, int32_t* stage_of) {
    for (int64_t r = 0; r < n; ++r) {
        int k = 0;
        while (k < K - 1 && !(conf[(int64_t)k * n + r] >= t[k])) ++k;
        stage_of[r] = k;
    }
}

/* ------------------------------------------------------------------------- */
/* D5. Offline threshold calibration (Accuracy-Preserving mode).             */
/*   P:457-479 Alg. 1 (threshold search; replaced by the north_star's exact  */
/*   deterministic sweep, reading G8), P:483-484 (AP: accuracy of the        */
/*   cascade equal to Acc(m_n), read as ">= tau" in integer counts, G9),     */
/*   P:441 ("exhaustively find the most energy-saving thresholds").          */
/* Grid: B = 2^q bins, bin(c) = min(B, floor(c * B)), NaN -> -1 (never        */
/* accepted).  Threshold index b in 0..B+1: t = b/B, b = B+1 = defer all     */
/* (G10, G11).  This implementation sorts the alive samples by bin and takes */
/* suffix sums ("by sort"); tests/ pins it against a simulation brute force. */
/* ------------------------------------------------------------------------- */
static int64_t bin_of(double c, int64_t B) {
    if (isnan(c)) return -1;
    double f = floor(c * (double)B);
    if (f < 0) f = 0;
    if (f > (double)B) f = (double)B;
    return (int64_t)f;
}

typedef struct { int64_t bin; int64_t d; int64_t ck; } cal_item_t;
static int cmp_bin(const void* a, const void* b) {
    int64_t x = ((const cal_item_t*)a)->bin, y = ((const cal_item_t*)b)->bin;
    return (x > y) - (x < y);
}

/* Among `m` alive items with weight d (the gain of answering here instead of
 * deeper), return the smallest b in 0..B+1 with base + S(b) >= tau where
 * S(b) = sum of d over items with bin >= b.  S is not monotone in b, so
 * every b is examined in increasing order. */
static int64_t select_min_b(cal_item_t* it, int64_t m, int64_t B, int64_t base, int64_t tau) {
    qsort(it, (size_t)m, sizeof(cal_item_t), cmp_bin);
    int64_t total = 0;
    for (int64_t i = 0; i < m; ++i) if (it[i].bin >= 0) total += it[i].d;
    int64_t below = 0;   /* sum of d over items with 0 <= bin < b */
    int64_t p = 0;
    while (p < m && it[p].bin < 0) ++p;
    for (int64_t b = 0; b <= B + 1; ++b) {
        while (p < m && it[p].bin < b) { below += it[p].d; ++p; }
        int64_t S = total - below;
        if (base + S >= tau) return b;
    }
    return B + 1;   /* unreachable when base >= tau (S(B+1) = 0) */
}

/* conf[k*N + r], k = 0..K-2 (stage K has no threshold); correct[k*N + r],
 * k = 0..K-1.  tau < 0 selects AP: tau = sum_r correct[K-1][r].
 * Outputs: b[K-1], reach[K], handled[K], *A_out (cascade correct count),
 * *tau_out.  Returns 0, or -1 on argument error. */
int hso_calibrate(int K, int64_t N, const double* conf, const uint8_t* correct, int q,
                  int64_t tau, int refine_passes, int32_t* b_out, int64_t* reach,
                  int64_t* handled, int64_t* A_out, int64_t* tau_out) {
    if (K < 2 || N <= 0 || q < 1 || q > 20) return -1;
    const int64_t B = (int64_t)1 << q;
    const uint8_t* cK = correct + (int64_t)(K - 1) * N;
    if (tau < 0) { tau = 0; for (int64_t r = 0; r < N; ++r) tau += cK[r]; }
    *tau_out = tau;

    int64_t* bins = (int64_t*)malloc(sizeof(int64_t) * (size_t)(K - 1) * (size_t)N);
    for (int64_t k = 0; k < K - 1; ++k)
        for (int64_t r = 0; r < N; ++r) bins[k * N + r] = bin_of(conf[k * N + r], B);
    uint8_t* alive = (uint8_t*)malloc((size_t)N);
    cal_item_t* it = (cal_item_t*)malloc(sizeof(cal_item_t) * (size_t)N);

    /* forward greedy pass */
    for (int64_t r = 0; r < N; ++r) alive[r] = 1;
    int64_t A = 0;
    for (int k = 0; k < K - 1; ++k) {
        const uint8_t* ck = correct + (int64_t)k * N;
        int64_t m = 0, G = 0;
        for (int64_t r = 0; r < N; ++r) {
            if (!alive[r]) continue;
            G += cK[r];
            cal_item_t x = {bins[k * N + r], (int64_t)ck[r] - (int64_t)cK[r], ck[r]};
            it[m++] = x;
        }
        int64_t b = select_min_b(it, m, B, A + G, tau);
        b_out[k] = (int32_t)b;
        for (int64_t r = 0; r < N; ++r)
            if (alive[r] && bins[k * N + r] >= b) { A += ck[r]; alive[r] = 0; }
    }

    /* optional refinement passes: re-pick each b_k given the
     * current downstream thresholds; never raises b_k. */
    for (int pass = 0; pass < refine_passes; ++pass) {
        int changed = 0;
        for (int k = 0; k < K - 1; ++k) {
            const uint8_t* ck = correct + (int64_t)k * N;
            int64_t Ak = 0, m = 0, Cdown = 0;
            for (int64_t r = 0; r < N; ++r) {
                /* replay stages < k under the current thresholds */
                int j = 0;
                while (j < k && bins[(int64_t)j * N + r] < b_out[j]) ++j;
                if (j < k) { Ak += correct[(int64_t)j * N + r]; continue; }
                /* downstream correctness C_{k+1}(r) */
                int d = k + 1;
                while (d < K - 1 && bins[(int64_t)d * N + r] < b_out[d]) ++d;
                int64_t Cd = correct[(int64_t)d * N + r];
                Cdown += Cd;
                cal_item_t x = {bins[k * N + r], (int64_t)ck[r] - Cd, ck[r]};
                it[m++] = x;
            }
            int64_t b = select_min_b(it, m, B, Ak + Cdown, tau);
            if (b != b_out[k]) { b_out[k] = (int32_t)b; changed = 1; }
        }
        if (!changed) break;
    }

    /* final replay under the chosen thresholds: reach, handled, A */
    for (int k = 0; k < K; ++k) { reach[k] = 0; handled[k] = 0; }
    A = 0;
    for (int64_t r = 0; r < N; ++r) {
        int j = 0;
        reach[0] += 1;
        while (j < K - 1 && bins[(int64_t)j * N + r] < b_out[j]) { ++j; reach[j] += 1; }
        handled[j] += 1;
        A += correct[(int64_t)j * N + r];
    }
    *A_out = A;
    free(bins); free(alive); free(it);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* NEXT-1: skip connections (§IV-C, Alg. 2 line 5 P:530).    */
/*   "The confidence interval below thresholds is uniformly partitioned into  */
/*   the number of successor models"; "the request with the lowest    */
/*   confidence should be routed to the largest model" and "requests with a   */
/*   confidence score close to the threshold are routed to the successor     */
/*   model".  Stage k (0-based, K models) has s = K-1-k successor  */
/*   models and s-1 band edges inside [0, t_k):                               */
/*     mode 0 (uniform):   e_i = t_k * (s - i) / s,  i = 1..s-1         */
/*     mode 1 (decade, "LogUniform" reading): e_i = t_k / 10^i          */
/*   each edge is rounded to fp32 (the value both the router and this oracle   */
/*   compare against).  A deferred request with confidence c goes to model    */
/*   k + 1 + j, j = #{i : c < e_i} (j = 0: immediate successor; c below every */
/*   edge: the largest model).  NaN confidences count as below every edge.    */
/* ------------------------------------------------------------------------- */
void hso_skip_edges(double t, int s, int mode, float* edges /* [s-1] */) {
    double p10 = 1.0;                      /* 10^i, exact in fp64 for i <= 22 */
    for (int i = 1; i < s; ++i) {
        p10 *= 10.0;
        double e = mode == 1 ? t / p10 : t * (double)(s - i) / (double)s;
        edges[i - 1] = (float)e;
    }
}

int hso_skip_band(double c, const float* edges, int s) {
    int j = 0;
    for (int i = 1; i < s; ++i)
        if (!(c >= (double)edges[i - 1])) ++j;   /* c < e_i, or NaN */
    return j;
}

/* Per request: the models it visits (bit k of visits[r]) and the one that
 * answers (stage_of[r]).  conf[k*n + r] as in hso_cascade; t[0..K-2]. */
void hso_cascade_skip(int K, int64_t n, const double* conf, const double* t, int mode,
                      int32_t* stage_of, uint32_t* visits) {
    float edges[64];
    for (int64_t r = 0; r < n; ++r) {
        int k = 0;
        uint32_t v = 0;
        while (1) {
            v |= 1u << k;
            if (k == K - 1) break;
            const double c = conf[(int64_t)k * n + r];
            if (c >= t[k]) break;
            const int s = K - 1 - k;
            hso_skip_edges(t[k], s, mode, edges);
            k = k + 1 + hso_skip_band(c, edges, s);
        }
        stage_of[r] = k;
        visits[r] = v;
    }
}

/* ------------------------------------------------------------------------- */
/* NEXT-4. Threshold performance graph (Alg. 1 lines 3-4).        */
/*   "Compute a on D_v and e = sum_i rho_i e_i" for every threshold set k in */
/*   K: the cascade statement replayed on the validation set for */
/*   each threshold vector.  Threshold index b_k on the D5 grid: t_k = b_k/B, */
/*   b_k = B+1 = +inf (defer all); the test is c >= t_k in fp64 on the fp32  */
/*   confidence (equivalent to bin(c) >= b_k, reading G10).  rho_i is read as */
/*   the REACH count (reading G14): energy = sum_k reach_k * w_k with   */
/*   integer weights w_k (reading G23).  bvec == NULL: the exhaustive grid,   */
/*   vector s has digits b_0 (most significant) .. b_{K-2} in base B+2, i.e. */
/*   itertools.product order.  Plain loops, one vector at a time.            */
/* ------------------------------------------------------------------------- */
void hso_replay(int K, int64_t N, const double* conf, const uint8_t* correct, int q,
                int64_t S, const int32_t* bvec, const int64_t* w, int64_t* out_correct,
                int64_t* out_energy, int64_t* out_reach /* [S*K] or NULL */) {
    const int64_t B = (int64_t)1 << q, R = B + 2;
    double t[64];
    int64_t reach[64];
    for (int64_t s = 0; s < S; ++s) {
        int64_t rem = s;
        for (int k = K - 2; k >= 0; --k) {
            int64_t b;
            if (bvec) {
                b = bvec[s * (K - 1) + k];
            } else {
                b = rem % R;
                rem /= R;
            }
            t[k] = (b == B + 1) ? INFINITY : (double)b / (double)B;
        }
        for (int k = 0; k < K; ++k) reach[k] = 0;
        int64_t ok = 0;
        for (int64_t r = 0; r < N; ++r) {
            int k = 0;
            reach[0] += 1;
            while (k < K - 1 && !(conf[(int64_t)k * N + r] >= t[k])) {
                ++k;
                reach[k] += 1;
            }
            ok += correct[(int64_t)k * N + r] ? 1 : 0;
        }
        int64_t e = 0;
        for (int k = 0; k < K; ++k) e += reach[k] * w[k];
        out_correct[s] = ok;
        out_energy[s] = e;
        if (out_reach)
            for (int k = 0; k < K; ++k) out_reach[s * K + k] = reach[k];
    }
}
