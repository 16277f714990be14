/*
 * oracle/lfo.c -- plain, slow, fp64 CPU oracle for LongFlow's decode step.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2603_11504_b200/) never imports, links or executes anything under oracle/,
 * and this file shares no code, header, table or constant with it.
 *
 * What it computes (citation key: P:n = /root/reference/PAPER.md line n,
 * S:n = SPEC.md line n; DESIGN.md "Readings" R1..R17 = SURVEY.md section 8(c) Q1..Q17):
 *
 *   per unit u = (sequence b, kv head h), query heads hq = h*G + g, g < G   (R2, R3)
 *   1. s_gj = scale * sum_l q_g[l] K_j[l]            Eq. 1, Alg. 1 line P:522
 *      s_g* = scale * q_g . k*                        new token attended
 *   2. m_g = max_j s_gj ; e_gj = exp(s_gj - m_g)      exact max (R5; shift invariance S:80)
 *      Z_g = sum_j e_gj (+ e_g*)                      Eq. 4 denominator
 *   3. alpha_gj = e_gj / Z_g                          Eq. 5
 *   4. o_g = sum_j alpha_gj V_j (+ alpha_g* v*)       Eq. 1
 *   5. lambda_j = sum_l |V_j[l]|                      Eq. 6
 *   6. I_j = (1/G) sum_g alpha_gj lambda_j            Eq. 6 per head, mean over group (R2)
 *   7. slot = lowest j attaining min_j I_j            P:145, Alg. 1; tie rule S:243 (R7)
 *
 * Every loop is a plain sequential fp64 loop in the order written above; there is
 * no blocking, fusion or reordering.  bf16 inputs are widened exactly to fp64.
 *
 * Step drivers:
 *   same-step mode (R1, default): attend over n cached + the new token, candidates are
 *     the n cached tokens only (Eq. 3 "i < t"); if n < N the new token is
 *     appended at slot n (R11), else it overwrites the argmin slot in this step.
 *   deferred mode (Fig. 2 literal; NEXT-f1): the new token first covers the
 *     slot chosen at the previous step (or is appended), then attention runs over the
 *     cache, every valid slot is a candidate (optionally excluding the newest), and the
 *     argmin becomes the slot covered at the next step.
 *
 * parity pins: tests/test_oracle_pins.py (closed forms, worked examples, Appendix-A
 * identities, invariants, brute force, torch fp64 SDPA).  Nothing here is "parity unpinned".
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static double bf16_to_f64(uint16_t b) {
    uint32_t u = ((uint32_t)b) << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return (double)f;
}

/* Pure function on one unit.
 *   q      [G][d] bf16 bits     K, V  [n][d] bf16 bits (row stride d)
 *   k_new, v_new [d] bf16 bits, or both NULL: then only the n cached rows are attended
 *   out    [G][d] fp64 (required)
 *   alpha  [G][n+1] fp64 or NULL  (column n holds alpha_g* when the new token is attended)
 *   scores [n] fp64 or NULL       I_j
 *   m, Z   [G] fp64 or NULL       max logit and denominator relative to it
 * returns: argmin slot (lowest index on exact ties), -1 when n == 0 (no candidate),
 *          -2 on an empty attention support (n == 0 and no new token), -3 on OOM. */
int lfo_unit_attend(int G, int d, int n, double scale,
                    const uint16_t *q, const uint16_t *K, const uint16_t *V,
                    const uint16_t *k_new, const uint16_t *v_new,
                    double *out, double *alpha, double *scores, double *m, double *Z) {
    int with_new = (k_new != NULL && v_new != NULL);
    int T = n + (with_new ? 1 : 0);
    if (T == 0) return -2;
    double *s = (double *)malloc(sizeof(double) * (size_t)G * (size_t)T);
    double *a = (double *)malloc(sizeof(double) * (size_t)G * (size_t)T);
    double *lam = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    if (!s || !a || !lam) { free(s); free(a); free(lam); return -3; }

    for (int g = 0; g < G; ++g) {
        const uint16_t *qg = q + (size_t)g * d;
        /* step 1: logits */
        for (int j = 0; j < T; ++j) {
            const uint16_t *kj = (j < n) ? K + (size_t)j * d : k_new;
            double dot = 0.0;
            for (int l = 0; l < d; ++l) dot += bf16_to_f64(qg[l]) * bf16_to_f64(kj[l]);
            s[(size_t)g * T + j] = scale * dot;
        }
        /* step 2: max, exponentials, denominator */
        double mg = s[(size_t)g * T];
        for (int j = 1; j < T; ++j)
            if (s[(size_t)g * T + j] > mg) mg = s[(size_t)g * T + j];
        double zg = 0.0;
        for (int j = 0; j < T; ++j) {
            a[(size_t)g * T + j] = exp(s[(size_t)g * T + j] - mg);
            zg += a[(size_t)g * T + j];
        }
        /* step 3: weights */
        for (int j = 0; j < T; ++j) a[(size_t)g * T + j] /= zg;
        /* step 4: output */
        double *og = out + (size_t)g * d;
        for (int l = 0; l < d; ++l) og[l] = 0.0;
        for (int j = 0; j < T; ++j) {
            const uint16_t *vj = (j < n) ? V + (size_t)j * d : v_new;
            double w = a[(size_t)g * T + j];
            for (int l = 0; l < d; ++l) og[l] += w * bf16_to_f64(vj[l]);
        }
        if (m) m[g] = mg;
        if (Z) Z[g] = zg;
        if (alpha)
            for (int j = 0; j < T; ++j) alpha[(size_t)g * (n + 1) + j] = a[(size_t)g * T + j];
    }
    /* step 5: value L1 norms */
    for (int j = 0; j < n; ++j) {
        double acc = 0.0;
        for (int l = 0; l < d; ++l) acc += fabs(bf16_to_f64(V[(size_t)j * d + l]));
        lam[j] = acc;
    }
    /* steps 6-7: scores and argmin */
    int best = -1;
    double best_v = 0.0;
    for (int j = 0; j < n; ++j) {
        double acc = 0.0;
        for (int g = 0; g < G; ++g) acc += a[(size_t)g * T + j] * lam[j];
        double I = acc / (double)G;
        if (scores) scores[j] = I;
        if (best < 0 || I < best_v) { best = j; best_v = I; }
    }
    free(s); free(a); free(lam);
    return best;
}

/* ------------------------------------------------------------------------- */
/* Step drivers over a whole cache.  Layouts (row-major):
 *   K, V     [B][Hkv][N][d] bf16 bits      n_valid [B][Hkv] int32
 *   q        [B][Hq][d]                    k_new, v_new [B][Hkv][d]
 *   out      [B][Hq][d] fp64               slot [B][Hkv] int32
 *   scores   [B][Hkv][N] fp64 or NULL  (+inf for j >= n)                      */

typedef struct {
    int B, Hq, Hkv, d, N;
    double scale;
    const uint16_t *K, *V;
    const int32_t *n_valid;
    const uint16_t *q, *k_new, *v_new;
    double *out, *scores;
    int32_t *slot;
    int attend_new;       /* 1: same-step (new token attended); 0: cache only */
    const int32_t *exclude; /* deferred: per unit slot excluded from candidates, or NULL / -1 */
    int u0, u1;
    int status;
} step_job;

static void *step_worker(void *arg) {
    step_job *jb = (step_job *)arg;
    int G = jb->Hq / jb->Hkv, d = jb->d, N = jb->N;
    double *sc = (double *)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
    if (!sc) { jb->status = -3; return NULL; }
    for (int u = jb->u0; u < jb->u1; ++u) {
        int b = u / jb->Hkv, h = u % jb->Hkv;
        int n = jb->n_valid[u];
        const uint16_t *Ku = jb->K + (size_t)u * N * d;
        const uint16_t *Vu = jb->V + (size_t)u * N * d;
        const uint16_t *qu = jb->q + ((size_t)b * jb->Hq + (size_t)h * G) * d;
        const uint16_t *kn = jb->attend_new ? jb->k_new + (size_t)u * d : NULL;
        const uint16_t *vn = jb->attend_new ? jb->v_new + (size_t)u * d : NULL;
        double *ou = jb->out + ((size_t)b * jb->Hq + (size_t)h * G) * d;
        int r = lfo_unit_attend(G, d, n, jb->scale, qu, Ku, Vu, kn, vn, ou, NULL, sc, NULL, NULL);
        if (r < -1) { jb->status = r; break; }
        int ex = jb->exclude ? jb->exclude[u] : -1;
        if (ex >= 0) { /* argmin over candidates other than `ex`, lowest index on ties */
            r = -1;
            for (int j = 0; j < n; ++j) {
                if (j == ex) continue;
                if (r < 0 || sc[j] < sc[r]) r = j;
            }
        }
        if (jb->scores) {
            double *su = jb->scores + (size_t)u * N;
            for (int j = 0; j < N; ++j) su[j] = (j < n) ? sc[j] : INFINITY;
        }
        jb->slot[u] = r;
    }
    free(sc);
    return NULL;
}

static int run_units(step_job *proto, int nthreads) {
    int U = proto->B * proto->Hkv;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > U) nthreads = U > 0 ? U : 1;
    step_job *jobs = (step_job *)calloc((size_t)nthreads, sizeof(step_job));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    if (!jobs || !th) { free(jobs); free(th); return -3; }
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = *proto;
        jobs[t].u0 = (int)((long long)U * t / nthreads);
        jobs[t].u1 = (int)((long long)U * (t + 1) / nthreads);
        jobs[t].status = 0;
    }
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, step_worker, &jobs[t]);
    step_worker(&jobs[0]);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
    int st = 0;
    for (int t = 0; t < nthreads; ++t) if (jobs[t].status) st = jobs[t].status;
    free(jobs); free(th);
    return st;
}

/* Same-step mode, compute only (no mutation).  slot[u] = n when n < N (append, R11),
 * else the argmin over the n cached tokens.  Returns 0 or a negative error. */
int lfo_step_compute(int B, int Hq, int Hkv, int d, int N, double scale,
                     const uint16_t *K, const uint16_t *V, const int32_t *n_valid,
                     const uint16_t *q, const uint16_t *k_new, const uint16_t *v_new,
                     double *out, int32_t *slot, double *scores, int nthreads) {
    if (B < 0 || Hkv < 1 || Hq < 1 || Hq % Hkv != 0 || d < 1 || N < 2) return -4;
    step_job jb;
    memset(&jb, 0, sizeof jb);
    jb.B = B; jb.Hq = Hq; jb.Hkv = Hkv; jb.d = d; jb.N = N; jb.scale = scale;
    jb.K = K; jb.V = V; jb.n_valid = n_valid; jb.q = q; jb.k_new = k_new; jb.v_new = v_new;
    jb.out = out; jb.scores = scores; jb.slot = slot; jb.attend_new = 1; jb.exclude = NULL;
    int st = run_units(&jb, nthreads);
    if (st) return st;
    for (int u = 0; u < B * Hkv; ++u)
        if (n_valid[u] < N) slot[u] = n_valid[u];
    return 0;
}

/* Same-step mode, commit: the new token's K/V (bf16 bits, copied) goes to slot[u];
 * an append (slot == n_valid < N) grows n_valid by one.  Returns 0, or -5 if a slot
 * is neither the append slot nor a valid slot of a full unit. */
int lfo_step_apply(int B, int Hkv, int d, int N, uint16_t *K, uint16_t *V, int32_t *n_valid,
                   const uint16_t *k_new, const uint16_t *v_new, const int32_t *slot) {
    for (int u = 0; u < B * Hkv; ++u) {
        int n = n_valid[u], s = slot[u];
        if (n < N) { if (s != n) return -5; n_valid[u] = n + 1; }
        else if (s < 0 || s >= N) return -5;
        memcpy(K + ((size_t)u * N + s) * d, k_new + (size_t)u * d, sizeof(uint16_t) * d);
        memcpy(V + ((size_t)u * N + s) * d, v_new + (size_t)u * d, sizeof(uint16_t) * d);
    }
    return 0;
}

/* Deferred mode (Fig. 2 literal).  pend[u] is the slot chosen at the previous
 * step (-1 if none).  (1) the new token covers pend[u] when the unit is full, else it
 * is appended at n; written[u] returns that slot.  (2) attention over the n cached
 * tokens (which now include the new one).  (3) pend[u] <- argmin over all valid slots,
 * or over all but the newest when exclude_newest != 0.  Mutates K, V, n_valid, pend. */
int lfo_step_deferred(int B, int Hq, int Hkv, int d, int N, double scale,
                      uint16_t *K, uint16_t *V, int32_t *n_valid, int32_t *pend,
                      const uint16_t *q, const uint16_t *k_new, const uint16_t *v_new,
                      double *out, int32_t *written, double *scores, int exclude_newest,
                      int nthreads) {
    if (B < 0 || Hkv < 1 || Hq < 1 || Hq % Hkv != 0 || d < 1 || N < 2) return -4;
    int U = B * Hkv;
    int32_t *ex = (int32_t *)malloc(sizeof(int32_t) * (size_t)(U > 0 ? U : 1));
    if (!ex) return -3;
    for (int u = 0; u < U; ++u) {
        int n = n_valid[u], s;
        if (n < N) { s = n; n_valid[u] = n + 1; }
        else { s = pend[u]; if (s < 0 || s >= N) { free(ex); return -5; } }
        memcpy(K + ((size_t)u * N + s) * d, k_new + (size_t)u * d, sizeof(uint16_t) * d);
        memcpy(V + ((size_t)u * N + s) * d, v_new + (size_t)u * d, sizeof(uint16_t) * d);
        written[u] = s;
        ex[u] = exclude_newest ? s : -1;
    }
    step_job jb;
    memset(&jb, 0, sizeof jb);
    jb.B = B; jb.Hq = Hq; jb.Hkv = Hkv; jb.d = d; jb.N = N; jb.scale = scale;
    jb.K = K; jb.V = V; jb.n_valid = n_valid; jb.q = q; jb.k_new = NULL; jb.v_new = NULL;
    jb.out = out; jb.scores = scores; jb.slot = pend; jb.attend_new = 0; jb.exclude = ex;
    int st = run_units(&jb, nthreads);
    free(ex);
    return st;
}

/* ------------------------------------------------------------------------- */
/* SnapKV prefill compression (NEXT-f3; "first use SnapKV to compress the tokens to the
 * budget size"; parameters per SPEC S:300-308; readings R22-R24 in DESIGN.md).
 * One unit (sequence, kv head) with a prompt of n tokens, G query heads and an observation window
 * of the last w prompt positions:
 *   1. for each observation query (g, k), k < w, at prompt position p = n - w + k:
 *        s_j = scale * q_{g,k} . K_j  for j <= p (causal), alpha = softmax over j <= p
 *   2. score_i = (1/(G w)) sum_{g,k} alpha_{g,k,i}       for prefix tokens i < n - w
 *   3. pooled_i = max_{|j - i| <= (ks-1)/2, 0 <= j < n-w} score_j   (1-D max pool, 'same')
 *   4. keep the (budget - w) prefix tokens with the largest pooled score (ties: lower index),
 *      plus the w window tokens; kept sorted ascending.
 * q_obs [G][w][d], K [n][d] bf16 bits.  kept [budget] output, score/pooled [n - w] optional.
 * Returns the number kept (= budget), or -4 on bad arguments (n <= budget, w > budget, ...). */
int lfo_snapkv_select(int G, int d, int n, int w, int ks, int budget, double scale,
                      const uint16_t *q_obs, const uint16_t *K, int32_t *kept,
                      double *score_out, double *pooled_out) {
    if (n <= budget || w < 1 || w > budget || w > n || ks < 1 || (ks % 2) == 0) return -4;
    int np = n - w;                  /* prefix tokens (candidates) */
    double *score = (double *)calloc((size_t)(np > 0 ? np : 1), sizeof(double));
    double *pooled = (double *)calloc((size_t)(np > 0 ? np : 1), sizeof(double));
    double *s = (double *)malloc(sizeof(double) * (size_t)n);
    char *taken = (char *)calloc((size_t)(np > 0 ? np : 1), 1);
    if (!score || !pooled || !s || !taken) { free(score); free(pooled); free(s); free(taken); return -3; }
    for (int g = 0; g < G; ++g) {
        for (int k = 0; k < w; ++k) {
            const uint16_t *qr = q_obs + ((size_t)g * w + k) * d;
            int p = n - w + k;
            double m = 0.0;
            for (int j = 0; j <= p; ++j) {           /* step 1: causal logits */
                double dot = 0.0;
                for (int l = 0; l < d; ++l) dot += bf16_to_f64(qr[l]) * bf16_to_f64(K[(size_t)j * d + l]);
                s[j] = scale * dot;
                if (j == 0 || s[j] > m) m = s[j];
            }
            double z = 0.0;
            for (int j = 0; j <= p; ++j) z += exp(s[j] - m);
            for (int i = 0; i < np; ++i) score[i] += exp(s[i] - m) / z;   /* step 2 (sum) */
        }
    }
    for (int i = 0; i < np; ++i) score[i] /= (double)(G * w);            /* step 2 (mean) */
    int r = (ks - 1) / 2;
    for (int i = 0; i < np; ++i) {                                        /* step 3 */
        double mx = score[i];
        for (int j = i - r; j <= i + r; ++j)
            if (j >= 0 && j < np && score[j] > mx) mx = score[j];
        pooled[i] = mx;
    }
    int want = budget - w;                                                /* step 4 */
    for (int c = 0; c < want; ++c) {
        int best = -1;
        for (int i = 0; i < np; ++i)
            if (!taken[i] && (best < 0 || pooled[i] > pooled[best])) best = i;
        taken[best] = 1;
    }
    int o = 0;
    for (int i = 0; i < np; ++i) if (taken[i]) kept[o++] = i;
    for (int k = 0; k < w; ++k) kept[o++] = np + k;
    if (score_out) memcpy(score_out, score, sizeof(double) * (size_t)np);
    if (pooled_out) memcpy(pooled_out, pooled, sizeof(double) * (size_t)np);
    free(score); free(pooled); free(s); free(taken);
    return o;
}

/* ------------------------------------------------------------------------- */
/* NEXT-f4: the eviction objective itself, by brute force (Eq. 3's right-hand side, P:110:
 * ||o_t - o_t^(\i)||^2 with the current query, "computed without the key-value pair of token
 * t_i").  For every cached candidate i < n the unit is re-attended from scratch over the
 * cache without row i (plus the current token, R1), with lfo_unit_attend, and
 *   E_i = (1/G) sum_g sum_l (o_g[l] - o_g^(\i)[l])^2         (mean over the group, R2/R25).
 * No closed form is used (App. A's exact remainder is only a check of this in the tests).
 *   E [n] fp64.  returns 0, or < 0 on error (n < 2: nothing to evict and keep attending). */
int lfo_exact_objective(int G, int d, int n, double scale,
                        const uint16_t *q, const uint16_t *K, const uint16_t *V,
                        const uint16_t *k_new, const uint16_t *v_new, double *E) {
    if (n < 1) return -1;
    double *o = (double *)malloc(sizeof(double) * (size_t)G * (size_t)d);
    double *oi = (double *)malloc(sizeof(double) * (size_t)G * (size_t)d);
    uint16_t *Ki = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)(n > 1 ? n - 1 : 1) * (size_t)d);
    uint16_t *Vi = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)(n > 1 ? n - 1 : 1) * (size_t)d);
    if (!o || !oi || !Ki || !Vi) { free(o); free(oi); free(Ki); free(Vi); return -3; }
    int r = lfo_unit_attend(G, d, n, scale, q, K, V, k_new, v_new, o, NULL, NULL, NULL, NULL);
    for (int i = 0; i < n && r >= -1; ++i) {
        /* the cache without row i, rows in their original order */
        int w = 0;
        for (int j = 0; j < n; ++j) {
            if (j == i) continue;
            memcpy(Ki + (size_t)w * d, K + (size_t)j * d, sizeof(uint16_t) * (size_t)d);
            memcpy(Vi + (size_t)w * d, V + (size_t)j * d, sizeof(uint16_t) * (size_t)d);
            ++w;
        }
        r = lfo_unit_attend(G, d, n - 1, scale, q, Ki, Vi, k_new, v_new, oi, NULL, NULL, NULL, NULL);
        double acc = 0.0;
        for (int g = 0; g < G; ++g)
            for (int l = 0; l < d; ++l) {
                double dl = o[(size_t)g * d + l] - oi[(size_t)g * d + l];
                acc += dl * dl;
            }
        E[i] = acc / (double)G;
    }
    free(o); free(oi); free(Ki); free(Vi);
    return r < -1 ? r : 0;
}
