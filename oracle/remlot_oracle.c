/*
 * remlot_oracle.c -- CPU restatement of the reference VND hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker for the CUDA path
 * (tests/, __graft_entry__.smoke()) and the CPU-baseline arm of bench.py.
 * No product code path links or calls it.
 *
 * It restates, in plain C with int64 arithmetic, the algorithm of the
 * reference package (`remlot`, a numba-JIT Python package) so that it can be
 * compiled with gcc and shipped to the GPU box (the Python reference cannot
 * travel).  Every function cites the reference lines it follows.  It is
 * pinned against fixtures produced by the live reference
 * (tests/golden/gen_golden.py -> tests/test_oracle_golden.py).
 *
 * The per-period recurrence is deliberately kept in the reference's form
 * (walk every period of every segment) rather than the closed form used on
 * the device, so the oracle and the CUDA path are independent derivations.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_INFEASIBLE ((int64_t)1 << 62) /* _kernels.py:11 */

typedef struct {
    int64_t K, T;
    const int64_t *dem, *ret;                 /* K x T, C order (model.py:48-49) */
    const int64_t *km, *kr, *hm, *hr, *pm, *pr; /* K vectors (model.py:54-59)   */
} orc_inst;

/* row_cost -- _kernels.py:46-97.  Leading periods without a setup must have
 * zero demand and accrue returns holding (:58-63); each setup period u
 * serves demand up to the next setup v (:65-72); remanufacture first from
 * recoverables y_r + R[u] (:73-76); remainder needs a manufacturing setup
 * (:77-82); setup cost only for positive quantities (:83-86); unit cost
 * (:87); per period inventory update and holding (:88-95). */
int64_t orc_row_cost(int64_t T, const uint8_t *sm, const uint8_t *sr,
                     const int64_t *dem, const int64_t *ret, int64_t km,
                     int64_t kr, int64_t hm, int64_t hr, int64_t pm, int64_t pr)
{
    int64_t cost = 0, rec = 0, stock = 0, t = 0;
    for (; t < T && !(sm[t] | sr[t]); ++t) {
        if (dem[t] > 0)
            return ORC_INFEASIBLE;
        rec += ret[t];
        cost += hr * rec;
    }
    while (t < T) {
        int64_t u = t, v = t + 1;
        while (v < T && !(sm[v] | sr[v]))
            ++v;
        int64_t need = 0;
        for (int64_t i = u; i < v; ++i)
            need += dem[i];
        int64_t have = rec + ret[u];
        int64_t xr = 0;
        if (sr[u])
            xr = need < have ? need : have;
        int64_t xm = need - xr;
        if (xm > 0 && !sm[u])
            return ORC_INFEASIBLE;
        if (xm < 0)
            xm = 0;
        if (xr > 0)
            cost += kr;
        if (xm > 0)
            cost += km;
        cost += pr * xr + pm * xm;
        for (int64_t i = u; i < v; ++i) {
            if (i == u) {
                stock += xm + xr;
                rec += ret[i] - xr;
            } else {
                rec += ret[i];
            }
            stock -= dem[i];
            cost += hm * stock + hr * rec;
        }
        t = v;
    }
    return cost;
}

/* product_costs -- _kernels.py:171-175 */
void orc_product_costs(const orc_inst *in, int64_t lo, int64_t hi,
                       const uint8_t *sm, const uint8_t *sr, int64_t *out)
{
    const int64_t T = in->T;
    for (int64_t k = lo; k < hi; ++k)
        out[k] = orc_row_cost(T, sm + k * T, sr + k * T, in->dem + k * T,
                              in->ret + k * T, in->km[k], in->kr[k], in->hm[k],
                              in->hr[k], in->pm[k], in->pr[k]);
}

/* list_moves -- _kernels.py:188-258.  N1 flips the manufacturing bit of
 * each period (:199-205), N2 the remanufacturing bit (:206-212), N3 moves a
 * set bit one period left then right within its row, manufacturing row first
 * (:213-249), N4 swaps the two bits of a period where they differ (:250-257).
 * mm1/mr1 are written as 0 for single-period moves (the reference leaves them
 * unwritten; callers only read them when mp1 >= 0). */
int64_t orc_list_moves(int nbh, int64_t T, const uint8_t *sm, const uint8_t *sr,
                       int64_t *mp0, uint8_t *mm0, uint8_t *mr0, int64_t *mp1,
                       uint8_t *mm1, uint8_t *mr1)
{
    int64_t n = 0;
#define PUT1(t, m, r) \
    do { mp0[n] = (t); mm0[n] = (m); mr0[n] = (r); mp1[n] = -1; \
         mm1[n] = 0; mr1[n] = 0; ++n; } while (0)
#define PUT2(t, m, r, t1, m1, r1) \
    do { mp0[n] = (t); mm0[n] = (m); mr0[n] = (r); mp1[n] = (t1); \
         mm1[n] = (m1); mr1[n] = (r1); ++n; } while (0)
    if (nbh == 1) {
        for (int64_t t = 0; t < T; ++t)
            PUT1(t, !sm[t], sr[t]);
    } else if (nbh == 2) {
        for (int64_t t = 0; t < T; ++t)
            PUT1(t, sm[t], !sr[t]);
    } else if (nbh == 3) {
        for (int64_t t = 0; t < T; ++t) {
            if (!sm[t])
                continue;
            if (t > 0 && !sm[t - 1])
                PUT2(t, 0, sr[t], t - 1, 1, sr[t - 1]);
            if (t + 1 < T && !sm[t + 1])
                PUT2(t, 0, sr[t], t + 1, 1, sr[t + 1]);
        }
        for (int64_t t = 0; t < T; ++t) {
            if (!sr[t])
                continue;
            if (t > 0 && !sr[t - 1])
                PUT2(t, sm[t], 0, t - 1, sm[t - 1], 1);
            if (t + 1 < T && !sr[t + 1])
                PUT2(t, sm[t], 0, t + 1, sm[t + 1], 1);
        }
    } else if (nbh == 4) {
        for (int64_t t = 0; t < T; ++t)
            if (sm[t] != sr[t])
                PUT1(t, sr[t], sm[t]);
    }
#undef PUT1
#undef PUT2
    return n;
}

typedef struct {
    int64_t *dec, *p0, *p1;
    uint8_t *m0, *r0, *m1, *r1;
} orc_scan_out;

typedef struct {
    int64_t *mp0, *mp1;
    uint8_t *mm0, *mr0, *mm1, *mr1, *srow, *rrow;
} orc_scratch;

static int scratch_alloc(orc_scratch *s, int64_t T)
{
    int64_t cap = 2 * T + 2;
    s->mp0 = malloc(cap * sizeof(int64_t));
    s->mp1 = malloc(cap * sizeof(int64_t));
    s->mm0 = malloc(cap * 6 + 2 * T + 2);
    if (!s->mp0 || !s->mp1 || !s->mm0)
        return -1;
    s->mr0 = s->mm0 + cap;
    s->mm1 = s->mr0 + cap;
    s->mr1 = s->mm1 + cap;
    s->srow = s->mr1 + cap;
    s->rrow = s->srow + T + 1;
    return 0;
}

static void scratch_free(orc_scratch *s)
{
    free(s->mp0);
    free(s->mp1);
    free(s->mm0);
}

/* scan_products -- _kernels.py:261-325.  Per product: base cost on a copy
 * of the rows (:281-285); defaults dec=0, p0=p1=-1 (:286-288); skip an
 * infeasible base (:289-290); enumerate (:291); apply each move in scratch,
 * cost it, restore (:294-314); keep the first strict minimum (:315-317);
 * emit the winner (:318-325).  Returns the number of candidate evaluations
 * (row_cost calls at :308). */
static int64_t scan_range(const orc_inst *in, int64_t lo, int64_t hi,
                          const uint8_t *sm, const uint8_t *sr, int nbh,
                          const orc_scan_out *o, orc_scratch *s)
{
    const int64_t T = in->T;
    int64_t evals = 0;
    for (int64_t k = lo; k < hi; ++k) {
        const int64_t *d = in->dem + k * T, *r = in->ret + k * T;
        memcpy(s->srow, sm + k * T, T);
        memcpy(s->rrow, sr + k * T, T);
        int64_t base = orc_row_cost(T, s->srow, s->rrow, d, r, in->km[k],
                                    in->kr[k], in->hm[k], in->hr[k], in->pm[k],
                                    in->pr[k]);
        o->dec[k] = 0;
        o->p0[k] = -1;
        o->p1[k] = -1;
        if (base == ORC_INFEASIBLE)
            continue;
        int64_t n = orc_list_moves(nbh, T, s->srow, s->rrow, s->mp0, s->mm0,
                                   s->mr0, s->mp1, s->mm1, s->mr1);
        evals += n;
        int64_t best = base, bi = -1;
        for (int64_t i = 0; i < n; ++i) {
            int64_t t0 = s->mp0[i], t1 = s->mp1[i];
            uint8_t om0 = s->srow[t0], or0 = s->rrow[t0], om1 = 0, or1 = 0;
            s->srow[t0] = s->mm0[i];
            s->rrow[t0] = s->mr0[i];
            if (t1 >= 0) {
                om1 = s->srow[t1];
                or1 = s->rrow[t1];
                s->srow[t1] = s->mm1[i];
                s->rrow[t1] = s->mr1[i];
            }
            int64_t c = orc_row_cost(T, s->srow, s->rrow, d, r, in->km[k],
                                     in->kr[k], in->hm[k], in->hr[k],
                                     in->pm[k], in->pr[k]);
            s->srow[t0] = om0;
            s->rrow[t0] = or0;
            if (t1 >= 0) {
                s->srow[t1] = om1;
                s->rrow[t1] = or1;
            }
            if (c < best) {
                best = c;
                bi = i;
            }
        }
        if (bi >= 0) {
            o->dec[k] = base - best;
            o->p0[k] = s->mp0[bi];
            o->m0[k] = s->mm0[bi];
            o->r0[k] = s->mr0[bi];
            o->p1[k] = s->mp1[bi];
            o->m1[k] = s->mm1[bi];
            o->r1[k] = s->mr1[bi];
        }
    }
    return evals;
}

int64_t orc_scan_products(const orc_inst *in, int64_t lo, int64_t hi,
                          const uint8_t *sm, const uint8_t *sr, int nbh,
                          int64_t *dec, int64_t *p0, uint8_t *m0, uint8_t *r0,
                          int64_t *p1, uint8_t *m1, uint8_t *r1)
{
    orc_scan_out o = {dec, p0, p1, m0, r0, m1, r1};
    orc_scratch s;
    if (scratch_alloc(&s, in->T))
        return -1;
    int64_t e = scan_range(in, lo, hi, sm, sr, nbh, &o, &s);
    scratch_free(&s);
    return e;
}

/* apply_scan -- _kernels.py:328-344: write winners into the rows and return
 * the product-ordered sum of decreases. */
int64_t orc_apply_scan(int64_t T, int64_t lo, int64_t hi, const int64_t *dec,
                       const int64_t *p0, const uint8_t *m0, const uint8_t *r0,
                       const int64_t *p1, const uint8_t *m1, const uint8_t *r1,
                       uint8_t *sm, uint8_t *sr)
{
    int64_t diff = 0;
    for (int64_t k = lo; k < hi; ++k) {
        if (dec[k] <= 0)
            continue;
        sm[k * T + p0[k]] = m0[k];
        sr[k * T + p0[k]] = r0[k];
        if (p1[k] >= 0) {
            sm[k * T + p1[k]] = m1[k];
            sr[k * T + p1[k]] = r1[k];
        }
        diff += dec[k];
    }
    return diff;
}

/* ---- product-parallel lockstep VND (vnd.py:191-206, :253-289) ---------- */

typedef struct {
    const orc_inst *in;
    uint8_t *sm, *sr;
    orc_scan_out o;
    int k_max, nthreads;
    pthread_barrier_t bar;
    int64_t *part_diff, *part_evals; /* per thread */
    volatile int stop;
    volatile int nbh;
} vnd_shared;

typedef struct {
    vnd_shared *sh;
    int id;
    int64_t lo, hi;
} vnd_worker;

static void *vnd_thread(void *arg)
{
    vnd_worker *w = arg;
    vnd_shared *sh = w->sh;
    orc_scratch s;
    if (scratch_alloc(&s, sh->in->T))
        abort();
    for (;;) {
        pthread_barrier_wait(&sh->bar); /* pass start */
        if (sh->stop)
            break;
        int64_t e = scan_range(sh->in, w->lo, w->hi, sh->sm, sh->sr, sh->nbh,
                               &sh->o, &s);
        sh->part_evals[w->id] += e;
        /* disjoint ranges: apply our own winners, keep the partial sum */
        sh->part_diff[w->id] = orc_apply_scan(
            sh->in->T, w->lo, w->hi, sh->o.dec, sh->o.p0, sh->o.m0, sh->o.r0,
            sh->o.p1, sh->o.m1, sh->o.r1, sh->sm, sh->sr);
        pthread_barrier_wait(&sh->bar); /* pass end */
    }
    scratch_free(&s);
    return NULL;
}

/* vnd -- vnd.py:253-289.  cost = evaluate(start) (:268), then repeated
 * sweeps over neighborhoods 1..k_max; each pass scans every product, applies
 * all winners and subtracts the summed decrease (:277-288).  The trace gets
 * the start cost and one entry per pass (:269-270, :285-286).  stats =
 * {candidate evaluations, moves applied, sweeps}.  Returns 0, or -1 when the
 * trace capacity was too small (the run still completes). */
int orc_vnd(const orc_inst *in, int k_max, uint8_t *sm, uint8_t *sr,
            int nthreads, int64_t *cost_out, int64_t *trace, int64_t trace_cap,
            int64_t *n_trace, int64_t *stats)
{
    const int64_t K = in->K;
    int64_t *costs = malloc(K * sizeof(int64_t));
    int64_t *i64 = malloc(3 * K * sizeof(int64_t));
    uint8_t *u8 = calloc(4 * K, 1);
    if (!costs || !i64 || !u8)
        return -2;
    orc_product_costs(in, 0, K, sm, sr, costs);
    int64_t cost = 0;
    int infeasible = 0;
    for (int64_t k = 0; k < K; ++k) {
        if (costs[k] == ORC_INFEASIBLE)
            infeasible = 1;
        cost += costs[k];
    }
    if (infeasible) /* plan.py:117-126: any infeasible product -> sentinel */
        cost = ORC_INFEASIBLE;
    free(costs);
    int64_t nt = 0, moves = 0, sweeps = 0, evals = 0;
    int rc = 0;
    if (nt < trace_cap)
        trace[nt] = cost;
    ++nt;

    if (nthreads < 1)
        nthreads = 1;
    if (nthreads > K)
        nthreads = (int)K;
    vnd_shared sh;
    memset(&sh, 0, sizeof sh);
    sh.in = in;
    sh.sm = sm;
    sh.sr = sr;
    sh.o = (orc_scan_out){i64, i64 + K, i64 + 2 * K, u8, u8 + K, u8 + 2 * K,
                          u8 + 3 * K};
    sh.k_max = k_max;
    sh.nthreads = nthreads;
    sh.part_diff = calloc(nthreads, sizeof(int64_t));
    sh.part_evals = calloc(nthreads, sizeof(int64_t));
    pthread_barrier_init(&sh.bar, NULL, nthreads + 1);
    pthread_t *th = malloc(nthreads * sizeof(pthread_t));
    vnd_worker *ws = malloc(nthreads * sizeof(vnd_worker));
    for (int i = 0; i < nthreads; ++i) {
        ws[i].sh = &sh;
        ws[i].id = i;
        ws[i].lo = K * i / nthreads;
        ws[i].hi = K * (i + 1) / nthreads;
        pthread_create(&th[i], NULL, vnd_thread, &ws[i]);
    }
    for (;;) {
        int improvement = 0;
        ++sweeps;
        for (int nbh = 1; nbh <= k_max; ++nbh) {
            sh.nbh = nbh;
            pthread_barrier_wait(&sh.bar);
            pthread_barrier_wait(&sh.bar);
            int64_t diff = 0;
            for (int i = 0; i < nthreads; ++i)
                diff += sh.part_diff[i];
            for (int64_t k = 0; k < K; ++k)
                moves += i64[k] > 0;
            if (diff > 0) {
                cost -= diff;
                improvement = 1;
            }
            if (nt < trace_cap)
                trace[nt] = cost;
            else
                rc = -1;
            ++nt;
        }
        if (!improvement)
            break;
    }
    sh.stop = 1;
    pthread_barrier_wait(&sh.bar);
    for (int i = 0; i < nthreads; ++i) {
        pthread_join(th[i], NULL);
        evals += sh.part_evals[i];
    }
    pthread_barrier_destroy(&sh.bar);
    free(th);
    free(ws);
    free(sh.part_diff);
    free(sh.part_evals);
    free(i64);
    free(u8);
    *cost_out = cost;
    *n_trace = nt;
    stats[0] = evals;
    stats[1] = moves;
    stats[2] = sweeps;
    return rc;
}

/* initial_solution -- plan.py:140-167: lot-for-lot, remanufacture first as
 * far as recoverables reach, manufacture the remainder. */
void orc_initial_solution(const orc_inst *in, uint8_t *sm, uint8_t *sr)
{
    const int64_t T = in->T;
    memset(sm, 0, in->K * T);
    memset(sr, 0, in->K * T);
    for (int64_t k = 0; k < in->K; ++k) {
        int64_t avail = 0;
        for (int64_t t = 0; t < T; ++t) {
            avail += in->ret[k * T + t];
            int64_t d = in->dem[k * T + t];
            if (d <= 0)
                continue;
            int64_t take = avail < d ? avail : d;
            if (take > 0) {
                sr[k * T + t] = 1;
                avail -= take;
            }
            if (d - take > 0)
                sm[k * T + t] = 1;
        }
    }
}

/* decode -- _kernels.py:100-168 (row_decode): quantities and stocks of one
 * product; rows are zeroed when infeasible.  Used to check flow balance. */
int64_t orc_row_decode(int64_t T, const uint8_t *sm, const uint8_t *sr,
                       const int64_t *dem, const int64_t *ret, int64_t km,
                       int64_t kr, int64_t hm, int64_t hr, int64_t pm,
                       int64_t pr, int64_t *xm_o, int64_t *xr_o, int64_t *ym_o,
                       int64_t *yr_o)
{
    int64_t c = orc_row_cost(T, sm, sr, dem, ret, km, kr, hm, hr, pm, pr);
    memset(xm_o, 0, T * sizeof(int64_t));
    memset(xr_o, 0, T * sizeof(int64_t));
    memset(ym_o, 0, T * sizeof(int64_t));
    memset(yr_o, 0, T * sizeof(int64_t));
    if (c == ORC_INFEASIBLE)
        return c;
    int64_t rec = 0, stock = 0, t = 0;
    for (; t < T && !(sm[t] | sr[t]); ++t) {
        rec += ret[t];
        yr_o[t] = rec;
    }
    while (t < T) {
        int64_t u = t, v = t + 1;
        while (v < T && !(sm[v] | sr[v]))
            ++v;
        int64_t need = 0;
        for (int64_t i = u; i < v; ++i)
            need += dem[i];
        int64_t have = rec + ret[u];
        int64_t xr = sr[u] ? (need < have ? need : have) : 0;
        int64_t xm = need - xr;
        xr_o[u] = xr;
        xm_o[u] = xm;
        for (int64_t i = u; i < v; ++i) {
            if (i == u) {
                stock += xm + xr;
                rec += ret[i] - xr;
            } else {
                rec += ret[i];
            }
            stock -= dem[i];
            ym_o[i] = stock;
            yr_o[i] = rec;
        }
        t = v;
    }
    return c;
}
