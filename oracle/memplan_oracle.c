/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Not part of the product path.
 *
 * Plain-C restatement of the reference `memplan` algorithms on the hot path,
 * used by tests/ (parity checker), __graft_entry__.smoke() (checker) and
 * bench.py's cpu_baseline leg (the "port" CPU baseline).  Nothing in
 * paper_1804_10001_b200/ links or calls this file.
 *
 * Parity is pinned: tests/test_oracle.py checks every function here against
 * golden vectors produced by the reference itself (tests/golden/make_golden.py,
 * which imports /root/reference/pkg/src/memplan in the build container).
 *
 * Reference (read-only, /root/reference/pkg/src/memplan):
 *   orc_solve_bestfit   <- bestfit.py:276-309 (solve_bestfit), with
 *                          OffsetLineSet bestfit.py:61-201 and
 *                          _RemainingBlocks.take_best bestfit.py:243-262
 *   orc_verify          <- verifier.py:44-81 (verify_plan) over
 *                          core.py:227-249 (colliding_pairs)
 *   orc_clique_lb       <- core.py:252-268 (clique_lower_bound)
 *
 * Data model: arrays indexed by block index k = id-1 (ids are 1..n in input
 * order, core.py:106-111).  Times and sizes are int64 (the reference uses
 * Python ints; callers reject values outside int64).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int64_t steps;      /* loop iterations of bestfit.py:295 */
    int64_t lifts;      /* iterations where take_best returned None */
    int64_t sum_wlive;  /* sum over steps of live entries in [i0,i1) */
    int64_t max_lines;  /* max number of alive offset lines seen */
} orc_stats;

/* ---- skyline: doubly linked lines + lazy min-heap (bestfit.py:61-122) ---- */
typedef struct {
    int64_t lo, hi, h;
    int64_t prev, next; /* -1 = none */
    int alive;
} oline;

typedef struct { int64_t h, lo, seq, idx; } hent;

typedef struct {
    oline *ln; int64_t nln, cap;
    hent *hp; int64_t nhp, hcap;
    int64_t seq, first, nalive;
} skyline;

static int hless(const hent *a, const hent *b) {
    if (a->h != b->h) return a->h < b->h;
    if (a->lo != b->lo) return a->lo < b->lo;
    return a->seq < b->seq;
}

static void hpush(skyline *s, int64_t idx) {
    if (s->nhp == s->hcap) {
        s->hcap = s->hcap ? 2 * s->hcap : 64;
        s->hp = (hent *)realloc(s->hp, (size_t)s->hcap * sizeof(hent));
    }
    hent e = {s->ln[idx].h, s->ln[idx].lo, s->seq++, idx};
    int64_t i = s->nhp++;
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (!hless(&e, &s->hp[p])) break;
        s->hp[i] = s->hp[p];
        i = p;
    }
    s->hp[i] = e;
}

static void hpop(skyline *s) {
    hent last = s->hp[--s->nhp];
    int64_t i = 0, n = s->nhp;
    for (;;) {
        int64_t c = 2 * i + 1;
        if (c >= n) break;
        if (c + 1 < n && hless(&s->hp[c + 1], &s->hp[c])) c++;
        if (!hless(&s->hp[c], &last)) break;
        s->hp[i] = s->hp[c];
        i = c;
    }
    if (n) s->hp[i] = last;
}

static int64_t new_line(skyline *s, int64_t lo, int64_t hi, int64_t h) {
    if (s->nln == s->cap) {
        s->cap = s->cap ? 2 * s->cap : 64;
        s->ln = (oline *)realloc(s->ln, (size_t)s->cap * sizeof(oline));
    }
    oline *l = &s->ln[s->nln];
    l->lo = lo; l->hi = hi; l->h = h; l->prev = -1; l->next = -1; l->alive = 1;
    return s->nln++;
}

/* _splice, bestfit.py:124-147: replace chain first..last by repl[0..nr) */
static void splice(skyline *s, int64_t first, int64_t last, const int64_t *repl, int nr) {
    int64_t before = s->ln[first].prev, after = s->ln[last].next;
    for (int64_t k = first;; k = s->ln[k].next) {
        s->ln[k].alive = 0; s->nalive--;
        if (k == last) break;
    }
    for (int i = 0; i + 1 < nr; i++) {
        s->ln[repl[i]].next = repl[i + 1];
        s->ln[repl[i + 1]].prev = repl[i];
    }
    s->ln[repl[0]].prev = before;
    s->ln[repl[nr - 1]].next = after;
    if (before < 0) s->first = repl[0]; else s->ln[before].next = repl[0];
    if (after >= 0) s->ln[after].prev = repl[nr - 1];
    for (int i = 0; i < nr; i++) { hpush(s, repl[i]); s->nalive++; }
}

/* choose_offset, bestfit.py:115-122 */
static int64_t choose(skyline *s) {
    while (s->nhp && !s->ln[s->hp[0].idx].alive) hpop(s);
    return s->nhp ? s->hp[0].idx : -1;
}

/* place, bestfit.py:149-178 */
static int64_t place(skyline *s, int64_t line, int64_t a, int64_t f, int64_t size) {
    int64_t lo = s->ln[line].lo, hi = s->ln[line].hi, h = s->ln[line].h;
    int64_t repl[3]; int nr = 0;
    if (lo < a) repl[nr++] = new_line(s, lo, a, h);
    int64_t raised = new_line(s, a, f, h + size);
    repl[nr++] = raised;
    if (f < hi) repl[nr++] = new_line(s, f, hi, h);
    splice(s, line, line, repl, nr);
    int64_t p = s->ln[raised].prev;
    if (p >= 0 && s->ln[p].h == s->ln[raised].h) {
        int64_t m = new_line(s, s->ln[p].lo, s->ln[raised].hi, s->ln[raised].h);
        splice(s, p, raised, &m, 1);
        raised = m;
    }
    int64_t q = s->ln[raised].next;
    if (q >= 0 && s->ln[q].h == s->ln[raised].h) {
        int64_t m = new_line(s, s->ln[raised].lo, s->ln[q].hi, s->ln[raised].h);
        splice(s, raised, q, &m, 1);
    }
    return h;
}

/* lift_up, bestfit.py:180-201; returns -1 on IllegalLift */
static int lift(skyline *s, int64_t line) {
    int64_t p = s->ln[line].prev, q = s->ln[line].next, m;
    if (p < 0 && q < 0) return -1;
    if (p < 0) {
        m = new_line(s, s->ln[line].lo, s->ln[q].hi, s->ln[q].h); splice(s, line, q, &m, 1);
    } else if (q < 0) {
        m = new_line(s, s->ln[p].lo, s->ln[line].hi, s->ln[p].h); splice(s, p, line, &m, 1);
    } else if (s->ln[p].h == s->ln[q].h) {
        m = new_line(s, s->ln[p].lo, s->ln[q].hi, s->ln[p].h); splice(s, p, q, &m, 1);
    } else if (s->ln[p].h < s->ln[q].h) {
        m = new_line(s, s->ln[p].lo, s->ln[line].hi, s->ln[p].h); splice(s, p, line, &m, 1);
    } else {
        m = new_line(s, s->ln[line].lo, s->ln[q].hi, s->ln[q].h); splice(s, line, q, &m, 1);
    }
    return 0;
}

/* ---- remaining blocks sorted by (alloc, id), bestfit.py:231-241 ---- */
static const int64_t *g_alloc_for_sort;
static int cmp_alloc_id(const void *x, const void *y) {
    int64_t i = *(const int64_t *)x, j = *(const int64_t *)y;
    int64_t ai = g_alloc_for_sort[i], aj = g_alloc_for_sort[j];
    if (ai != aj) return ai < aj ? -1 : 1;
    return i < j ? -1 : (i > j);
}

static int64_t lower_bound(const int64_t *v, int64_t n, int64_t x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (v[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/*
 * solve_bestfit (bestfit.py:276-309).  offsets_out[k] receives the offset of
 * block id k+1.  Returns 0 on success, 1 if the loop bound assert
 * (bestfit.py:297) fires, 2 on IllegalLift (bestfit.py:185-186).
 */
int orc_solve_bestfit(int64_t n, const int64_t *alloc, const int64_t *free_,
                      const int64_t *size, int64_t *offsets_out,
                      int64_t *peak_out, orc_stats *st) {
    orc_stats local = {0, 0, 0, 0};
    if (!st) st = &local;
    memset(st, 0, sizeof(*st));
    *peak_out = 0;
    if (n == 0) return 0; /* R1, bestfit.py:285-286 */
    int64_t t_lo = alloc[0], t_hi = free_[0];
    for (int64_t k = 1; k < n; k++) {
        if (alloc[k] < t_lo) t_lo = alloc[k];
        if (free_[k] > t_hi) t_hi = free_[k];
    }
    skyline s; memset(&s, 0, sizeof(s));
    s.first = new_line(&s, t_lo, t_hi, 0);
    hpush(&s, s.first); s.nalive = 1;

    /* SoA columns in (alloc, id) order; compacted like bestfit.py:264-273 */
    int64_t *ord = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    for (int64_t k = 0; k < n; k++) ord[k] = k;
    g_alloc_for_sort = alloc;
    qsort(ord, (size_t)n, sizeof(int64_t), cmp_alloc_id);
    int64_t *sa = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *sf = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *ss = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    unsigned char *live = (unsigned char *)malloc((size_t)n);
    for (int64_t i = 0; i < n; i++) {
        int64_t k = ord[i];
        sa[i] = alloc[k]; sf[i] = free_[k]; ss[i] = size[k]; live[i] = 1;
    }
    int64_t m = n, dead = 0;

    int rc = 0;
    int64_t placed = 0, peak = 0;
    while (placed < n) {
        st->steps++;
        if (st->steps > 3 * n + 4) { rc = 1; break; } /* R8 */
        if (s.nalive > st->max_lines) st->max_lines = s.nalive;
        int64_t line = choose(&s);
        int64_t lo = s.ln[line].lo, hi = s.ln[line].hi;
        /* take_best (bestfit.py:243-262): window, fit mask, key max of
         * (lifetime, size, -id) */
        int64_t i0 = lower_bound(sa, m, lo), i1 = lower_bound(sa, m, hi);
        int64_t best = -1, bl = 0, bs = 0, bk = 0;
        for (int64_t i = i0; i < i1; i++) {
            if (!live[i]) continue;
            st->sum_wlive++;
            if (sf[i] > hi) continue;
            int64_t life = sf[i] - sa[i];
            if (best < 0 || life > bl || (life == bl && (ss[i] > bs ||
                (ss[i] == bs && ord[i] < bk)))) {
                best = i; bl = life; bs = ss[i]; bk = ord[i];
            }
        }
        if (best < 0) {
            st->lifts++;
            if (lift(&s, line)) { rc = 2; break; }
            continue;
        }
        live[best] = 0;
        dead++;
        int64_t k = ord[best];
        int64_t off = place(&s, line, alloc[k], free_[k], size[k]);
        offsets_out[k] = off;
        if (off + size[k] > peak) peak = off + size[k];
        placed++;
        if (dead * 2 > m) {
            int64_t w = 0;
            for (int64_t i = 0; i < m; i++) {
                if (!live[i]) continue;
                sa[w] = sa[i]; sf[w] = sf[i]; ss[w] = ss[i]; ord[w] = ord[i]; live[w] = 1;
                w++;
            }
            m = w;
            dead = 0;
        }
    }
    *peak_out = peak;
    free(ord); free(sa); free(sf); free(ss); free(live); free(s.ln); free(s.hp);
    return rc;
}

/* ---- verification (verifier.py:44-81 over core.py:227-249) ---- */
typedef struct {
    int64_t i, j;            /* 1-based ids, i < j */
    int64_t overlap_bytes;
    int64_t overlap_ticks;
} orc_violation;

typedef struct {
    int64_t n_violations;
    int64_t peak;            /* peak_recomputed */
    int32_t offsets_ok;      /* all offsets >= 0 */
    int32_t pad;
    uint64_t used_lo, used_hi; /* sum size*lifetime as unsigned 128-bit */
} orc_verify_out;

static int cmp_viol(const void *x, const void *y) {
    const orc_violation *a = (const orc_violation *)x, *b = (const orc_violation *)y;
    if (a->i != b->i) return a->i < b->i ? -1 : 1;
    return a->j < b->j ? -1 : (a->j > b->j);
}

/*
 * Enumerates exactly the colliding pairs E (intersecting half-open
 * lifetimes) with a sort+sweep — independent of the GPU validator's tiling —
 * and reports every pair whose address ranges intersect.  Violations are
 * sorted by (i, j) like verifier.py:57; at most viol_cap are stored.
 */
int orc_verify(int64_t n, const int64_t *alloc, const int64_t *free_,
               const int64_t *size, const int64_t *offsets,
               orc_verify_out *out, orc_violation *viol, int64_t viol_cap) {
    memset(out, 0, sizeof(*out));
    out->offsets_ok = 1;
    unsigned __int128 used = 0;
    for (int64_t k = 0; k < n; k++) {
        if (offsets[k] < 0) out->offsets_ok = 0;
        if (offsets[k] + size[k] > out->peak) out->peak = offsets[k] + size[k];
        used += (unsigned __int128)(uint64_t)size[k] * (uint64_t)(free_[k] - alloc[k]);
    }
    out->used_lo = (uint64_t)used;
    out->used_hi = (uint64_t)(used >> 64);
    if (n == 0) return 0;
    int64_t *ord = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    for (int64_t k = 0; k < n; k++) ord[k] = k;
    g_alloc_for_sort = alloc;
    qsort(ord, (size_t)n, sizeof(int64_t), cmp_alloc_id);
    int64_t stored = 0;
    for (int64_t p = 0; p < n; p++) {
        int64_t a = ord[p];
        for (int64_t q = p + 1; q < n; q++) {
            int64_t b = ord[q];
            if (alloc[b] >= free_[a]) break; /* sorted: no later q collides */
            int64_t lo = offsets[a] > offsets[b] ? offsets[a] : offsets[b];
            int64_t ea = offsets[a] + size[a], eb = offsets[b] + size[b];
            int64_t hi = ea < eb ? ea : eb;
            if (hi > lo) {
                out->n_violations++;
                if (stored < viol_cap) {
                    orc_violation *v = &viol[stored++];
                    v->i = (a < b ? a : b) + 1;
                    v->j = (a < b ? b : a) + 1;
                    v->overlap_bytes = hi - lo;
                    int64_t tl = alloc[a] > alloc[b] ? alloc[a] : alloc[b];
                    int64_t th = free_[a] < free_[b] ? free_[a] : free_[b];
                    v->overlap_ticks = th - tl;
                }
            }
        }
    }
    free(ord);
    if (stored > 1) qsort(viol, (size_t)stored, sizeof(orc_violation), cmp_viol);
    return 0;
}

/* ---- clique_lower_bound (core.py:252-268): frees sort before allocs ---- */
typedef struct { int64_t t; int kind; int64_t sz; } oev;
static int cmp_ev(const void *x, const void *y) {
    const oev *a = (const oev *)x, *b = (const oev *)y;
    if (a->t != b->t) return a->t < b->t ? -1 : 1;
    if (a->kind != b->kind) return a->kind - b->kind;
    return a->sz < b->sz ? -1 : (a->sz > b->sz);
}

int64_t orc_clique_lb(int64_t n, const int64_t *alloc, const int64_t *free_,
                      const int64_t *size) {
    oev *ev = (oev *)malloc((size_t)(2 * n + 1) * sizeof(oev));
    for (int64_t k = 0; k < n; k++) {
        ev[2 * k] = (oev){alloc[k], 1, size[k]};
        ev[2 * k + 1] = (oev){free_[k], 0, size[k]};
    }
    qsort(ev, (size_t)(2 * n), sizeof(oev), cmp_ev);
    int64_t live = 0, best = 0;
    for (int64_t i = 0; i < 2 * n; i++) {
        if (ev[i].kind == 0) live -= ev[i].sz;
        else { live += ev[i].sz; if (live > best) best = live; }
    }
    free(ev);
    return best;
}
