/*
 * cc_oracle.c -- plain, slow, single-threaded CPU oracle for the FoF-connectivity correction
 * of arXiv 2604.18801 ("Preserving Clusters in Error-Bounded Lossy Compression of Particle
 * Data").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header, table or constant
 * generator with the CUDA path (paper_2604_18801_b200/csrc); neither side includes the other.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (one paragraph per line), with the
 * section / equation / algorithm it falls in.  "R<k>" = the reading k listed in DESIGN.md §3
 * (where the paper is silent or ambiguous).
 *
 * Arithmetic contract (R4): every distance is the fp32 expression
 *     dx = fl(xj - xi); periodic: if dx > hL: dx = fl(dx - L) else if dx < -hL: dx = fl(dx + L)
 *     d2 = fl(fl(fl(dx*dx) + fl(dy*dy)) + fl(dz*dz))
 * compiled with -ffp-contract=off (no FMA), no -ffast-math, SSE fp32 (FLT_EVAL_METHOD 0).
 *
 * Parity status of each entry point is stated in DESIGN.md §4; every function here is pinned
 * by a -m "not gpu" test against something other than itself (brute force, scipy, sklearn,
 * torch.optim.Adam, finite differences, worked examples).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OC_VERSION 1

typedef struct {
    double L;            /* cubic box side */
    int periodic;        /* 1: minimum-image distances (§III intro) */
    double b;            /* linking length, absolute (§II-B) */
    double xi;           /* absolute per-coordinate error bound (§III-A); rounded to fp32 */
    int m;               /* edit bit depth (Alg. 1 REQUIRE; m = 16) */
    double alpha, beta1, beta2, eps_adam; /* Adam */
    int t_max;           /* Alg. 1 T_max */
    double eps_loss;     /* Alg. 1 epsilon_L */
    int stop_mode;       /* 0: stop when no L_tight-active pair (R11); 1: L_tight <= eps_loss
                            (Alg. 1 line 6); 2: never stop early (exactly t_max updates);
                            3: L_tight <= eps_loss and every link status restored (MCC = 1) */
    int optimizer;       /* 0: Adam; 1: vanilla projected gradient */
    double vanilla_step; /* step for optimizer 1 (Alg. 1 line 9 "P - alpha g") */
} oc_cfg;

typedef struct {
    float Lf, hLf;       /* fl32(L), fl32(L/2) */
    float xi_f;          /* fl32(xi): THE bound of every invariant (R6) */
    float xip_f;         /* RD32(xi (1 - 2^-m)): xi' (Alg. 1 line 2; R8) */
    float b2;            /* fl32(b^2): link iff d2 <= b2 (R3) */
    float lo2, hi2;      /* band (b - 2 sqrt3 xi, b + 2 sqrt3 xi] squared, fp32 (R2) */
    float c_b, c_f;      /* fl32(b -/+ 2 sqrt3 eps_q): L_tight thresholds (Eq. 3) */
    float pad;
    double xi, eps_q, mu, band_lo, band_hi;
} oc_th;

typedef struct {
    int64_t iterations;      /* updates performed (R27) */
    int64_t active0;         /* L_tight-active pairs at P_hat^(0) */
    int64_t active_final;    /* L_tight-active pairs at the returned positions */
    int64_t violated0;       /* pairs whose link status differs at P_hat^(0) (Eq. 1 support) */
    int64_t violated_final;
    double loss0, loss_final;/* L_tight: the exact sum of the fp32 terms e^2, rounded (R16) */
    int64_t n_editable;
    int converged;           /* active_final == 0 (stop_mode 0/2) or loss_final <= eps_loss (1) */
    int pad;
} oc_corr_info;

int oc_version(void) { return OC_VERSION; }
void oc_free(void* p) { free(p); }

/* ---------------------------------------------------------------------------------------- */
/* directed fp32 rounding of an exact sum a + b of two doubles (R8)                        */
static float rd32_sum(double a, double b) {
    double s = a + b, bb = s - a, err = (a - (s - bb)) + (b - bb);
    float f = (float)s;
    if ((double)f > s || ((double)f == s && err < 0)) f = nextafterf(f, -INFINITY);
    return f;
}
static float ru32_sum(double a, double b) {
    double s = a + b, bb = s - a, err = (a - (s - bb)) + (b - bb);
    float f = (float)s;
    if ((double)f < s || ((double)f == s && err > 0)) f = nextafterf(f, INFINITY);
    return f;
}

/* S0 parameters -- Alg. 1 lines 1-3, §III-B. */
int oc_thresholds(const oc_cfg* c, oc_th* t) {
    if (!c || !t) return 64;
    if (!(c->L > 0) || !(c->b > 0) || !(c->xi >= 0) || c->m < 2 || c->m > 52) return 64;
    memset(t, 0, sizeof(*t));
    t->xi_f = (float)c->xi;
    double xi = (double)t->xi_f;
    t->xi = xi;
    t->xip_f = rd32_sum(xi * (1.0 - ldexp(1.0, -c->m)), 0.0);          /* xi' = xi(1-2^-m) */
    t->eps_q = 2.0 * xi / (ldexp(1.0, c->m) - 1.0);                      /* eps_q = 2xi/(2^m-1) */
    t->mu = 2.0 * sqrt(3.0) * t->eps_q;                                  /* margin 2 sqrt3 eps_q */
    t->c_b = (float)(c->b - t->mu);
    t->c_f = (float)(c->b + t->mu);
    double s = 2.0 * sqrt(3.0) * xi;                                     /* 2 sqrt3 xi */
    t->band_lo = c->b - s;
    t->band_hi = c->b + s;
    t->lo2 = t->band_lo > 0 ? (float)(t->band_lo * t->band_lo) : -1.0f;
    t->hi2 = (float)(t->band_hi * t->band_hi);
    t->b2 = (float)(c->b * c->b);
    t->Lf = (float)c->L;
    t->hLf = (float)(0.5 * c->L);
    return 0;
}

/* pinned fp32 minimum-image component (R4, R5) */
static float mi(float d, const oc_th* t, int periodic) {
    if (periodic) {
        if (d > t->hLf) d = d - t->Lf;
        else if (d < -t->hLf) d = d + t->Lf;
    }
    return d;
}

/* pinned fp32 squared distance from particle i to particle j (R4) */
static float dist2(float xi_, float yi, float zi, float xj, float yj, float zj, const oc_th* t,
                   int periodic) {
    float dx = mi(xj - xi_, t, periodic);
    float dy = mi(yj - yi, t, periodic);
    float dz = mi(zj - zi, t, periodic);
    float s = dx * dx;
    s = s + dy * dy;
    s = s + dz * dz;
    return s;
}

float oc_dist2(const float* pi, const float* pj, const oc_cfg* c) {
    oc_th t;
    if (oc_thresholds(c, &t)) return -1.0f;
    return dist2(pi[0], pi[1], pi[2], pj[0], pj[1], pj[2], &t, c->periodic);
}

/* ---------------------------------------------------------------------------------------- */
/* a plain uniform grid (§II-B-1; §III-B): n cells per axis of width L/n >= wmin, */
/* at most max(N,1) cells (SPEC S:112's rule); cell of a coordinate computed in fp64.        */
typedef struct {
    int64_t n;            /* cells per axis */
    double w;
    int64_t* start;       /* n^3 + 1 */
    int64_t* idx;         /* particle indices grouped by cell */
} grid_t;

static int64_t cell_of(double x, const grid_t* g, double L, int periodic) {
    if (periodic) x = x - L * floor(x / L);
    int64_t c = (int64_t)floor(x / g->w);
    if (c < 0) c = 0;
    if (c > g->n - 1) c = g->n - 1;
    return c;
}

static int grid_build(grid_t* g, int64_t n, const float* x, const float* y, const float* z,
                      double L, double wmin, int periodic) {
    double kd = floor(L / wmin);
    int64_t cap = n > 1 ? n : 1;
    double kc = floor(cbrt((double)cap)) + 1.0;
    int64_t k = (int64_t)(kd < kc ? kd : kc);
    if (k < 1) k = 1;
    while (k > 1 && k * k * k > cap) k--;
    g->n = k;
    g->w = L / (double)k;
    int64_t nc = k * k * k;
    g->start = (int64_t*)calloc((size_t)(nc + 1), sizeof(int64_t));
    g->idx = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    int64_t* key = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    if (!g->start || !g->idx || !key) { free(key); return 67; }
    for (int64_t i = 0; i < n; i++) {
        int64_t cx = cell_of(x[i], g, L, periodic), cy = cell_of(y[i], g, L, periodic),
                cz = cell_of(z[i], g, L, periodic);
        key[i] = (cz * k + cy) * k + cx;
        g->start[key[i] + 1]++;
    }
    for (int64_t c = 0; c < nc; c++) g->start[c + 1] += g->start[c];
    int64_t* fill = (int64_t*)malloc((size_t)nc * sizeof(int64_t));
    if (!fill) { free(key); return 67; }
    memcpy(fill, g->start, (size_t)nc * sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) g->idx[fill[key[i]]++] = i;
    free(fill);
    free(key);
    return 0;
}

static void grid_free(grid_t* g) {
    free(g->start);
    free(g->idx);
}

/* distinct neighbour cells (offsets -1..1 per axis, periodic wrap, de-duplicated: R1) */
static int grid_neigh(const grid_t* g, int64_t c, int periodic, int64_t* out) {
    int64_t k = g->n, cx = c % k, cy = (c / k) % k, cz = c / (k * k);
    int cnt = 0;
    for (int dz = -1; dz <= 1; dz++)
        for (int dy = -1; dy <= 1; dy++)
            for (int dx = -1; dx <= 1; dx++) {
                int64_t nx = cx + dx, ny = cy + dy, nz = cz + dz;
                if (periodic) {
                    nx = (nx + k) % k; ny = (ny + k) % k; nz = (nz + k) % k;
                } else if (nx < 0 || ny < 0 || nz < 0 || nx >= k || ny >= k || nz >= k) {
                    continue;
                }
                int64_t cc = (nz * k + ny) * k + nx;
                int dup = 0;
                for (int q = 0; q < cnt; q++) dup |= (out[q] == cc);
                if (!dup) out[cnt++] = cc;
            }
    return cnt;
}

/* ---------------------------------------------------------------------------------------- */
/* growable pair list */
typedef struct { int64_t n, cap; int64_t* i; int64_t* j; uint8_t* f; } plist_t;

static int plist_push(plist_t* p, int64_t i, int64_t j, uint8_t f) {
    if (p->n == p->cap) {
        int64_t nc = p->cap ? p->cap * 2 : 1024;
        int64_t* ni = (int64_t*)realloc(p->i, (size_t)nc * sizeof(int64_t));
        if (!ni) return 67;
        p->i = ni;
        int64_t* nj = (int64_t*)realloc(p->j, (size_t)nc * sizeof(int64_t));
        if (!nj) return 67;
        p->j = nj;
        uint8_t* nf = (uint8_t*)realloc(p->f, (size_t)nc);
        if (!nf) return 67;
        p->f = nf;
        p->cap = nc;
    }
    p->i[p->n] = i; p->j[p->n] = j; p->f[p->n] = f; p->n++;
    return 0;
}

static const uint32_t* g_sort_gid;
static int64_t* g_sort_pi;
static int64_t* g_sort_pj;
static int cmp_pair(const void* a, const void* b) {
    int64_t ka = *(const int64_t*)a, kb = *(const int64_t*)b;
    uint32_t ai = g_sort_gid ? g_sort_gid[g_sort_pi[ka]] : (uint32_t)g_sort_pi[ka];
    uint32_t bi = g_sort_gid ? g_sort_gid[g_sort_pi[kb]] : (uint32_t)g_sort_pi[kb];
    if (ai != bi) return ai < bi ? -1 : 1;
    uint32_t aj = g_sort_gid ? g_sort_gid[g_sort_pj[ka]] : (uint32_t)g_sort_pj[ka];
    uint32_t bj = g_sort_gid ? g_sort_gid[g_sort_pj[kb]] : (uint32_t)g_sort_pj[kb];
    if (aj != bj) return aj < bj ? -1 : 1;
    return 0;
}

/*
 * O2 -- vulnerable pairs V (§III-A; Alg. 1 line 3 P:421):
 *   (i,j) in V  iff  lo2 < d2(p_i,p_j) <= hi2   (half-open band, R2),
 * each pair tagged bit0 = original link (d2 <= b2, R3) and
 *                  bit1 = decompressed link (d2(p_hat_i, p_hat_j) <= b2).
 * mode 0: cell grid of width >= sqrt(hi2)(1+1e-5); mode 1: brute force O(N^2).
 * Output: canonical list (gid[i] < gid[j]) sorted by (gid[i], gid[j]); arrays malloc'ed,
 * caller frees with oc_free.  Returns |V| or a negative status.
 */
int64_t oc_find_pairs(int64_t n, const float* x, const float* y, const float* z,
                      const float* xh, const float* yh, const float* zh, const uint32_t* gid,
                      const oc_cfg* c, int mode, int64_t** out_i, int64_t** out_j,
                      uint8_t** out_f) {
    oc_th t;
    int st = oc_thresholds(c, &t);
    if (st) return -st;
    plist_t p = {0, 0, NULL, NULL, NULL};
    int per = c->periodic;
#define OC_TEST_PAIR(I, J)                                                                   \
    do {                                                                                      \
        int64_t a_ = (I), b_ = (J);                                                           \
        float d2_ = dist2(x[a_], y[a_], z[a_], x[b_], y[b_], z[b_], &t, per);                 \
        if (t.lo2 < d2_ && d2_ <= t.hi2) {                                                    \
            float h2_ = dist2(xh[a_], yh[a_], zh[a_], xh[b_], yh[b_], zh[b_], &t, per);       \
            uint8_t f_ = (uint8_t)((d2_ <= t.b2 ? 1 : 0) | (h2_ <= t.b2 ? 2 : 0));            \
            uint32_t ga_ = gid ? gid[a_] : (uint32_t)a_, gb_ = gid ? gid[b_] : (uint32_t)b_;  \
            if (ga_ < gb_) st = plist_push(&p, a_, b_, f_);                                   \
            else st = plist_push(&p, b_, a_, f_);                                             \
            if (st) goto fail;                                                                \
        }                                                                                     \
    } while (0)
    if (mode == 1) {
        for (int64_t i = 0; i < n; i++)
            for (int64_t j = i + 1; j < n; j++) OC_TEST_PAIR(i, j);
    } else {
        grid_t g;
        st = grid_build(&g, n, x, y, z, c->L, sqrt((double)t.hi2) * (1.0 + 1e-5), per);
        if (st) { grid_free(&g); goto fail; }
        int64_t nc = g.n * g.n * g.n, nb[27];
        for (int64_t cc = 0; cc < nc; cc++) {
            if (g.start[cc] == g.start[cc + 1]) continue;
            int cnt = grid_neigh(&g, cc, per, nb);
            for (int64_t a = g.start[cc]; a < g.start[cc + 1]; a++) {
                int64_t i = g.idx[a];
                for (int q = 0; q < cnt; q++)
                    for (int64_t bq = g.start[nb[q]]; bq < g.start[nb[q] + 1]; bq++) {
                        int64_t j = g.idx[bq];
                        if (j > i) OC_TEST_PAIR(i, j);
                    }
            }
        }
        grid_free(&g);
    }
#undef OC_TEST_PAIR
    {
        int64_t* ord = (int64_t*)malloc((size_t)(p.n > 0 ? p.n : 1) * sizeof(int64_t));
        int64_t* oi = (int64_t*)malloc((size_t)(p.n > 0 ? p.n : 1) * sizeof(int64_t));
        int64_t* oj = (int64_t*)malloc((size_t)(p.n > 0 ? p.n : 1) * sizeof(int64_t));
        uint8_t* of = (uint8_t*)malloc((size_t)(p.n > 0 ? p.n : 1));
        if (!ord || !oi || !oj || !of) { free(ord); free(oi); free(oj); free(of); st = 67; goto fail; }
        for (int64_t k = 0; k < p.n; k++) ord[k] = k;
        g_sort_gid = gid; g_sort_pi = p.i; g_sort_pj = p.j;
        qsort(ord, (size_t)p.n, sizeof(int64_t), cmp_pair);
        for (int64_t k = 0; k < p.n; k++) { oi[k] = p.i[ord[k]]; oj[k] = p.j[ord[k]]; of[k] = p.f[ord[k]]; }
        free(ord);
        free(p.i); free(p.j); free(p.f);
        *out_i = oi; *out_j = oj; *out_f = of;
        return p.n;
    }
fail:
    free(p.i); free(p.j); free(p.f);
    return -st;
}

/* per-pair link status on arbitrary positions (for MCC, §IV-A): out[k] = d2 <= b2 */
int oc_pair_links(int64_t np, const int64_t* pi, const int64_t* pj, const float* x,
                  const float* y, const float* z, const oc_cfg* c, uint8_t* out) {
    oc_th t;
    int st = oc_thresholds(c, &t);
    if (st) return st;
    for (int64_t k = 0; k < np; k++) {
        int64_t i = pi[k], j = pj[k];
        out[k] = dist2(x[i], y[i], z[i], x[j], y[j], z[j], &t, c->periodic) <= t.b2;
    }
    return 0;
}

/* ---------------------------------------------------------------------------------------- */
/*
 * O6 -- FoF labels (§II-B, Fig. 1): edge iff d2(p_i,p_j) <= b2 (pinned fp32, R3/R4);
 * clusters = connected components; label = minimum gid of the component (R20).
 * Sequential union-find (path compression + union by size).  mode 0: grid of width
 * >= sqrt(b2)(1+1e-5) built on the positions being labelled; mode 1: brute force.
 * Returns the number of components, or a negative status.
 */
static int64_t uf_find(int64_t* par, int64_t a) {
    int64_t r = a;
    while (par[r] != r) r = par[r];
    while (par[a] != r) { int64_t nx = par[a]; par[a] = r; a = nx; }
    return r;
}
static void uf_union(int64_t* par, int64_t* sz, int64_t a, int64_t b) {
    a = uf_find(par, a); b = uf_find(par, b);
    if (a == b) return;
    if (sz[a] < sz[b]) { int64_t tmp = a; a = b; b = tmp; }
    par[b] = a;
    sz[a] += sz[b];
}

int64_t oc_fof(int64_t n, const float* x, const float* y, const float* z, const uint32_t* gid,
               const oc_cfg* c, int mode, uint32_t* labels) {
    oc_th t;
    int st = oc_thresholds(c, &t);
    if (st) return -st;
    int per = c->periodic;
    int64_t* par = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    int64_t* sz = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    if (!par || !sz) { free(par); free(sz); return -67; }
    for (int64_t i = 0; i < n; i++) { par[i] = i; sz[i] = 1; }
    if (mode == 1) {
        for (int64_t i = 0; i < n; i++)
            for (int64_t j = i + 1; j < n; j++)
                if (dist2(x[i], y[i], z[i], x[j], y[j], z[j], &t, per) <= t.b2) uf_union(par, sz, i, j);
    } else {
        grid_t g;
        st = grid_build(&g, n, x, y, z, c->L, sqrt((double)t.b2) * (1.0 + 1e-5), per);
        if (st) { grid_free(&g); free(par); free(sz); return -st; }
        int64_t nc = g.n * g.n * g.n, nb[27];
        for (int64_t cc = 0; cc < nc; cc++) {
            if (g.start[cc] == g.start[cc + 1]) continue;
            int cnt = grid_neigh(&g, cc, per, nb);
            for (int64_t a = g.start[cc]; a < g.start[cc + 1]; a++) {
                int64_t i = g.idx[a];
                for (int q = 0; q < cnt; q++)
                    for (int64_t bq = g.start[nb[q]]; bq < g.start[nb[q] + 1]; bq++) {
                        int64_t j = g.idx[bq];
                        if (j > i && dist2(x[i], y[i], z[i], x[j], y[j], z[j], &t, per) <= t.b2)
                            uf_union(par, sz, i, j);
                    }
            }
        }
        grid_free(&g);
    }
    /* canonical labels: min gid over each component */
    uint32_t* mn = (uint32_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(uint32_t));
    if (!mn) { free(par); free(sz); return -67; }
    for (int64_t i = 0; i < n; i++) mn[i] = 0xFFFFFFFFu;
    int64_t groups = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t r = uf_find(par, i);
        uint32_t gi = gid ? gid[i] : (uint32_t)i;
        if (r == i) groups++;
        if (gi < mn[r]) mn[r] = gi;
    }
    for (int64_t i = 0; i < n; i++) labels[i] = mn[uf_find(par, i)];
    free(mn); free(par); free(sz);
    return groups;
}

/* ---------------------------------------------------------------------------------------- */
/*
 * L_tight pair term in the pinned fp32 form used by the PGD (Eq. 3; R13, R14):
 *   r   = minimg(p_hat_i - p_hat_j) (fp32),  dh = sqrt_rn(fl(fl(rx^2 + ry^2) + rz^2))
 *   broken side  (orig linked):   active iff dh >  c_b,  e = fl(dh - c_b)
 *   false side   (orig unlinked): active iff dh <= c_f,  e = fl(dh - c_f)
 *   term (reporting) = (double)e * (double)e
 */
static int tight_pair(const float* P, int64_t i, int64_t j, int olink, const oc_th* t,
                      int periodic, float r[3], float* dh, float* e) {
    r[0] = mi(P[3 * i + 0] - P[3 * j + 0], t, periodic);
    r[1] = mi(P[3 * i + 1] - P[3 * j + 1], t, periodic);
    r[2] = mi(P[3 * i + 2] - P[3 * j + 2], t, periodic);
    float s = r[0] * r[0];
    s = s + r[1] * r[1];
    s = s + r[2] * r[2];
    float d = sqrtf(s);
    *dh = d;
    if (olink) {
        if (d > t->c_b) { *e = d - t->c_b; return 1; }
    } else {
        if (d <= t->c_f) { *e = d - t->c_f; return 1; }
    }
    *e = 0.0f;
    return 0;
}

/* gradient contribution of one active pair to endpoint i (R14, R15):
 *   g_i += fl(k * r)  with  k = fl(fl(2e) / dh)          if dh > 0
 *   g_i.x += fl(2e) * (+1 if gid_i < gid_j else -1)      if dh == 0 (coincident)           */
static void grad_add(float g[3], const float r[3], float dh, float e, int i_is_lower) {
    float two_e = 2.0f * e;
    if (dh > 0.0f) {
        float k = two_e / dh;
        g[0] = g[0] + k * r[0];
        g[1] = g[1] + k * r[1];
        g[2] = g[2] + k * r[2];
    } else {
        g[0] = g[0] + (i_is_lower ? two_e : -two_e);
    }
}

typedef struct { int64_t j; uint32_t gj; int olink; } rent_t;

/* gradient summation order (R14): chunks of GC terms, trees over groups of GG chunk sums */
#define GC 16
#define GG 32
static int cmp_rent(const void* a, const void* b) {
    uint32_t x = ((const rent_t*)a)->gj, y = ((const rent_t*)b)->gj;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* Exact sum of doubles (R16, R28): the real number L_tight = sum of e^2 (each e^2 exact in fp64,
 * e being fp32) is held as a nonoverlapping expansion -- Shewchuk's "grow-expansion", the
 * partials of Python's math.fsum -- so the stop test L_tight <= eps_L (Alg. 1 line 6)
 * is decided on the exact value, not on a rounded running sum.  Components are nonoverlapping
 * and increase in magnitude; at most ~40 are non-zero for doubles. */
typedef struct { int n; double p[96]; } xsum_t;

static void xsum_add(xsum_t* s, double x) {
    int i = 0;
    for (int k = 0; k < s->n; k++) {
        double y = s->p[k];
        if (fabs(x) < fabs(y)) { double tmp = x; x = y; y = tmp; }
        double hi = x + y, lo = y - (hi - x);
        if (lo != 0.0) s->p[i++] = lo;
        x = hi;
    }
    s->p[i++] = x;
    s->n = i;
}

/* sign of (exact sum - v): the sign of the largest non-zero component of the expansion */
static int xsum_cmp(const xsum_t* s, double v) {
    xsum_t t = *s;
    xsum_add(&t, -v);
    for (int k = t.n - 1; k >= 0; k--)
        if (t.p[k] != 0.0) return t.p[k] > 0.0 ? 1 : -1;
    return 0;
}

/* the exact sum rounded (largest component first; reporting only) */
static double xsum_value(const xsum_t* s) {
    double r = 0.0;
    for (int k = s->n - 1; k >= 0; k--) r += s->p[k];
    return r;
}

/* evaluate L_tight (active count, exact loss, violated count) over the pair list in order */
static void eval_pairs(const float* P, int64_t np, const int64_t* pi, const int64_t* pj,
                       const uint8_t* pf, const oc_th* t, int periodic, int64_t* active,
                       xsum_t* loss, int64_t* violated) {
    int64_t a = 0, v = 0;
    loss->n = 0;
    for (int64_t k = 0; k < np; k++) {
        float r[3], dh, e;
        int ol = pf[k] & 1;
        if (tight_pair(P, pi[k], pj[k], ol, t, periodic, r, &dh, &e)) {
            a++;
            xsum_add(loss, (double)e * (double)e);
        }
        float s = r[0] * r[0];
        s = s + r[1] * r[1];
        s = s + r[2] * r[2];
        if ((s <= t->b2) != (ol != 0)) v++;
    }
    *active = a;
    *violated = v;
}

/* pinned fp32 evaluation exported for tests: count, loss and the dense gradient (3n). */
int oc_tight_eval_f32(int64_t n, const float* xh, const float* yh, const float* zh,
                      const uint32_t* gid, int64_t np, const int64_t* pi, const int64_t* pj,
                      const uint8_t* pf, const oc_cfg* c, int64_t* active, double* loss,
                      float* grad) {
    oc_th t;
    int st = oc_thresholds(c, &t);
    if (st) return st;
    float* P = (float*)malloc((size_t)(n > 0 ? n : 1) * 3 * sizeof(float));
    if (!P) return 67;
    for (int64_t i = 0; i < n; i++) { P[3 * i] = xh[i]; P[3 * i + 1] = yh[i]; P[3 * i + 2] = zh[i]; }
    int64_t viol;
    xsum_t xs;
    eval_pairs(P, np, pi, pj, pf, &t, c->periodic, active, &xs, &viol);
    *loss = xsum_value(&xs);
    if (grad) {
        memset(grad, 0, (size_t)n * 3 * sizeof(float));
        for (int64_t k = 0; k < np; k++) {
            float r[3], dh, e;
            int64_t i = pi[k], j = pj[k];
            if (!tight_pair(P, i, j, pf[k] & 1, &t, c->periodic, r, &dh, &e)) continue;
            uint32_t gi = gid ? gid[i] : (uint32_t)i, gj = gid ? gid[j] : (uint32_t)j;
            float gi3[3] = {grad[3 * i], grad[3 * i + 1], grad[3 * i + 2]};
            grad_add(gi3, r, dh, e, gi < gj);
            grad[3 * i] = gi3[0]; grad[3 * i + 1] = gi3[1]; grad[3 * i + 2] = gi3[2];
            float rj[3] = {-r[0], -r[1], -r[2]};
            float gj3[3] = {grad[3 * j], grad[3 * j + 1], grad[3 * j + 2]};
            grad_add(gj3, rj, dh, e, gj < gi);
            grad[3 * j] = gj3[0]; grad[3 * j + 1] = gj3[1]; grad[3 * j + 2] = gj3[2];
        }
    }
    free(P);
    return 0;
}

/* fp64 versions of Eq. (1) and Eq. (3) with the analytic gradient, for the finite-difference
 * and worked-example pins.  Positions as doubles. */
static double mi64(double d, double L, int periodic) {
    if (periodic) {
        if (d > 0.5 * L) d -= L;
        else if (d < -0.5 * L) d += L;
    }
    return d;
}
double oc_loss_eq1_f64(const double* P, int64_t np, const int64_t* pi, const int64_t* pj,
                       const uint8_t* pf, double b, double L, int periodic) {
    double l = 0.0;
    for (int64_t k = 0; k < np; k++) {
        int64_t i = pi[k], j = pj[k];
        double rx = mi64(P[3 * i] - P[3 * j], L, periodic), ry = mi64(P[3 * i + 1] - P[3 * j + 1], L, periodic),
               rz = mi64(P[3 * i + 2] - P[3 * j + 2], L, periodic);
        double d = sqrt(rx * rx + ry * ry + rz * rz);
        if ((pf[k] & 1) && b < d) l += (d - b) * (d - b);           /* broken: d <= b < d_hat */
        if (!(pf[k] & 1) && d <= b) l += (b - d) * (b - d);         /* false:  d_hat <= b < d */
    }
    return l;
}
double oc_tight_f64(const double* P, int64_t np, const int64_t* pi, const int64_t* pj,
                    const uint8_t* pf, double b, double eps_q, double L, int periodic,
                    double* grad /* 3n or NULL, accumulated */) {
    double mu = 2.0 * sqrt(3.0) * eps_q, l = 0.0;
    for (int64_t k = 0; k < np; k++) {
        int64_t i = pi[k], j = pj[k];
        double r[3] = {mi64(P[3 * i] - P[3 * j], L, periodic), mi64(P[3 * i + 1] - P[3 * j + 1], L, periodic),
                       mi64(P[3 * i + 2] - P[3 * j + 2], L, periodic)};
        double d = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]), c, e;
        if (pf[k] & 1) {                      /* d <= b, d_hat > b - mu: (d_hat - b + mu)^2 */
            c = b - mu;
            if (!(d > c)) continue;
        } else {                              /* d > b, d_hat <= b + mu: (b + mu - d_hat)^2 */
            c = b + mu;
            if (!(d <= c)) continue;
        }
        e = d - c;
        l += e * e;
        if (grad && d > 0) {
            for (int q = 0; q < 3; q++) {
                grad[3 * i + q] += 2.0 * e * r[q] / d;
                grad[3 * j + q] -= 2.0 * e * r[q] / d;
            }
        }
    }
    return l;
}

/* ---------------------------------------------------------------------------------------- */
/*
 * O4/O5 -- Alg. 1 lines 4-10 with PGD (§III-B) and Adam,
 * tightened loss (Eq. 3) and box projection onto B(xi') around the ORIGINAL positions:
 *
 *   P_hat <- P_hat^(0)
 *   for t = 1 .. T_max:
 *       if stop(P_hat): break                      (R11: active count == 0; or L_tight<=eps_L)
 *       g <- grad L_tight(P_hat)                   (all gradients from the same state)
 *       P_hat <- P_hat - step(g)                   (Adam, fp32, R9; or vanilla alpha*g)
 *       P_hat <- proj_B(xi')(P_hat)                (every editable coordinate, R8/R24)
 *
 * Editable particles = endpoints of the given pairs; only they move.  Each particle's
 * gradient is summed over its incident pairs in ascending partner gid (R14).
 * Outputs xo,yo,zo for all n particles (non-editable = decompressed input, bit-exact).
 * trace_active/trace_loss (optional, length t_max+1) record each stop check.
 */
int oc_correct(int64_t n, const float* x, const float* y, const float* z, const float* xh,
               const float* yh, const float* zh, const uint32_t* gid, int64_t np,
               const int64_t* pi, const int64_t* pj, const uint8_t* pf, const oc_cfg* c,
               float* xo, float* yo, float* zo, oc_corr_info* info, int64_t* trace_active,
               double* trace_loss, int64_t* trace_violated) {
    oc_th t;
    int st = oc_thresholds(c, &t);
    if (st) return st;
    int per = c->periodic;
    memset(info, 0, sizeof(*info));
    /* input contract: |x_hat - x| <= xi_f per coordinate */
    for (int64_t i = 0; i < n; i++) {
        if (fabs((double)xh[i] - (double)x[i]) > (double)t.xi_f ||
            fabs((double)yh[i] - (double)y[i]) > (double)t.xi_f ||
            fabs((double)zh[i] - (double)z[i]) > (double)t.xi_f)
            return 66;
    }
    size_t n1 = (size_t)(n > 0 ? n : 1);
    float* P = (float*)malloc(n1 * 3 * sizeof(float));
    float* Q = (float*)malloc(n1 * 3 * sizeof(float));
    int64_t* eidx = (int64_t*)malloc(n1 * sizeof(int64_t));
    if (!P || !Q || !eidx) { free(P); free(Q); free(eidx); return 67; }
    for (int64_t i = 0; i < n; i++) {
        P[3 * i] = xh[i]; P[3 * i + 1] = yh[i]; P[3 * i + 2] = zh[i];
        eidx[i] = -1;
    }
    /* editable set E and its incidence rows, sorted by partner gid */
    int64_t ne = 0;
    int64_t* deg = (int64_t*)calloc(n1, sizeof(int64_t));
    int64_t* emap = NULL;
    int64_t* rp = NULL;
    rent_t* rows = NULL;
    float* mom = NULL;
    float* box = NULL;
    if (!deg) { st = 67; goto done; }
    for (int64_t k = 0; k < np; k++) { deg[pi[k]]++; deg[pj[k]]++; }
    for (int64_t i = 0; i < n; i++) if (deg[i] > 0) eidx[i] = ne++;
    emap = (int64_t*)malloc((size_t)(ne > 0 ? ne : 1) * sizeof(int64_t));
    rp = (int64_t*)calloc((size_t)ne + 1, sizeof(int64_t));
    rows = (rent_t*)malloc((size_t)(2 * np > 0 ? 2 * np : 1) * sizeof(rent_t));
    mom = (float*)calloc((size_t)(ne > 0 ? ne : 1) * 6, sizeof(float));
    box = (float*)malloc((size_t)(ne > 0 ? ne : 1) * 6 * sizeof(float));
    if (!emap || !rp || !rows || !mom || !box) { st = 67; goto done; }
    for (int64_t i = 0; i < n; i++) if (eidx[i] >= 0) { emap[eidx[i]] = i; rp[eidx[i] + 1] = deg[i]; }
    for (int64_t e = 0; e < ne; e++) rp[e + 1] += rp[e];
    {
        int64_t* fill = (int64_t*)malloc((size_t)(ne > 0 ? ne : 1) * sizeof(int64_t));
        if (!fill) { st = 67; goto done; }
        for (int64_t e = 0; e < ne; e++) fill[e] = rp[e];
        for (int64_t k = 0; k < np; k++) {
            int64_t i = pi[k], j = pj[k];
            rent_t a = {j, gid ? gid[j] : (uint32_t)j, pf[k] & 1};
            rent_t b = {i, gid ? gid[i] : (uint32_t)i, pf[k] & 1};
            rows[fill[eidx[i]]++] = a;
            rows[fill[eidx[j]]++] = b;
        }
        free(fill);
        for (int64_t e = 0; e < ne; e++)
            qsort(rows + rp[e], (size_t)(rp[e + 1] - rp[e]), sizeof(rent_t), cmp_rent);
    }
    /* projection box B(xi') around the ORIGINAL positions, directed rounding (R8) */
    for (int64_t e = 0; e < ne; e++) {
        int64_t i = emap[e];
        const float o[3] = {x[i], y[i], z[i]};
        for (int q = 0; q < 3; q++) {
            box[6 * e + 2 * q + 0] = ru32_sum((double)o[q], -(double)t.xip_f);
            box[6 * e + 2 * q + 1] = rd32_sum((double)o[q], (double)t.xip_f);
        }
    }
    info->n_editable = ne;
    {
        const float b1 = (float)c->beta1, b2 = (float)c->beta2;
        const float omb1 = (float)(1.0 - c->beta1), omb2 = (float)(1.0 - c->beta2);
        const float alpha = (float)c->alpha, eps = (float)c->eps_adam;
        const float vstep = (float)c->vanilla_step;
        double p1 = 1.0, p2 = 1.0;
        int64_t act, viol;
        xsum_t loss;
        eval_pairs(P, np, pi, pj, pf, &t, per, &act, &loss, &viol);
        info->active0 = act; info->loss0 = xsum_value(&loss); info->violated0 = viol;
        int64_t t_it;
        for (t_it = 1; t_it <= c->t_max; t_it++) {
            if (t_it > 1) eval_pairs(P, np, pi, pj, pf, &t, per, &act, &loss, &viol);
            if (trace_active) trace_active[t_it - 1] = act;
            if (trace_loss) trace_loss[t_it - 1] = xsum_value(&loss);
            if (trace_violated) trace_violated[t_it - 1] = viol;
            /* Alg. 1 line 6 on the exact L_tight (R11, R16) */
            const int loss_le = xsum_cmp(&loss, c->eps_loss) <= 0;
            if (c->stop_mode == 0 && act == 0) break;
            if (c->stop_mode == 1 && loss_le) break;
            if (c->stop_mode == 3 && viol == 0 && loss_le) break;
            p1 = p1 * c->beta1;
            p2 = p2 * c->beta2;
            const float bc1 = (float)(1.0 - p1), bc2 = (float)(1.0 - p2);
            memcpy(Q, P, (size_t)n * 3 * sizeof(float));
            for (int64_t e = 0; e < ne; e++) {
                int64_t i = emap[e];
                uint32_t gi = gid ? gid[i] : (uint32_t)i;
                /* R14: the row's terms in ascending partner gid (an inactive pair's term is 0);
                 * chunks of GC consecutive terms summed left to right from +0; the chunk sums
                 * of each group of GG chunks combined by the adjacent-pairwise tree (zero
                 * padded); group results summed left to right from +0. */
                float g[3] = {0.0f, 0.0f, 0.0f};
                for (int64_t g0 = rp[e]; g0 < rp[e + 1]; g0 += GC * GG) {
                    float cs[GG][3];
                    memset(cs, 0, sizeof(cs));
                    for (int j = 0; j < GG; j++)
                        for (int q = 0; q < GC; q++) {
                            const int64_t k = g0 + (int64_t)GC * j + q;
                            if (k >= rp[e + 1]) break;
                            float r[3], dh, ee;
                            if (tight_pair(P, i, rows[k].j, rows[k].olink, &t, per, r, &dh, &ee))
                                grad_add(cs[j], r, dh, ee, gi < rows[k].gj);
                        }
                    for (int off = 1; off < GG; off *= 2)
                        for (int l = 0; l < GG; l += 2 * off)
                            for (int q = 0; q < 3; q++) cs[l][q] = cs[l][q] + cs[l + off][q];
                    for (int q = 0; q < 3; q++) g[q] = g[q] + cs[0][q];
                }
                for (int q = 0; q < 3; q++) {
                    float xq = P[3 * i + q];
                    if (c->optimizer == 0) {
                        float* m = &mom[6 * e + q];
                        float* v = &mom[6 * e + 3 + q];
                        *m = b1 * *m + omb1 * g[q];
                        *v = b2 * *v + omb2 * (g[q] * g[q]);
                        float mh = *m / bc1;
                        float vh = *v / bc2;
                        float den = sqrtf(vh) + eps;
                        float step = alpha * (mh / den);
                        xq = xq - step;
                    } else {
                        xq = xq - vstep * g[q];
                    }
                    float lo = box[6 * e + 2 * q], hi = box[6 * e + 2 * q + 1];
                    if (xq < lo) xq = lo;
                    if (xq > hi) xq = hi;
                    Q[3 * i + q] = xq;
                }
            }
            float* tmp = P; P = Q; Q = tmp;
            info->iterations++;
        }
        eval_pairs(P, np, pi, pj, pf, &t, per, &act, &loss, &viol);
        if (trace_active) trace_active[info->iterations] = act;
        if (trace_loss) trace_loss[info->iterations] = xsum_value(&loss);
        if (trace_violated) trace_violated[info->iterations] = viol;
        info->active_final = act;
        info->loss_final = xsum_value(&loss);
        info->violated_final = viol;
        const int loss_le = xsum_cmp(&loss, c->eps_loss) <= 0;
        if (c->stop_mode == 1) info->converged = loss_le;
        else if (c->stop_mode == 3) info->converged = viol == 0 && loss_le;
        else info->converged = act == 0;
    }
    for (int64_t i = 0; i < n; i++) { xo[i] = P[3 * i]; yo[i] = P[3 * i + 1]; zo[i] = P[3 * i + 2]; }
done:
    free(P); free(Q); free(eidx); free(deg); free(emap); free(rp); free(rows); free(mom); free(box);
    return st;
}

/* ---------------------------------------------------------------------------------------------
 * f1 -- edit log: compaction + m-bit quantisation (Alg. 1 lines 11-13; §III-B
 * "Compaction, quantization, and lossless compression") and reconstruction (§III-B
 * "Reconstruction of the edited decompressed data").  Readings R29-R31:
 *   R29  coordinate k = 3 i + a (particle i in input order, axis a = x,y,z); flags bit k is bit
 *        (k mod 8) of byte k/8 (LSB first); ceil(3n/8) bytes; bit set iff fl32 corrected !=
 *        fl32 decompressed (Delta != 0, "bitmask of non-zero entries in Delta").
 *   R30  Delta_k = (double)corrected - (double)decompressed (exact in fp64); uniform quantiser
 *        on the lattice s = xi_f 2^(1-m) (2^(m+1)+1 levels over [-2 xi, 2 xi], "uniform
 *        quantization into 2^m intervals" per xi of half-width): q = rint(Delta / s) in fp64
 *        (round half to even), |Delta| <= 2 xi_f required (else 66, CC_E_BOUND).  Max
 *        reconstruction error s/2 = xi 2^-m = xi - xi' < eps_q.
 *   R31  reconstruction: x_rec = fl32((double)x_hat0 + (double)q * s) for a flagged coordinate,
 *        x_hat0 unchanged otherwise ("element-wise addition ... to the initial output").
 *   R32  bound-safe index: xi' + s/2 = xi leaves no room for the fp32 rounding of x_rec where
 *        ulp(x) < s, so the encoder (which holds P, Alg. 1 REQUIRE) checks the decoder's value
 *        and, while |x_rec - x| > xi_f, moves q one lattice step toward x (at most 8 steps,
 *        else 66).  |x_rec - x| <= xi_f then holds exactly (Eq. 2).
 * The Huffman+ZSTD stage is a lossless host stage, not part of this oracle.
 * ------------------------------------------------------------------------------------------- */
static double oc_edit_step(const oc_cfg* c) {
    return ldexp((double)(float)c->xi, 1 - c->m);
}

/* Returns 0, 64 (arguments), 66 (|Delta| > 2 xi_f) or 67 (more edits than cap; *n_edits set). */
int oc_edit_encode(int64_t n, const float* x, const float* y, const float* z,
                   const float* xh0, const float* yh0, const float* zh0,
                   const float* xc, const float* yc, const float* zc, const oc_cfg* c,
                   uint8_t* flags, int64_t* q, int64_t cap, int64_t* n_edits) {
    if (n < 0 || !c || !n_edits || c->m < 2 || c->m > 40 || !(c->xi > 0)) return 64;
    const double s = oc_edit_step(c), xi_f = (double)(float)c->xi, lim = 2.0 * xi_f;
    const float* o[3] = {x, y, z};
    const float* h[3] = {xh0, yh0, zh0};
    const float* p[3] = {xc, yc, zc};
    memset(flags, 0, (size_t)((3 * n + 7) / 8));
    int64_t ne = 0;
    for (int64_t i = 0; i < n; i++) {
        for (int a = 0; a < 3; a++) {
            int64_t k = 3 * i + a;
            if (p[a][i] == h[a][i]) continue;                 /* Delta = 0: no flag */
            double delta = (double)p[a][i] - (double)h[a][i];  /* exact (R30) */
            if (fabs(delta) > lim) return 66;
            flags[k / 8] |= (uint8_t)(1u << (k % 8));
            int64_t qi = (int64_t)rint(delta / s);
            for (int step = 0;; step++) {                       /* R32 */
                float r = (float)((double)h[a][i] + (double)qi * s);
                double dev = (double)r - (double)o[a][i];
                if (fabs(dev) <= xi_f) break;
                if (step == 8) return 66;
                qi += dev > 0 ? -1 : 1;
            }
            if (ne < cap) q[ne] = qi;
            ne++;
        }
    }
    *n_edits = ne;
    return ne > cap ? 67 : 0;
}

/* x_rec (R31).  Returns 0, 64 (arguments) or 65 (popcount(flags) != n_edits). */
int oc_edit_decode(int64_t n, const float* xh0, const float* yh0, const float* zh0,
                   const uint8_t* flags, const int64_t* q, int64_t n_edits, const oc_cfg* c,
                   float* xr, float* yr, float* zr) {
    if (n < 0 || !c || c->m < 2 || c->m > 40 || !(c->xi > 0)) return 64;
    const double s = oc_edit_step(c);
    const float* h[3] = {xh0, yh0, zh0};
    float* r[3] = {xr, yr, zr};
    int64_t e = 0;
    for (int64_t i = 0; i < n; i++) {
        for (int a = 0; a < 3; a++) {
            int64_t k = 3 * i + a;
            if (flags[k / 8] >> (k % 8) & 1u) {
                if (e >= n_edits) return 65;
                r[a][i] = (float)((double)h[a][i] + (double)q[e] * s);
                e++;
            } else {
                r[a][i] = h[a][i];
            }
        }
    }
    return e == n_edits ? 0 : 65;
}

/* ---------------------------------------------------------------------------------------------
 * f1 -- m-bit packing of the quantised edits (Alg. 1 line 13, "edits <- non-zero values of
 * Delta, quantized to m bits"; reading R33).  An edit index q satisfies
 * |q| <= 2^m (|Delta| <= 2 xi_f on the lattice s = xi_f 2^(1-m), R30), so it is stored as an
 * (m+2)-bit two's-complement field; field e occupies bits [e (m+2), (e+1)(m+2)) of a stream of
 * 32-bit words, bit b of the stream = bit (b mod 32) of word b / 32 (LSB first).  Written bit by
 * bit on purpose (plain and obviously correct).  Returns 0, or 64 for |q| > 2^m / bad m.
 * ------------------------------------------------------------------------------------------- */
int64_t oc_edit_packed_words(int64_t n_edits, int m) {
    return (n_edits * (int64_t)(m + 2) + 31) / 32;
}

int oc_edit_pack(const int64_t* q, int64_t n_edits, int m, uint32_t* words) {
    if (m < 2 || m > 40 || n_edits < 0) return 64;
    const int w = m + 2;
    const int64_t nw = oc_edit_packed_words(n_edits, m);
    for (int64_t k = 0; k < nw; k++) words[k] = 0u;
    const int64_t lim = (int64_t)1 << m;
    for (int64_t e = 0; e < n_edits; e++) {
        if (q[e] > lim || q[e] < -lim) return 64;
        const uint64_t u = (uint64_t)q[e];  /* two's complement, low w bits kept */
        for (int b = 0; b < w; b++) {
            const int64_t bit = e * w + b;
            if ((u >> b) & 1u) words[bit / 32] |= 1u << (bit % 32);
        }
    }
    return 0;
}

int oc_edit_unpack(const uint32_t* words, int64_t n_edits, int m, int64_t* q) {
    if (m < 2 || m > 40 || n_edits < 0) return 64;
    const int w = m + 2;
    for (int64_t e = 0; e < n_edits; e++) {
        uint64_t u = 0;
        for (int b = 0; b < w; b++) {
            const int64_t bit = e * w + b;
            u |= (uint64_t)((words[bit / 32] >> (bit % 32)) & 1u) << b;
        }
        if ((u >> (w - 1)) & 1u) u |= ~(uint64_t)0 << w;  /* sign extension */
        q[e] = (int64_t)u;
    }
    return 0;
}
