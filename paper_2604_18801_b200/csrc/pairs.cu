// pairs.cu -- K2, vulnerable-pair search (S2) and CSR rows of the editable set (S3).
//
// Paper: §III-A P:396 (vulnerable pairs: original distance in (b - 2 sqrt3 xi, b + 2 sqrt3 xi];
// editable particles = their endpoints), Alg. 1 line 3 P:421, §III-B P:442 (cell side
// w >= b + 2 sqrt3 xi; same and adjacent cells), §III-C P:463 (two-pass count/fill, direct-address
// map of editable particles), §IV-C P:178.
//
// B200 form: one thread per particle in cell-sorted order scans the 27-cell neighbourhood
// (x-adjacent cells merged into one contiguous slot range, so 9 ranges), reading float4
// records that neighbouring threads share through L1/L2.  Pass 1 counts each particle's band
// partners (the row length, no atomics); an exclusive scan gives row offsets AND the editable
// ranks (the paper's direct-address map, without atomicCAS); pass 2 writes each row's u32
// entries (partner editable index | partner-gid-above bit | original-link bit).  Rows are then
// sorted by partner gid so the PGD gradient sum has one defined order on any grid / rank (R14).
// Each unordered pair is tested from both endpoints: both see the identical pinned fp32 d2.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "cc_internal.cuh"

namespace cc {
namespace {

constexpr int PAIR_THREADS = 256;

// the count sweep's per-candidate work (shared by the two count kernels): band pair -> degrees;
// stable link -> the stable forest; near shell -> the near list
// mode bits: CM_DEG = band pairs -> degrees (S2, cc_find_vulnerable); CM_FOREST = stable links ->
// the stable forest and the near-shell list (S6 data, built at the first FoF labelling)
constexpr int CM_DEG = 1, CM_FOREST = 2;

struct CountCtx {
    int mode;
    const float4* __restrict__ dec4;
    const Th& t;  // the kernel's parameter (no copy)
    uint32_t n_own;
    bool multi, ghost, inner;
    float lo2s, hi2s;
    uint32_t s;
    float4 p;
    uint32_t cnt, rs, ntest;
    uint32_t* __restrict__ deg;
    uint32_t* __restrict__ par_base;
    uint2* __restrict__ near;
    unsigned long long* __restrict__ near_n;
    unsigned long long near_cap;
    __device__ __forceinline__ CountCtx(int mode_, int64_t n, const float4* dec4_, const Grid& g, const Th& t_,
                                        uint32_t n_own_, uint32_t* deg_, uint32_t* par_base_, uint2* near_,
                                        unsigned long long* near_n_, unsigned long long near_cap_, uint32_t s_,
                                        const float4& p_)
        : mode(mode_), dec4(dec4_), t(t_), n_own(n_own_), s(s_), p(p_), cnt(0), rs(s_), ntest(0), deg(deg_), par_base(par_base_),
          near(near_), near_n(near_n_), near_cap(near_cap_) {
        multi = n_own < (uint32_t)n;
        ghost = multi && __float_as_uint(dec4[s].w) >= n_own;
        inner = interior(p.x, p.y, p.z, g, t);
        lo2s = inner ? t.lo2s_i : t.lo2s_w;
        hi2s = inner ? t.hi2s_i : t.hi2s_w;
    }
    __device__ __forceinline__ void operator()(uint32_t j, const float4& q) {
        ntest++;
        const float d2 = inner ? dist2_nw(p, q) : dist2(p, q, t);
        if (t.lo2 < d2 && d2 <= t.hi2) {
            if (!(mode & CM_DEG)) return;
            const bool gj = multi && __float_as_uint(dec4[j].w) >= n_own;
            if (!ghost) {
                cnt++;
                if (gj) atomicOr(&deg[j], 0x80000000u);
                else atomicAdd(&deg[j], 1u);
            } else if (!gj) {
                atomicAdd(&deg[j], 1u);
                atomicOr(&deg[s], 0x80000000u);
            }
        } else if (!(mode & CM_FOREST)) {
            return;
        } else if (d2 <= lo2s) {
            // a stable FoF link: provably linked in the original, decompressed and corrected
            // positions alike (Th::lo2s, fof.cu)
            uf_link(par_base, s, j, rs);
        } else if (d2 <= hi2s) {
            // near shell (lo2s, lo2] or (hi2, hi2s]: not vulnerable, but fp32 rounding could flip
            // its link in other positions -- listed, re-tested by every FoF labelling
            const unsigned long long qn = atomicAdd(near_n, 1ull);
            if (qn < near_cap) near[qn] = make_uint2(s, j | (d2 <= t.b2 ? 0x80000000u : 0u));
        }
    }
};

// pass 1 (each unordered pair once, for_each_pair_forward): deg[] = band partners per slot
// (atomics for the far endpoint), ghost endpoints of band pairs with an owned partner get bit 31
// of their deg word (multi-GPU: they become ghost editables); stable links (d2 <= lo2s) are
// united into the stable FoF forest in the same sweep.  (General grid; k_pairs_count_tiled below
// is the default-grid form.)
__global__ void __launch_bounds__(PAIR_THREADS)
k_pairs_count(int mode, int64_t n, const float4* __restrict__ orig4, const float4* __restrict__ dec4,
              const uint32_t* __restrict__ xk, const uint32_t* __restrict__ cs, Grid g, Th t, double r, uint32_t n_own,
              uint32_t* __restrict__ deg, uint32_t* __restrict__ par_base, uint2* __restrict__ near,
              unsigned long long* __restrict__ near_n, unsigned long long near_cap, unsigned long long* __restrict__ tests) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const float4 p = orig4[s];
    double u;
    int cx, cy, cz;
    cell_of(p.x, p.y, p.z, g, u, cx, cy, cz);
    CountCtx k(mode, n, dec4, g, t, n_own, deg, par_base, near, near_n, near_cap, (uint32_t)s, p);
    auto test = [&](uint32_t j) { k(j, orig4[j]); };
    for_each_pair_forward(g, cs, xk, (uint32_t)s, u, cy, cz, r, t.periodic != 0, test);
    if (k.cnt) atomicAdd(&deg[s], k.cnt);
    warp_count(tests, k.ntest);
}

// ---- the default grid, warp-flattened (the default K2 count when cells are rows): a warp takes
// 32 consecutive home slots; each lane finds its candidate slot RANGES in the 5 rows of its half
// shell (x-window key bounds once, a binary search per row, a key scan to the window end), the
// warp sums the range lengths, and then every lane tests one (home, candidate) pair per step
// across the whole warp's concatenated candidate list.  The per-lane sweep left 9 of 32 lanes
// active on average (ncu r02q: candidate loops of different lengths and the stable-forest
// unions of halo cores serialised on single lanes); here tests and unions are spread over all
// lanes.  Results are those of k_pairs_count (the same pair set; union order does not change
// the forest's components; degrees are sums).
constexpr int CW_NR = 10;       // ranges per home particle: own row (forward, wrap part), 4 rows x 2 windows
constexpr int CW_WARPS = PAIR_THREADS / 32;

template <int MODE>
__global__ void __launch_bounds__(PAIR_THREADS)
k_pairs_count_warp(int64_t n, const float4* __restrict__ orig4, const float4* __restrict__ dec4,
                   const uint32_t* __restrict__ xk, const uint32_t* __restrict__ cs, Grid g, Th t, double r,
                   uint32_t n_own, uint32_t* __restrict__ deg, uint32_t* __restrict__ par_base,
                   uint2* __restrict__ near, unsigned long long* __restrict__ near_n, unsigned long long near_cap,
                   unsigned long long* __restrict__ tests) {
    __shared__ uint32_t r_start[CW_WARPS][CW_NR][32];  // range starts, [range][lane]
    __shared__ uint32_t r_cum[CW_WARPS][CW_NR][32];      // exclusive running counts, [range][lane]
    __shared__ uint8_t l_nr[CW_WARPS][32];               // ranges per home
    __shared__ uint32_t l_ex[CW_WARPS][33];              // warp-exclusive pair offsets per lane
    __shared__ float4 l_p[CW_WARPS][32];
    __shared__ uint8_t l_fl[CW_WARPS][32];               // bit 0 ghost, bit 1 interior
    __shared__ uint32_t l_rs[CW_WARPS][32];              // per home: a cached stable-forest ancestor
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t s = ((int64_t)blockIdx.x * CW_WARPS + w) * 32 + lane;
    const bool multi = n_own < (uint32_t)n;
    uint32_t nr = 0u, tot = 0u;
    auto add_range = [&](uint32_t a, uint32_t b) {
        if (b > a) {
            r_start[w][nr][lane] = a;
            r_cum[w][nr][lane] = tot;
            tot += b - a;
            nr++;
        }
    };
    if (s < n) {
        const float4 p = orig4[s];
        double u;
        int cx, cy, cz;
        cell_of(p.x, p.y, p.z, g, u, cx, cy, cz);
        const bool ghost = multi && __float_as_uint(dec4[s].w) >= n_own;
        const bool inner = interior(p.x, p.y, p.z, g, t);
        l_p[w][lane] = p;
        l_fl[w][lane] = (uint8_t)((ghost ? 1 : 0) | (inner ? 2 : 0));
        double a = u - r, b = u + r, a1 = 0.0, b1 = -1.0;
        bool up = false;
        if (g.xwrap) {
            if (a < 0.0) {
                a1 = a + g.L;
                b1 = g.L;
                a = 0.0;
            } else if (b >= g.L) {
                a1 = 0.0;
                b1 = b - g.L;
                b = g.L;
                up = true;
            }
        } else {
            if (a < 0.0) a = 0.0;
            if (b > g.ext_x) b = g.ext_x;
        }
        const bool two = b1 >= a1;
        const uint32_t klo0 = key_lo(a, g), khi0 = key_hi(b, g);
        const uint32_t klo1 = two ? key_lo(a1, g) : 0u, khi1 = two ? key_hi(b1, g) : 0u;
        const bool periodic = t.periodic != 0;
        {   // own row: forward in slot (= x) order, then the part above the seam at the row start
            const int64_t row = (int64_t)cz * g.ny + cy;
            const uint32_t r0 = cs[row], r1 = cs[row + 1];
            uint32_t j = (uint32_t)s + 1u;
            while (j < r1 && xk[j] <= khi0) j++;
            add_range((uint32_t)s + 1u, j);
            if (two && up) {
                uint32_t j2 = r0;
                while (j2 < (uint32_t)s && xk[j2] <= khi1) j2++;
                add_range(r0, j2);
            }
        }
        const int rows_dz[4] = {0, 1, 1, 1};
        const int rows_dy[4] = {1, -1, 0, 1};
#pragma unroll
        for (int k = 0; k < 4; k++) {
            int zz = cz + rows_dz[k], yy = cy + rows_dy[k];
            if (periodic) {
                zz = wrapi(zz, g.nz);
                yy = wrapi(yy, g.ny);
            } else if (zz < 0 || zz >= g.nz || yy < 0 || yy >= g.ny) {
                continue;
            }
            const int64_t row = (int64_t)zz * g.ny + yy;
            const uint32_t j0 = cs[row], j1 = cs[row + 1];
            uint32_t lo = lower_bound_key(xk, j0, j1, klo0), hi = lo;
            while (hi < j1 && xk[hi] <= khi0) hi++;
            add_range(lo, hi);
            if (two) {
                lo = lower_bound_key(xk, j0, j1, klo1);
                hi = lo;
                while (hi < j1 && xk[hi] <= khi1) hi++;
                add_range(lo, hi);
            }
        }
    }
    l_nr[w][lane] = (uint8_t)nr;
    l_rs[w][lane] = (uint32_t)s;
    // warp-exclusive offsets of the lanes' candidate lists
    uint32_t inc = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    l_ex[w][lane] = inc - tot;
    const uint32_t T = __shfl_sync(0xffffffffu, inc, 31);
    if (lane == 31) l_ex[w][32] = T;
    __syncwarp();
    // the flattened tests: pair q = (home lane o, its candidate q - ex[o])
    for (uint32_t base = 0; base < T; base += 32u) {
        const uint32_t q = base + (uint32_t)lane;
        if (q < T) {
            int o = 0;  // largest o with ex[o] <= q
#pragma unroll
            for (int st = 16; st > 0; st >>= 1)
                if (l_ex[w][o + st] <= q) o += st;
            const uint32_t qo = q - l_ex[w][o];
            int k = 0;  // the range: largest k with cum[k] <= qo
            const int nro = l_nr[w][o];
            while (k + 1 < nro && r_cum[w][k + 1][o] <= qo) k++;
            const uint32_t j = r_start[w][k][o] + (qo - r_cum[w][k][o]);
            const uint32_t so = (uint32_t)(s - lane + o);
            const float4 pp = l_p[w][o];
            const uint8_t fl = l_fl[w][o];
            const bool ghost = fl & 1u, inner = (fl & 2u) != 0;
            const float4 qq = orig4[j];
            const float d2 = inner ? dist2_nw(pp, qq) : dist2(pp, qq, t);
            if (t.lo2 < d2 && d2 <= t.hi2) {
                if (!(MODE & CM_DEG)) continue;
                const bool gj = multi && __float_as_uint(dec4[j].w) >= n_own;
                if (!ghost) {
                    atomicAdd(&deg[so], 1u);
                    if (gj) atomicOr(&deg[j], 0x80000000u);
                    else atomicAdd(&deg[j], 1u);
                } else if (!gj) {
                    atomicAdd(&deg[j], 1u);
                    atomicOr(&deg[so], 0x80000000u);
                }
            } else if (!(MODE & CM_FOREST)) {
                continue;
            } else if (d2 <= (inner ? t.lo2s_i : t.lo2s_w)) {
                // a stable FoF link (see CountCtx).  The home's cached ancestor is shared by the
                // lanes testing its candidates: any value once an ancestor of the home stays
                // valid for uf_link's filter (sets only merge), so the benign races are harmless
                uint32_t rs = l_rs[w][o];
                const uint32_t rs0 = rs;
                uf_link(par_base, so, j, rs);
                if (rs != rs0) l_rs[w][o] = rs;
            } else if (d2 <= (inner ? t.hi2s_i : t.hi2s_w)) {
                const unsigned long long qn = atomicAdd(near_n, 1ull);
                if (qn < near_cap) near[qn] = make_uint2(so, j | (d2 <= t.b2 ? 0x80000000u : 0u));
            }
        }
    }
    if (lane == 0 && T) atomicAdd(tests, (unsigned long long)T);
}

// ---- the default grid (cells = whole rows, periodic or not, >= 3 rows per axis): a block takes
// a strip of TROWS consecutive rows of one z-row and stages in shared memory every row the strip's
// half-shell visits -- rows y0..y0+TROWS of z-row z and y0-1..y0+TROWS of z-row z+1, contiguous
// slot ranges loaded coalesced -- then each thread searches its home particle's windows with
// binary searches and candidate reads in shared memory (the north_star's staged home cell).  The
// per-particle global form is latency-bound on dependent window loads (ncu: ISETP stalls on the
// binary-search loads).  A strip whose rows exceed the staging capacity (dense halo cores) runs
// the global form for its home particles.
constexpr int TROWS_MAX = 16;
constexpr int TCAP = 2048;
constexpr int TDIR = 2 * TROWS_MAX + 3;

struct RowDir {
    uint32_t g0;  // global slot of the row's first particle
    uint32_t n;   // particles (0: row outside a non-periodic domain)
    uint32_t s0;  // its first staged index
};

template <class F>
__device__ __forceinline__ void scan_staged(const uint32_t* sxk, const float4* so4, const RowDir& d, uint32_t klo,
                                            uint32_t khi, F& f) {
    uint32_t lo = d.s0, hi = d.s0 + d.n;
    while (lo < hi) {  // first staged index with key >= klo
        const uint32_t m = (lo + hi) >> 1;
        if (sxk[m] < klo) lo = m + 1;
        else hi = m;
    }
    for (uint32_t k = lo; k < d.s0 + d.n; k++) {
        if (sxk[k] > khi) break;
        f(d.g0 + (k - d.s0), so4[k]);
    }
}

__global__ void __launch_bounds__(PAIR_THREADS)
k_pairs_count_tiled(int64_t n, const float4* __restrict__ orig4, const float4* __restrict__ dec4,
                    const uint32_t* __restrict__ xk, const uint32_t* __restrict__ cs, Grid g, Th t, double r,
                    uint32_t n_own, uint32_t* __restrict__ deg, uint32_t* __restrict__ par_base,
                    uint2* __restrict__ near, unsigned long long* __restrict__ near_n, unsigned long long near_cap,
                    unsigned long long* __restrict__ tests, int64_t ntiles, int tiles_y, int trows) {
    __shared__ float4 so4[TCAP];
    __shared__ uint32_t sxk[TCAP];
    __shared__ RowDir dir[TDIR];
    __shared__ uint32_t total_sh;
    const bool periodic = t.periodic != 0;
    unsigned ntest = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int z = (int)(tile / tiles_y), y0 = (int)(tile % tiles_y) * trows;
        const int ky = min(trows, g.ny - y0);
        const int nd = 2 * ky + 3;  // dir: [0, ky] z-row z, rows y0..y0+ky; [ky+1, 2ky+2] z-row z+1, y0-1..y0+ky
        if (threadIdx.x < nd) {
            const int idx = threadIdx.x;
            int zz, yy;
            bool use = true;
            if (idx <= ky) {
                zz = z;
                yy = y0 + idx;
            } else {
                zz = z + 1;
                yy = y0 - 1 + (idx - ky - 1);
            }
            if (periodic) {
                zz = wrapi(zz, g.nz);
                yy = wrapi(yy, g.ny);
            } else if (zz < 0 || zz >= g.nz || yy < 0 || yy >= g.ny) {
                use = false;
            }
            RowDir d;
            d.g0 = 0u;
            d.n = 0u;
            if (use) {
                const int64_t row = (int64_t)zz * g.ny + yy;
                d.g0 = cs[row];
                d.n = cs[row + 1] - d.g0;
            }
            dir[idx] = d;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t off = 0;
            for (int i = 0; i < nd; i++) {
                dir[i].s0 = off;
                off += dir[i].n;
            }
            total_sh = off;
        }
        __syncthreads();
        const uint32_t total = total_sh;
        const uint32_t h0 = dir[0].g0;
        const uint32_t h1 = cs[(int64_t)z * g.ny + y0 + ky];  // home rows: contiguous slots
        if (total > (uint32_t)TCAP) {
            // crowded strip: the global per-particle form for its home particles
            for (uint32_t s = h0 + threadIdx.x; s < h1; s += blockDim.x) {
                const float4 p = orig4[s];
                double u;
                int cx, cy, cz;
                cell_of(p.x, p.y, p.z, g, u, cx, cy, cz);
                CountCtx k(CM_DEG | CM_FOREST, n, dec4, g, t, n_own, deg, par_base, near, near_n, near_cap, s, p);
                auto test = [&](uint32_t j) { k(j, orig4[j]); };
                for_each_pair_forward(g, cs, xk, s, u, cy, cz, r, periodic, test);
                if (k.cnt) atomicAdd(&deg[s], k.cnt);
                ntest += k.ntest;
            }
            __syncthreads();
            continue;
        }
        // stage the rows (each a contiguous slot range; a warp per row)
        for (int i = threadIdx.x >> 5; i < nd; i += blockDim.x >> 5) {
            const RowDir d = dir[i];
            for (uint32_t q = threadIdx.x & 31u; q < d.n; q += 32u) {
                so4[d.s0 + q] = orig4[d.g0 + q];
                sxk[d.s0 + q] = xk[d.g0 + q];
            }
        }
        __syncthreads();
        for (uint32_t s = h0 + threadIdx.x; s < h1; s += blockDim.x) {
            // home row of s: the dir entry whose slot range holds s
            int hr = 0;
            while (hr + 1 < ky && s >= dir[hr + 1].g0) hr++;
            const RowDir hd = dir[hr];
            const uint32_t si = hd.s0 + (s - hd.g0);  // staged index of s
            const float4 p = so4[si];
            const double u = local_u((double)p.x, g);
            CountCtx k(CM_DEG | CM_FOREST, n, dec4, g, t, n_own, deg, par_base, near, near_n, near_cap, s, p);
            // x-window key bounds, once for all rows (as for_each_pair_forward)
            double a = u - r, b = u + r, a1 = 0.0, b1 = -1.0;
            bool up = false;
            if (g.xwrap) {
                if (a < 0.0) {
                    a1 = a + g.L;
                    b1 = g.L;
                    a = 0.0;
                } else if (b >= g.L) {
                    a1 = 0.0;
                    b1 = b - g.L;
                    b = g.L;
                    up = true;
                }
            } else {
                if (a < 0.0) a = 0.0;
                if (b > g.ext_x) b = g.ext_x;
            }
            const bool two = b1 >= a1;
            const uint32_t klo0 = key_lo(a, g), khi0 = key_hi(b, g);
            const uint32_t klo1 = two ? key_lo(a1, g) : 0u, khi1 = two ? key_hi(b1, g) : 0u;
            // own row: forward in slot (= x) order, then the part above the seam at the row start
            for (uint32_t q = si + 1; q < hd.s0 + hd.n; q++) {
                if (sxk[q] > khi0) break;
                k(hd.g0 + (q - hd.s0), so4[q]);
            }
            if (two && up)
                for (uint32_t q = hd.s0; q < si; q++) {
                    if (sxk[q] > khi1) break;
                    k(hd.g0 + (q - hd.s0), so4[q]);
                }
            // (z, y+1), (z+1, y-1), (z+1, y), (z+1, y+1)
#pragma unroll 1
            for (int q = 0; q < 4; q++) {
                const RowDir d = dir[q == 0 ? hr + 1 : ky + q + hr];
                if (d.n == 0u) continue;
                scan_staged(sxk, so4, d, klo0, khi0, k);
                if (two) scan_staged(sxk, so4, d, klo1, khi1, k);
            }
            if (k.cnt) atomicAdd(&deg[s], k.cnt);
            ntest += k.ntest;
        }
        __syncthreads();
    }
    warp_count(tests, ntest);
}

// pass 2 (each unordered pair once again): both entries of every band pair, placed by a
// per-row cursor (the order inside a row is fixed afterwards by the gid sort).  One thread per
// EDITABLE particle (slotE; a band pair has two editable endpoints, so the forward search from
// editables alone finds every pair): all lanes busy, and the class-major numbering gives a
// warp neighbours of similar row length.
__global__ void __launch_bounds__(PAIR_THREADS)
k_pairs_fill(uint32_t e_all, const uint32_t* __restrict__ slotE, const float4* __restrict__ orig4,
             const uint32_t* __restrict__ xk, const uint32_t* __restrict__ cs, Grid g, Th t, double r,
             const uint32_t* __restrict__ eidx, uint32_t e_own, const unsigned long long* __restrict__ rowptr,
             uint32_t* __restrict__ cur, uint32_t* __restrict__ rows, unsigned long long* __restrict__ tests) {
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= e_all) return;
    unsigned ntest = 0;
    const uint32_t s = slotE[e];
    const float4 p = orig4[s];
    const uint32_t gp = __float_as_uint(p.w);
    const uint32_t es = e;
    double u;
    int cx, cy, cz;
    cell_of(p.x, p.y, p.z, g, u, cx, cy, cz);
    const bool inner = interior(p.x, p.y, p.z, g, t);
    auto emit = [&](uint32_t j) {
        ntest++;
        const float4 q = orig4[j];
        const float d2 = inner ? dist2_nw(p, q) : dist2(p, q, t);
        if (t.lo2 < d2 && d2 <= t.hi2) {
            const uint32_t ej = eidx[j], gq = __float_as_uint(q.w);
            const uint32_t ol = d2 <= t.b2 ? ENT_OLINK : 0u;
            if (es < e_own) rows[rowptr[es] + atomicAdd(&cur[es], 1u)] = ej | (gq > gp ? ENT_UPPER : 0u) | ol;
            if (ej < e_own) rows[rowptr[ej] + atomicAdd(&cur[ej], 1u)] = es | (gp > gq ? ENT_UPPER : 0u) | ol;
        }
    };
    for_each_pair_forward(g, cs, xk, (uint32_t)s, u, cy, cz, r, t.periodic != 0, emit);
    warp_count(tests, ntest);
}

// compaction: editable e -> slot, row start, original and starting position
__global__ void k_rowptr_tail(unsigned long long* rowptr, uint32_t e_all, unsigned long long nent) {
    rowptr[e_all] = nent;
}

constexpr int LONG_SORT_MAX = 4096;  // block bitonic capacity (entries)

__device__ __forceinline__ unsigned long long row_key(uint32_t ent, const float4* __restrict__ posA) {
    return ((unsigned long long)__float_as_uint(posA[ent & ENT_IDX].w) << 32) | ent;
}

// sort each row by partner gid (R14's summation order).  The key (partner gid << 32 | entry) is
// unique and carries the entry, so a sort of keys alone suffices.  Rows of classes 0-2 (<= 4,
// <= 16, <= 32 entries): a group of W lanes per row, one key per lane, a W-wide bitonic network
// of shuffles; class 3: k_sort_wide (<= 512) and the block kernel beyond.
template <int W>
__device__ __forceinline__ unsigned long long group_sort(unsigned long long k, int gl) {
#pragma unroll
    for (int kk = 2; kk <= W; kk <<= 1) {
#pragma unroll
        for (int j = kk >> 1; j > 0; j >>= 1) {
            const unsigned long long pk = __shfl_xor_sync(0xffffffffu, k, j);
            const bool up = (gl & kk) == 0;
            const bool lower = (gl & j) == 0;
            if (lower ? ((k > pk) == up) : ((k < pk) == up)) k = pk;
        }
    }
    return k;
}

template <int W>
__global__ void __launch_bounds__(PAIR_THREADS)
k_sort_group(uint32_t e_lo, uint32_t e_hi, const unsigned long long* __restrict__ rowptr,
             const float4* __restrict__ posA, uint32_t* __restrict__ rows) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t e = e_lo + t / W;
    const int gl = (int)(t % W);
    int len = 0;
    unsigned long long a = 0ull;
    if (e < e_hi) {
        a = rowptr[e];
        len = (int)(rowptr[e + 1] - a);
    }
    unsigned long long k = gl < len ? row_key(rows[a + gl], posA) : ~0ull;
    k = group_sort<W>(k, gl);  // every lane takes part (the shuffles span the warp)
    if (len > 1 && gl < len) rows[a + gl] = (uint32_t)k;
}

// class-3 rows of 33..512 entries: one warp per row; <= 64 two keys per lane (register network),
// longer ones a bitonic sort in the warp's slice of shared memory (__syncwarp steps)
constexpr int SORT_WIDE = 512;
constexpr int SW_WARPS = 8;

__global__ void __launch_bounds__(32 * SW_WARPS)
k_sort_wide(uint32_t e_lo, uint32_t e_hi, const unsigned long long* __restrict__ rowptr,
            const float4* __restrict__ posA, uint32_t* __restrict__ rows) {
    __shared__ unsigned long long shk[SW_WARPS][SORT_WIDE];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned long long* sk = shk[w];
    const uint32_t nw = gridDim.x * SW_WARPS;
    for (uint32_t e = e_lo + blockIdx.x * SW_WARPS + w; e < e_hi; e += nw) {
        const unsigned long long a = rowptr[e];
        const int len = (int)(rowptr[e + 1] - a);
        if (len > SORT_WIDE) continue;  // the block kernel's
        if (len <= 64) {
            unsigned long long k0 = lane < len ? row_key(rows[a + lane], posA) : ~0ull;
            unsigned long long k1 = lane + 32 < len ? row_key(rows[a + lane + 32], posA) : ~0ull;
            for (int kk = 2; kk <= 64; kk <<= 1) {
                for (int j = kk >> 1; j > 0; j >>= 1) {
                    if (j == 32) {  // partners in the same lane: elements lane and lane + 32
                        if (k0 > k1) {  // kk == 64: ascending
                            const unsigned long long tk = k0;
                            k0 = k1;
                            k1 = tk;
                        }
                    } else {
#pragma unroll
                        for (int h = 0; h < 2; h++) {
                            unsigned long long& kr = h ? k1 : k0;
                            const int idx = lane + 32 * h;
                            const unsigned long long pk = __shfl_xor_sync(0xffffffffu, kr, j);
                            const bool up = (idx & kk) == 0;
                            const bool lower = (lane & j) == 0;
                            if (lower ? ((kr > pk) == up) : ((kr < pk) == up)) kr = pk;
                        }
                    }
                }
            }
            if (lane < len) rows[a + lane] = (uint32_t)k0;
            if (lane + 32 < len) rows[a + lane + 32] = (uint32_t)k1;
            continue;
        }
        int p2 = 128;
        while (p2 < len) p2 <<= 1;
        for (int i = lane; i < p2; i += 32) sk[i] = i < len ? row_key(rows[a + i], posA) : ~0ull;
        __syncwarp();
        for (int kk = 2; kk <= p2; kk <<= 1) {
            for (int j = kk >> 1; j > 0; j >>= 1) {
                for (int t = lane; t < (p2 >> 1); t += 32) {
                    const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
                    const int ij = i | j;
                    const bool up = (i & kk) == 0;
                    const unsigned long long x0 = sk[i], x1 = sk[ij];
                    if ((x0 > x1) == up) {
                        sk[i] = x1;
                        sk[ij] = x0;
                    }
                }
                __syncwarp();
            }
        }
        for (int i = lane; i < len; i += 32) rows[a + i] = (uint32_t)sk[i];
        __syncwarp();
    }
}

// long rows (> SORT_WIDE): one block per row, bitonic sort in shared memory (<= LONG_SORT_MAX
// entries), in global memory beyond that (rare: only at xi ~ spacing)
__global__ void __launch_bounds__(512)
k_sort_long(uint32_t e_lo, uint32_t e_hi, const unsigned long long* __restrict__ rowptr,
            const float4* __restrict__ posA, uint32_t* __restrict__ rows) {
    __shared__ unsigned long long sh[LONG_SORT_MAX];
    for (uint32_t e = e_lo + blockIdx.x; e < e_hi; e += gridDim.x) {
        const unsigned long long a = rowptr[e], b = rowptr[e + 1];
        const int len = (int)(b - a);
        if (len <= SORT_WIDE) continue;  // k_sort_wide's
        if (len <= LONG_SORT_MAX) {
            int p2 = 1;
            while (p2 < len) p2 <<= 1;
            for (int i = threadIdx.x; i < p2; i += blockDim.x)
                sh[i] = i < len ? row_key(rows[a + i], posA) : ~0ull;
            __syncthreads();
            for (int k = 2; k <= p2; k <<= 1) {
                for (int j = k >> 1; j > 0; j >>= 1) {
                    for (int i = threadIdx.x; i < p2; i += blockDim.x) {
                        int ij = i ^ j;
                        if (ij > i) {
                            bool up = (i & k) == 0;
                            unsigned long long x = sh[i], y = sh[ij];
                            if ((x > y) == up) {
                                sh[i] = y;
                                sh[ij] = x;
                            }
                        }
                    }
                    __syncthreads();
                }
            }
            for (int i = threadIdx.x; i < len; i += blockDim.x) rows[a + i] = (uint32_t)sh[i];
            __syncthreads();
        } else {  // beyond shared memory: in place in global memory, keys gathered per comparator
            __syncthreads();
            block_sort_global(rows + a, (int64_t)len, [posA](uint32_t x) { return row_key(x, posA); });
        }
    }
}

}  // namespace

// one candidate sweep of the count form in the given mode (CM_DEG / CM_FOREST), counting tests
static cc_status count_sweep(cc_ctx* c, int mode, unsigned long long* tests) {
    const int64_t n = c->n;
    if (n <= 0) return CC_OK;
    const bool half = !c->th.periodic || (c->g.ny >= 3 && c->g.nz >= 3);
    const char* env = std::getenv("CC_K2_TILED");
    const unsigned long long cap = (unsigned long long)c->near.cap;
    if (c->g.nx == 1 && half && !(env && (env[0] == '0' || env[0] == '1'))) {
        const int64_t nwarp = (n + 31) / 32;
        const unsigned nb = (unsigned)((nwarp + CW_WARPS - 1) / CW_WARPS);
        if (mode == CM_DEG)
            CCL(c, k_pairs_count_warp<CM_DEG><<<nb, PAIR_THREADS, 0, c->stream>>>(
                n, c->orig4.p, c->dec4.p, c->xk.p, c->cell_start.p, c->g, c->th, c->r_pair, (uint32_t)c->n_in, c->deg.p,
                c->parent_base.p, c->near.p, c->near_n.p, cap, tests));
        else
            CCL(c, k_pairs_count_warp<CM_FOREST><<<nb, PAIR_THREADS, 0, c->stream>>>(
                n, c->orig4.p, c->dec4.p, c->xk.p, c->cell_start.p, c->g, c->th, c->r_pair, (uint32_t)c->n_in, c->deg.p,
                c->parent_base.p, c->near.p, c->near_n.p, cap, tests));
    } else if (c->g.nx == 1 && half && env && env[0] == '1') {  // A/B variant (slower)
        if (mode != CM_DEG) return CC_OK;  // it does both in the degree sweep
        const double per_row = (double)n / ((double)c->g.ny * c->g.nz);
        const int trows = std::max(1, std::min(TROWS_MAX, (int)(240.0 / std::max(per_row, 1.0))));
        const int tiles_y = (c->g.ny + trows - 1) / trows;
        const int64_t ntiles = (int64_t)c->g.nz * tiles_y;
        const unsigned nbk = (unsigned)std::min<int64_t>(ntiles, 148 * 8);
        CCL(c, k_pairs_count_tiled<<<nbk, PAIR_THREADS, 0, c->stream>>>(
            n, c->orig4.p, c->dec4.p, c->xk.p, c->cell_start.p, c->g, c->th, c->r_pair, (uint32_t)c->n_in, c->deg.p,
            c->parent_base.p, c->near.p, c->near_n.p, cap, tests, ntiles, tiles_y, trows));
    } else {
        CCL(c, k_pairs_count<<<(unsigned)((n + PAIR_THREADS - 1) / PAIR_THREADS), PAIR_THREADS, 0, c->stream>>>(
            mode, n, c->orig4.p, c->dec4.p, c->xk.p, c->cell_start.p, c->g, c->th, c->r_pair, (uint32_t)c->n_in,
            c->deg.p, c->parent_base.p, c->near.p, c->near_n.p, cap, tests));
    }
    CC_CUDA(c, cudaGetLastError());
    return CC_OK;
}

// S2's count: band partners per slot (the degrees) -- no FoF work (the stable-forest
// unions of round 1's count sweep were S6 work inside the S1-S5 timing)
cc_status pairs_count(cc_ctx* c) {
    const int64_t n = c->n;
    CC_TRY(cc_ensure(c, c->deg, (size_t)std::max<int64_t>(n, 1), "deg"));
    CC_CUDA(c, cudaMemsetAsync(c->deg.p, 0, (size_t)std::max<int64_t>(n, 1) * sizeof(uint32_t), c->stream));
    const int64_t near_cap = std::max<int64_t>(4096, n / 128);
    CC_TRY(cc_ensure(c, c->near, (size_t)near_cap, "near-shell pairs"));
    CC_TRY(cc_ensure(c, c->near_n, 1, "near-shell count"));
    CC_TRY(cc_ensure(c, c->parent_base, (size_t)std::max<int64_t>(n, 1), "stable forest"));
    CC_CUDA(c, cudaMemsetAsync(c->near_n.p, 0, sizeof(unsigned long long), c->stream));
    c->base_valid = false;
    const char* env = std::getenv("CC_K2_TILED");
    const bool tiled = env && env[0] == '1';
    if (tiled) CC_TRY(fof_base_begin(c));  // the A/B variant builds the forest in the same sweep
    int tok = cc_prof_begin(c, "K2_count");
    CC_TRY(count_sweep(c, CM_DEG, work_counters(c) + 2));
    cc_prof_end(c, tok);
    if (tiled) {
        CC_TRY(fof_base_end(c));
        CC_TRY(read_near_count(c));
    }
    return CC_OK;
}

// S6 data, built at the first FoF labelling after cc_find_vulnerable: the stable forest (links
// with original d2 <= lo2s, provably linked in every position set within xi_f) and the near-shell
// list, by the same candidate sweep in CM_FOREST mode
cc_status fof_base_build(cc_ctx* c) {
    if (c->base_valid) return CC_OK;
    CC_CUDA(c, cudaMemsetAsync(c->near_n.p, 0, sizeof(unsigned long long), c->stream));
    CC_TRY(fof_base_begin(c));
    CC_TRY(count_sweep(c, CM_FOREST, work_counters(c) + 4));
    CC_TRY(fof_base_end(c));
    return read_near_count(c);
}

cc_status read_near_count(cc_ctx* c) {
    CC_CUDA(c, cudaMemcpyAsync(c->h_counters + 11, c->near_n.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                               c->stream));
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    c->near_count = (int64_t)c->h_counters[11];
    return CC_OK;
}

// totals_h = the 56-byte VDeg total (scan.cu): entries per class, editables per class, ghosts
cc_status rows_resolve(cc_ctx* c, const unsigned long long* totals_h) {
    uint32_t cnt[4], ghosts;
    std::memcpy(cnt, totals_h + 4, sizeof(cnt));
    std::memcpy(&ghosts, totals_h + 6, sizeof(ghosts));
    int64_t e = 0, ent = 0;
    for (int k = 0; k < 4; k++) {
        c->E_cls[k] = cnt[k];
        e += cnt[k];
        ent += (int64_t)totals_h[k];
    }
    c->E = e;
    c->E_all = e + ghosts;
    c->nent = ent;
    return CC_OK;  // eidx and the per-editable arrays were written by the class scan (scan.cu)
}

cc_status pairs_fill(cc_ctx* c) {
    const int64_t n = c->n;
    CC_TRY(cc_ensure(c, c->rows, (size_t)c->nent + 8, "rows"));  // +8: k_pgd<1> reads whole 16-byte vectors
    if (n > 0 && c->nent > 0) {
        int tok = cc_prof_begin(c, "K2_fill");
        CC_TRY(cc_ensure(c, c->scratch_u32, (size_t)std::max<int64_t>(c->E, 1), "row cursors"));
        CC_CUDA(c, cudaMemsetAsync(c->scratch_u32.p, 0, (size_t)std::max<int64_t>(c->E, 1) * sizeof(uint32_t),
                                   c->stream));
        CCL(c, k_pairs_fill<<<(unsigned)((c->E_all + PAIR_THREADS - 1) / PAIR_THREADS), PAIR_THREADS, 0,
                              c->stream>>>(
            (uint32_t)c->E_all, c->slotE.p, c->orig4.p, c->xk.p, c->cell_start.p, c->g, c->th, c->r_pair, c->eidx.p,
            (uint32_t)c->E,
            reinterpret_cast<const unsigned long long*>(c->rowptr.p), c->scratch_u32.p, c->rows.p,
            work_counters(c) + 3));
        cc_prof_end(c, tok);
        CC_CUDA(c, cudaGetLastError());
    }
    return CC_OK;
}

cc_status rows_finish(cc_ctx* c) {
    const int64_t Ea = c->E_all;
    unsigned long long* rowptr = reinterpret_cast<unsigned long long*>(c->rowptr.p);
    CCL(c, k_rowptr_tail<<<1, 1, 0, c->stream>>>(rowptr, (uint32_t)Ea, (unsigned long long)c->nent));
    CC_CUDA(c, cudaGetLastError());
    CC_TRY(pairs_fill(c));
    const uint32_t e_short = (uint32_t)(c->E_cls[0] + c->E_cls[1] + c->E_cls[2]);
    if (c->E > 0 && c->nent > 0) {
        int t2 = cc_prof_begin(c, "K2_sort");
        const uint32_t e0 = (uint32_t)c->E_cls[0], e1 = e0 + (uint32_t)c->E_cls[1];
        auto groups = [&](uint64_t rows_n, int w) { return (unsigned)((rows_n * w + PAIR_THREADS - 1) / PAIR_THREADS); };
        if (c->E_cls[0] > 0)
            CCL(c, k_sort_group<4><<<groups(c->E_cls[0], 4), PAIR_THREADS, 0, c->stream>>>(0u, e0, rowptr, c->posA.p,
                                                                                            c->rows.p));
        if (c->E_cls[1] > 0)
            CCL(c, k_sort_group<16><<<groups(c->E_cls[1], 16), PAIR_THREADS, 0, c->stream>>>(e0, e1, rowptr,
                                                                                              c->posA.p, c->rows.p));
        if (c->E_cls[2] > 0)
            CCL(c, k_sort_group<32><<<groups(c->E_cls[2], 32), PAIR_THREADS, 0, c->stream>>>(e1, e_short, rowptr,
                                                                                              c->posA.p, c->rows.p));
        if (c->E_cls[3] > 0) {
            CCL(c, k_sort_wide<<<(unsigned)std::min<int64_t>((c->E_cls[3] + SW_WARPS - 1) / SW_WARPS, 148 * 8),
                                 32 * SW_WARPS, 0, c->stream>>>(e_short, (uint32_t)c->E, rowptr, c->posA.p,
                                                                c->rows.p));
            CCL(c, k_sort_long<<<(unsigned)std::min<int64_t>(c->E_cls[3], 148 * 8), 512, 0, c->stream>>>(
                e_short, (uint32_t)c->E, rowptr, c->posA.p, c->rows.p));
        }
        cc_prof_end(c, t2);
        CC_CUDA(c, cudaGetLastError());
    }
    return CC_OK;
}

}  // namespace cc
