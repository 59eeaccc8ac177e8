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
#include <cstring>

#include "cc_internal.cuh"

namespace cc {
namespace {

constexpr int PAIR_THREADS = 256;

// pass 1 (each unordered pair once, for_each_pair_forward): deg[] = band partners per slot
// (atomics for the far endpoint), ghost endpoints of band pairs with an owned partner get bit 31
// of their deg word (multi-GPU: they become ghost editables); stable links (d2 <= lo2) are
// united into the stable FoF forest in the same sweep.
__global__ void __launch_bounds__(PAIR_THREADS)
k_pairs_count(int64_t n, const float4* __restrict__ orig4, const float4* __restrict__ dec4,
              const uint32_t* __restrict__ xk, const uint32_t* __restrict__ cs, Grid g, Th t, double r, uint32_t n_own,
              uint32_t* __restrict__ deg, uint32_t* __restrict__ par_base, uint2* __restrict__ near,
              unsigned long long* __restrict__ near_n, unsigned long long near_cap, unsigned long long* __restrict__ tests) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    unsigned ntest = 0;  // pair tests (candidates evaluated), reported as tests/s
    const bool multi = n_own < (uint32_t)n;
    const bool ghost = multi && __float_as_uint(dec4[s].w) >= n_own;
    const float4 p = orig4[s];
    double u;
    int cx, cy, cz;
    cell_of(p.x, p.y, p.z, g, u, cx, cy, cz);
    const bool inner = interior(p.x, p.y, p.z, g, t);
    const float lo2s = inner ? t.lo2s_i : t.lo2s_w, hi2s = inner ? t.hi2s_i : t.hi2s_w;
    uint32_t cnt = 0;
    uint32_t rs = (uint32_t)s;  // cached ancestor of s in the stable forest (uf_link)
    auto test = [&](uint32_t j) {
        ntest++;
        const float4 q = orig4[j];
        const float d2 = inner ? dist2_nw(p, q) : dist2(p, q, t);
        if (t.lo2 < d2 && d2 <= t.hi2) {
            const bool gj = multi && __float_as_uint(dec4[j].w) >= n_own;
            if (!ghost) {
                cnt++;
                if (gj) atomicOr(&deg[j], 0x80000000u);
                else atomicAdd(&deg[j], 1u);
            } else if (!gj) {
                atomicAdd(&deg[j], 1u);
                atomicOr(&deg[s], 0x80000000u);
            }
        } else if (d2 <= lo2s) {
            // a stable FoF link: provably linked in the original, decompressed and corrected
            // positions alike (Th::lo2s, fof.cu), united here in the same candidate sweep
            uf_link(par_base, (uint32_t)s, j, rs);
        } else if (d2 <= hi2s) {
            // near shell (lo2s, lo2] or (hi2, hi2s]: not vulnerable, but fp32 rounding could flip
            // its link in other positions -- listed, re-tested by every FoF labelling
            const unsigned long long q = atomicAdd(near_n, 1ull);
            if (q < near_cap) near[q] = make_uint2((uint32_t)s, j | (d2 <= t.b2 ? 0x80000000u : 0u));
        }
    };
    for_each_pair_forward(g, cs, xk, (uint32_t)s, u, cy, cz, r, t.periodic != 0, test);
    if (cnt) atomicAdd(&deg[s], cnt);
    warp_count(tests, ntest);
}

// after the scan: editable ranks and row offsets become global (class-major numbering: class
// bases first, ghost editables after all owned ones)
struct ClassBases {
    uint32_t e[4];
    unsigned long long off[4];
};
__global__ void k_resolve(int64_t n, const uint32_t* __restrict__ cls, ClassBases cb, uint32_t e_own,
                          uint32_t* __restrict__ eidx, unsigned long long* __restrict__ rowoff) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const uint32_t k = cls[s];
    if (k <= 3u) {
        eidx[s] += cb.e[k];
        rowoff[s] += cb.off[k];
    } else if (k == 4u) {
        eidx[s] += e_own;
    } else {
        eidx[s] = 0xFFFFFFFFu;
    }
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
             uint32_t* __restrict__ cur, uint32_t* __restrict__ rows, uint32_t* __restrict__ par_orig,
             unsigned long long* __restrict__ tests) {
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
    uint32_t rs = (uint32_t)s;  // cached ancestor of s in the ORIG forest (uf_link)
    auto emit = [&](uint32_t j) {
        ntest++;
        const float4 q = orig4[j];
        const float d2 = inner ? dist2_nw(p, q) : dist2(p, q, t);
        if (t.lo2 < d2 && d2 <= t.hi2) {
            const uint32_t ej = eidx[j], gq = __float_as_uint(q.w);
            const uint32_t ol = d2 <= t.b2 ? ENT_OLINK : 0u;
            if (es < e_own) rows[rowptr[es] + atomicAdd(&cur[es], 1u)] = ej | (gq > gp ? ENT_UPPER : 0u) | ol;
            if (ej < e_own) rows[rowptr[ej] + atomicAdd(&cur[ej], 1u)] = es | (gp > gq ? ENT_UPPER : 0u) | ol;
            // FoF(ORIG) = the stable forest + the original-linked band pairs (an owned endpoint;
            // ghost-ghost pairs belong to their owner rank)
            if (ol && (es < e_own || ej < e_own)) uf_link(par_orig, (uint32_t)s, j, rs);
        }
    };
    for_each_pair_forward(g, cs, xk, (uint32_t)s, u, cy, cz, r, t.periodic != 0, emit);
    warp_count(tests, ntest);
}

// compaction: editable e -> slot, row start, original and starting position
__global__ void __launch_bounds__(PAIR_THREADS)
k_compact(int64_t n, const uint32_t* __restrict__ deg, const uint32_t* __restrict__ eidx,
          const unsigned long long* __restrict__ rowoff, const float4* __restrict__ orig4,
          const float4* __restrict__ dec4, uint32_t e_own, unsigned long long nent, uint32_t* __restrict__ slotE,
          unsigned long long* __restrict__ rowptr, float4* __restrict__ origE, float4* __restrict__ posA) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const uint32_t e = eidx[s];
    if (e == 0xFFFFFFFFu) return;
    const float4 o = orig4[s], d = dec4[s];
    slotE[e] = (uint32_t)s;
    rowptr[e] = (e < e_own) ? rowoff[s] : nent;
    origE[e] = o;
    posA[e] = make_float4(d.x, d.y, d.z, o.w);
}

__global__ void k_rowptr_tail(unsigned long long* rowptr, uint32_t e_all, unsigned long long nent) {
    rowptr[e_all] = nent;
}

constexpr int SHORT_ROW = 32;
constexpr int LONG_SORT_MAX = 4096;  // block bitonic capacity (entries)

__device__ __forceinline__ unsigned long long row_key(uint32_t ent, const float4* __restrict__ posA) {
    return ((unsigned long long)__float_as_uint(posA[ent & ENT_IDX].w) << 32) | ent;
}

// sort each row by partner gid: rows of classes 0-2 (<= 32 entries) in registers (insertion
// sort); class-3 rows by the block kernel
__global__ void __launch_bounds__(PAIR_THREADS)
k_sort_short(uint32_t e_end, const unsigned long long* __restrict__ rowptr, const float4* __restrict__ posA,
             uint32_t* __restrict__ rows) {
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= e_end) return;
    const unsigned long long a = rowptr[e], b = rowptr[e + 1];
    const int len = (int)(b - a);
    if (len <= 1 || len > SHORT_ROW) return;
    unsigned long long v[SHORT_ROW];
    for (int i = 0; i < len; i++) {
        unsigned long long x = row_key(rows[a + i], posA);
        int j = i - 1;
        while (j >= 0 && v[j] > x) {
            v[j + 1] = v[j];
            j--;
        }
        v[j + 1] = x;
    }
    for (int i = 0; i < len; i++) rows[a + i] = (uint32_t)v[i];
}

// long rows: one block per row, bitonic sort in shared memory (<= LONG_SORT_MAX entries), and
// a serial in-place insertion sort by one thread beyond that (rare: only at xi ~ spacing)
__global__ void __launch_bounds__(512)
k_sort_long(uint32_t e_lo, uint32_t e_hi, const unsigned long long* __restrict__ rowptr,
            const float4* __restrict__ posA, uint32_t* __restrict__ rows) {
    __shared__ unsigned long long sh[LONG_SORT_MAX];
    for (uint32_t e = e_lo + blockIdx.x; e < e_hi; e += gridDim.x) {
        const unsigned long long a = rowptr[e], b = rowptr[e + 1];
        const int len = (int)(b - a);
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
        } else if (threadIdx.x == 0) {
            for (int i = 1; i < len; i++) {
                uint32_t x = rows[a + i];
                unsigned long long kx = row_key(x, posA);
                int j = i - 1;
                while (j >= 0 && row_key(rows[a + j], posA) > kx) {
                    rows[a + j + 1] = rows[a + j];
                    j--;
                }
                rows[a + j + 1] = x;
            }
        }
    }
}

}  // namespace

cc_status pairs_count(cc_ctx* c) {
    const int64_t n = c->n;
    CC_TRY(cc_ensure(c, c->deg, (size_t)std::max<int64_t>(n, 1), "deg"));
    CC_CUDA(c, cudaMemsetAsync(c->deg.p, 0, (size_t)std::max<int64_t>(n, 1) * sizeof(uint32_t), c->stream));
    CC_TRY(fof_base_begin(c));  // the stable FoF forest is built inside the count sweep
    const int64_t near_cap = std::max<int64_t>(4096, n / 128);
    CC_TRY(cc_ensure(c, c->near, (size_t)near_cap, "near-shell pairs"));
    CC_TRY(cc_ensure(c, c->near_n, 1, "near-shell count"));
    CC_CUDA(c, cudaMemsetAsync(c->near_n.p, 0, sizeof(unsigned long long), c->stream));
    if (n > 0) {
        int tok = cc_prof_begin(c, "K2_count");
        CCL(c, k_pairs_count<<<(unsigned)((n + PAIR_THREADS - 1) / PAIR_THREADS), PAIR_THREADS, 0, c->stream>>>(
            n, c->orig4.p, c->dec4.p, c->xk.p, c->cell_start.p, c->g, c->th, c->r_pair, (uint32_t)c->n_in, c->deg.p,
            c->parent_base.p, c->near.p, c->near_n.p, (unsigned long long)c->near.cap, work_counters(c) + 2));
        cc_prof_end(c, tok);
        CC_CUDA(c, cudaGetLastError());
    }
    return fof_base_end(c);
}

// totals_h = the 56-byte VDeg total (scan.cu): entries per class, editables per class, ghosts
cc_status rows_resolve(cc_ctx* c, const unsigned long long* totals_h) {
    uint32_t cnt[4], ghosts;
    std::memcpy(cnt, totals_h + 4, sizeof(cnt));
    std::memcpy(&ghosts, totals_h + 6, sizeof(ghosts));
    int64_t e = 0, ent = 0;
    ClassBases cb;
    for (int k = 0; k < 4; k++) {
        cb.e[k] = (uint32_t)e;
        cb.off[k] = (unsigned long long)ent;
        c->E_cls[k] = cnt[k];
        e += cnt[k];
        ent += (int64_t)totals_h[k];
    }
    c->E = e;
    c->E_all = e + ghosts;
    c->nent = ent;
    if (c->E_all >= MAX_LOCAL) return CC_OK;  // caller reports
    const int64_t n = c->n;
    if (n > 0)
        CCL(c, k_resolve<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(
            n, c->key.p, cb, (uint32_t)e, c->eidx.p, reinterpret_cast<unsigned long long*>(c->rowoff.p)));
    CC_CUDA(c, cudaGetLastError());
    return CC_OK;
}

cc_status pairs_fill(cc_ctx* c) {
    const int64_t n = c->n;
    CC_TRY(cc_ensure(c, c->parent_orig, (size_t)std::max<int64_t>(n, 1), "ORIG forest"));
    if (n > 0)
        CC_CUDA(c, cudaMemcpyAsync(c->parent_orig.p, c->parent_base.p, (size_t)n * sizeof(uint32_t),
                                   cudaMemcpyDeviceToDevice, c->stream));
    c->orig_valid = true;
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
            c->parent_orig.p, work_counters(c) + 3));
        cc_prof_end(c, tok);
        CC_CUDA(c, cudaGetLastError());
    }
    return union_near(c, nullptr, c->parent_orig.p);  // + the near shell's original links
}

cc_status rows_finish(cc_ctx* c) {
    const int64_t n = c->n, Ea = c->E_all;
    const size_t e1 = (size_t)std::max<int64_t>(Ea, 1);
    CC_TRY(cc_ensure(c, c->slotE, e1, "slotE"));
    CC_TRY(cc_ensure(c, c->rowptr, e1 + 1, "rowptr"));
    CC_TRY(cc_ensure(c, c->origE, e1, "origE"));
    CC_TRY(cc_ensure(c, c->posA, e1, "posA"));
    CC_TRY(cc_ensure(c, c->posB, e1, "posB"));
    unsigned long long* rowptr = reinterpret_cast<unsigned long long*>(c->rowptr.p);
    int tok = cc_prof_begin(c, "K2_compact");
    if (n > 0)
        CCL(c, k_compact<<<(unsigned)((n + PAIR_THREADS - 1) / PAIR_THREADS), PAIR_THREADS, 0, c->stream>>>(
            n, c->deg.p, c->eidx.p, reinterpret_cast<const unsigned long long*>(c->rowoff.p), c->orig4.p, c->dec4.p,
            (uint32_t)c->E, (unsigned long long)c->nent, c->slotE.p, rowptr, c->origE.p, c->posA.p));
    CCL(c, k_rowptr_tail<<<1, 1, 0, c->stream>>>(rowptr, (uint32_t)Ea, (unsigned long long)c->nent));
    cc_prof_end(c, tok);
    CC_CUDA(c, cudaGetLastError());
    CC_TRY(pairs_fill(c));
    const uint32_t e_short = (uint32_t)(c->E_cls[0] + c->E_cls[1] + c->E_cls[2]);
    if (c->E > 0 && c->nent > 0) {
        int t2 = cc_prof_begin(c, "K2_sort");
        if (e_short > 0)
            CCL(c, k_sort_short<<<(e_short + PAIR_THREADS - 1) / PAIR_THREADS, PAIR_THREADS, 0, c->stream>>>(
                e_short, rowptr, c->posA.p, c->rows.p));
        if (c->E_cls[3] > 0)
            CCL(c, k_sort_long<<<(unsigned)std::min<int64_t>(c->E_cls[3], 148 * 8), 512, 0, c->stream>>>(
                e_short, (uint32_t)c->E, rowptr, c->posA.p, c->rows.p));
        cc_prof_end(c, t2);
        CC_CUDA(c, cudaGetLastError());
    }
    return CC_OK;
}

}  // namespace cc
