// fof.cu -- K4 FoF labelling (S6) and K5 MCC / halo-size counters (S7).
//
// Paper: §II-B P:362 and Fig. 1 (edge iff d(p_i,p_j) <= b; FoF clusters = connected
// components), §II-B-1 P:381 (cell linking, forward neighbour cells), §II-B-2 P:387 (halo mass
// M_i ~ N_i, HMF), §IV-A P:9-15 (MCC over vulnerable pairs: FP = unlinked->linked,
// FN = linked->broken).  The paper does not describe its own FoF code (it cites HACC's).
//
// B200 form: one thread per particle tests the pinned fp32 d2 <= fl32(b^2) against the
// half-shell of its cell neighbourhood (13.5 cells) and unites on the fly with a lock-free
// union-find (atomicCAS hooks the larger root under the smaller index, path halving), then
// pointer jumping flattens the forest and atomicMin gives each component its min gid (R20).
// The same cell-sorted grid serves ORIG, DECOMP and CORR positions: its cells are >= b + 2 sqrt3
// xi wide and every position lies within xi of its original (R1).
#include <algorithm>

#include "cc_internal.cuh"

namespace cc {
namespace {

constexpr int FOF_THREADS = 256;

__global__ void k_iota(int64_t n, uint32_t* __restrict__ par) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s < n) par[s] = (uint32_t)s;
}

// link pass over the x-sorted rows: the half-shell of rows (own row forward in slot order,
// then rows (dz=0,dy=+1) and (dz=+1,dy=-1..1)) visits every unordered pair once; with fewer
// than 3 periodic rows per axis it falls back to all 9 rows with j > s.  The search radius r
// is b (ORIG) or b + 2 sqrt3 xi (DECOMP / CORR, whose positions are within xi of the original
// ones that built the structure), with the fp32 rounding margin.
__global__ void __launch_bounds__(FOF_THREADS)
k_fof_link(int64_t n, const float4* __restrict__ P, const float4* __restrict__ orig4, const uint32_t* __restrict__ xk,
           const uint32_t* __restrict__ cs, Grid g, Th t, double r, float thr2, uint32_t* __restrict__ par,
           unsigned long long* __restrict__ tests) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    unsigned ntest = 0;
    const float4 o = orig4[s];
    const float4 p = P[s];
    double u;
    int cx, cy, cz;
    cell_of(o.x, o.y, o.z, g, u, cx, cy, cz);
    const bool periodic_yz = t.periodic != 0;
    uint32_t rs = (uint32_t)s;  // cached ancestor of s (uf_link)
    auto link = [&](uint32_t j) {
        ntest++;
        const float4 q = P[j];
        if (dist2(p, q, t) <= thr2) uf_link(par, (uint32_t)s, j, rs);
    };
    for_each_pair_forward(g, cs, xk, (uint32_t)s, u, cy, cz, r, periodic_yz, link);
    warp_count(tests, ntest);
}

// read-only root walk: the flatten pass must not path-halve, or a halving write could land
// after another thread's final par[x] = root and leave x pointing at a non-root
__device__ __forceinline__ uint32_t uf_root(const uint32_t* par, uint32_t x) {
    uint32_t p = ld_rlx(par + x);
    while (p != x) {
        x = p;
        p = ld_rlx(par + x);
    }
    return x;
}

__global__ void k_flatten(int64_t n, uint32_t* __restrict__ par) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const uint32_t r = uf_root(par, (uint32_t)s);
    par[s] = r;  // only ever replaces par[s] by an ancestor of s: safe for concurrent walkers
}

__global__ void k_mingid(int64_t n, const uint32_t* __restrict__ par, const float4* __restrict__ orig4,
                         uint32_t* __restrict__ mingid, uint32_t* __restrict__ gsize,
                         unsigned long long* __restrict__ n_roots) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned int root = 0;
    // neighbouring slots mostly share a root (halo cores): one atomic per distinct root per warp
    const uint32_t r = s < n ? par[s] : 0xFFFFFFFFu;
    const uint32_t gid = s < n ? __float_as_uint(orig4[s].w) : 0xFFFFFFFFu;
    const unsigned int same = __match_any_sync(0xffffffffu, r);
    const uint32_t mn = __reduce_min_sync(same, gid);
    if (s < n) {
        if ((threadIdx.x & 31) == (unsigned)(__ffs(same) - 1)) {
            atomicMin(&mingid[r], mn);
            atomicAdd(&gsize[r], (uint32_t)__popc(same));
        }
        root = (r == (uint32_t)s);
    }
    const unsigned int cnt = __syncthreads_count(root);
    if (threadIdx.x == 0 && cnt) atomicAdd(n_roots, (unsigned long long)cnt);
}

// labels: first in slot order (par and, for the many singletons, mingid are read in order),
// then gathered into input order (a random 4-byte read per particle instead of a random partial
// sector write)
__global__ void k_labels_slot(int64_t n, const uint32_t* __restrict__ par, const uint32_t* __restrict__ mingid,
                              uint32_t* __restrict__ lab_s) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s < n) lab_s[s] = mingid[par[s]];
}
__global__ void k_labels(int64_t n_in, const uint32_t* __restrict__ slot_of, const uint32_t* __restrict__ lab_s,
                         uint32_t* __restrict__ labels) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_in) labels[i] = lab_s[slot_of[i]];
}

// MCC counters over the vulnerable pairs owned here (lower-gid endpoint, R17)
__global__ void __launch_bounds__(256)
k_mcc(uint32_t E, const unsigned long long* __restrict__ rowptr, const uint32_t* __restrict__ rows,
      const float4* __restrict__ W, const uint32_t* __restrict__ slotE, int via_slot, Th t,
      unsigned long long* __restrict__ out /* tp, tn, fp, fn */) {
    unsigned int c[4] = {0, 0, 0, 0};
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
        const float4 p = via_slot ? W[slotE[e]] : W[e];
        for (unsigned long long k = rowptr[e]; k < rowptr[e + 1]; k++) {
            const uint32_t ent = rows[k];
            if (!(ent & ENT_UPPER)) continue;
            const uint32_t j = ent & ENT_IDX;
            const float4 q = via_slot ? W[slotE[j]] : W[j];
            const bool lk = dist2(p, q, t) <= t.b2;
            const bool ol = (ent & ENT_OLINK) != 0;
            c[ol ? (lk ? 0 : 3) : (lk ? 2 : 1)]++;
        }
    }
    for (int q = 0; q < 4; q++) {
        unsigned int v = c[q];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&out[q], (unsigned long long)v);
    }
}

__global__ void __launch_bounds__(256)
k_get_pairs(uint32_t E, const unsigned long long* __restrict__ rowptr, const uint32_t* __restrict__ rows,
            const float4* __restrict__ posE, const float4* __restrict__ dec4, const uint32_t* __restrict__ slotE, Th t,
            int64_t cap, uint32_t* __restrict__ gi, uint32_t* __restrict__ gj, uint8_t* __restrict__ fl,
            unsigned long long* __restrict__ cnt) {
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
        const float4 pd = dec4[slotE[e]];
        const uint32_t g0 = __float_as_uint(posE[e].w);
        for (unsigned long long k = rowptr[e]; k < rowptr[e + 1]; k++) {
            const uint32_t ent = rows[k];
            if (!(ent & ENT_UPPER)) continue;
            const uint32_t j = ent & ENT_IDX;
            const float4 qd = dec4[slotE[j]];
            const uint8_t f = (uint8_t)(((ent & ENT_OLINK) ? 1 : 0) | (dist2(pd, qd, t) <= t.b2 ? 2 : 0));
            const unsigned long long q = atomicAdd(cnt, 1ull);
            if ((int64_t)q < cap) {
                gi[q] = g0;
                gj[q] = __float_as_uint(posE[j].w);
                fl[q] = f;
            }
        }
    }
}

__global__ void k_halo_collect(int64_t n, const uint32_t* __restrict__ par, const uint32_t* __restrict__ gsize,
                               uint32_t min_size, uint32_t* __restrict__ out, unsigned long long* __restrict__ cnt) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    if (par[s] == (uint32_t)s && gsize[s] >= min_size) {
        const unsigned long long q = atomicAdd(cnt, 1ull);
        out[q] = gsize[s];
    }
}

}  // namespace

// vulnerable-pair links on top of the stable forest: pair (e, j) is linked in the positions W
// (ORIG: its original-link bit; CORR: the pinned d2 <= b2 on the result positions)
__global__ void __launch_bounds__(256)
k_union_rows(uint32_t E, const unsigned long long* __restrict__ rowptr, const uint32_t* __restrict__ rows,
             const uint32_t* __restrict__ slotE, const float4* __restrict__ W, int use_orig_bit, Th t,
             uint32_t* __restrict__ par) {
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
        const unsigned long long k0 = rowptr[e], k1 = rowptr[e + 1];
        if (k0 == k1) continue;
        const uint32_t se = slotE[e];
        uint32_t rs = se;
        const float4 p = use_orig_bit ? make_float4(0.f, 0.f, 0.f, 0.f) : W[e];
        for (unsigned long long k = k0; k < k1; k++) {
            const uint32_t ent = rows[k];
            const uint32_t j = ent & ENT_IDX;
            if (!(ent & ENT_UPPER) && j < E) continue;  // each owned pair once; ghost partners always
            const bool lk = use_orig_bit ? (ent & ENT_OLINK) != 0 : dist2(p, W[j], t) <= t.b2;
            if (lk) uf_link(par, se, slotE[j], rs);
        }
    }
}

// near-shell pairs (K2 count, Th::lo2s/hi2s): linked in the original iff bit 31 (P == nullptr),
// else iff the pinned d2 <= b2 on the slot-order positions P
__global__ void __launch_bounds__(256)
k_union_near(unsigned long long m, const uint2* __restrict__ near, const float4* __restrict__ P, Th t,
             uint32_t* __restrict__ par) {
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const uint2 e = near[i];
        const uint32_t s = e.x, j = e.y & 0x7FFFFFFFu;
        const bool lk = P ? dist2(P[s], P[j], t) <= t.b2 : (e.y >> 31) != 0u;
        if (lk) {
            uint32_t rs = s;
            uf_link(par, s, j, rs);
        }
    }
}

cc_status union_near(cc_ctx* c, const float4* P, uint32_t* par) {
    const unsigned long long m = (unsigned long long)std::min<int64_t>(c->near_count, (int64_t)c->near.cap);
    if (m == 0) return CC_OK;
    const unsigned nb = (unsigned)std::min<unsigned long long>((m + 255) / 256, 148 * 8);
    CCL(c, k_union_near<<<nb, 256, 0, c->stream>>>(m, c->near.p, P, c->th, par));
    CC_CUDA(c, cudaGetLastError());
    return CC_OK;
}

// The stable forest: links with original d2 <= lo2s (provably linked in the original,
// decompressed and corrected positions alike, Th) are united ONCE per build, by the count form's
// candidate sweep in forest mode (pairs.cu fof_base_build, at the first labelling); each FoF
// labelling then adds the near shell and the vulnerable rows.  These bracket that sweep.
cc_status fof_base_begin(cc_ctx* c) {
    const int64_t n = c->n;
    CC_TRY(cc_ensure(c, c->parent_base, (size_t)std::max<int64_t>(n, 1), "stable forest"));
    c->base_valid = false;
    if (n > 0) CCL(c, k_iota<<<(unsigned)((n + FOF_THREADS - 1) / FOF_THREADS), FOF_THREADS, 0, c->stream>>>(
                          n, c->parent_base.p));
    CC_CUDA(c, cudaGetLastError());
    return CC_OK;
}

cc_status fof_base_end(cc_ctx* c) {
    const int64_t n = c->n;
    if (n > 0) CCL(c, k_flatten<<<(unsigned)((n + FOF_THREADS - 1) / FOF_THREADS), FOF_THREADS, 0, c->stream>>>(
                          n, c->parent_base.p));
    CC_CUDA(c, cudaGetLastError());
    c->base_valid = true;
    return CC_OK;
}

cc_status fof_run(cc_ctx* c, int which, uint32_t* labels, int64_t* n_groups) {
    CC_TRY(ensure_slot_of(c));
    const int64_t n = c->n;
    const size_t n1 = (size_t)std::max<int64_t>(n, 1);
    CC_TRY(cc_ensure(c, c->parent, n1, "parent"));
    CC_TRY(cc_ensure(c, c->mingid, n1, "mingid"));
    CC_TRY(cc_ensure(c, c->gsize, n1, "gsize"));
    CC_TRY(cc_ensure(c, c->counters, 16, "counters"));
    if (which == CC_CORR) CC_TRY(ensure_cor4(c));
    const float4* P = which == CC_ORIG ? c->orig4.p : (which == CC_DECOMP ? c->dec4.p : c->cor4.p);
    // ORIG and CORR: the stable forest (provably linked in both, Th::lo2s) + the near shell
    // re-tested + the vulnerable rows (the near list overflowing its buffer: direct search)
    int tok = cc_prof_begin(c, "K4_fof");
    if (c->state >= 2 && (which == CC_ORIG || which == CC_CORR)) CC_TRY(fof_base_build(c));
    const bool near_ok = c->near_count <= (int64_t)c->near.cap;
    const bool via_base = c->state >= 2 && c->base_valid && near_ok && (which == CC_ORIG || which == CC_CORR);
    CC_CUDA(c, cudaMemsetAsync(c->mingid.p, 0xFF, n1 * sizeof(uint32_t), c->stream));
    CC_CUDA(c, cudaMemsetAsync(c->gsize.p, 0, n1 * sizeof(uint32_t), c->stream));
    CC_CUDA(c, cudaMemsetAsync(c->counters.p + 8, 0, sizeof(unsigned long long), c->stream));
    const unsigned nb = (unsigned)((n + FOF_THREADS - 1) / FOF_THREADS);
    if (n > 0) {
        if (via_base) {
            CC_CUDA(c, cudaMemcpyAsync(c->parent.p, c->parent_base.p, (size_t)n * sizeof(uint32_t),
                                       cudaMemcpyDeviceToDevice, c->stream));
            if (c->E > 0) {
                const int nbe = (int)std::min<int64_t>((c->E + 255) / 256, 148 * 8);
                CCL(c, k_union_rows<<<nbe, 256, 0, c->stream>>>(
                           (uint32_t)c->E, reinterpret_cast<const unsigned long long*>(c->rowptr.p), c->rows.p,
                           c->slotE.p, which == CC_ORIG ? nullptr : pgd_result(c), which == CC_ORIG ? 1 : 0, c->th,
                           c->parent.p));
            }
            CC_TRY(union_near(c, which == CC_ORIG ? nullptr : c->cor4.p, c->parent.p));
        } else {
            CCL(c, k_iota<<<nb, FOF_THREADS, 0, c->stream>>>(n, c->parent.p));
            CCL(c, k_fof_link<<<nb, FOF_THREADS, 0, c->stream>>>(n, P, c->orig4.p, c->xk.p, c->cell_start.p, c->g,
                                                                 c->th, which == CC_ORIG ? c->r_link : c->r_pair,
                                                                 c->th.b2, c->parent.p, work_counters(c) + 4));
        }
        CCL(c, k_flatten<<<nb, FOF_THREADS, 0, c->stream>>>(n, c->parent.p));
        CCL(c, k_mingid<<<nb, FOF_THREADS, 0, c->stream>>>(n, c->parent.p, c->orig4.p, c->mingid.p, c->gsize.p,
                                                    c->counters.p + 8));
    }
    if (c->nranks > 1) CC_TRY(dist_fof_merge(c, n_groups));  // global labels across slabs (X4)
    if (n > 0 && labels && c->n_in > 0) {
        CC_TRY(cc_ensure(c, c->lab_s, n1, "slot labels"));
        CCL(c, k_labels_slot<<<nb, FOF_THREADS, 0, c->stream>>>(n, c->parent.p, c->mingid.p, c->lab_s.p));
        CCL(c, k_labels<<<(unsigned)((c->n_in + FOF_THREADS - 1) / FOF_THREADS), FOF_THREADS, 0, c->stream>>>(
                   c->n_in, c->slot_of.p, c->lab_s.p, labels));
    }
    cc_prof_end(c, tok);
    CC_CUDA(c, cudaGetLastError());
    if (n_groups && c->nranks == 1) {
        CC_CUDA(c, cudaMemcpyAsync(c->h_counters, c->counters.p + 8, sizeof(unsigned long long),
                                   cudaMemcpyDeviceToHost, c->stream));
        CC_CUDA(c, cudaStreamSynchronize(c->stream));
        *n_groups = (int64_t)c->h_counters[0];
    }
    return CC_OK;
}

cc_status mcc_run(cc_ctx* c, int which, unsigned long long* counts_dev) {
    CC_CUDA(c, cudaMemsetAsync(counts_dev, 0, 4 * sizeof(unsigned long long), c->stream));
    if (c->E == 0) return CC_OK;
    const float4* W;
    int via_slot;
    if (which == CC_DECOMP) {
        W = c->dec4.p;
        via_slot = 1;
    } else if (which == CC_ORIG) {
        W = c->orig4.p;
        via_slot = 1;
    } else {
        W = pgd_result(c);
        via_slot = 0;
    }
    int nb = (int)std::min<int64_t>((c->E + 255) / 256, 148 * 8);
    int tok = cc_prof_begin(c, "K5_mcc");
    CCL(c, k_mcc<<<nb, 256, 0, c->stream>>>((uint32_t)c->E, reinterpret_cast<const unsigned long long*>(c->rowptr.p),
                                     c->rows.p, W, c->slotE.p, via_slot, c->th, counts_dev));
    cc_prof_end(c, tok);
    CC_CUDA(c, cudaGetLastError());
    return CC_OK;
}

// canonical order (§8(b): gi < gj, sorted by (gi, gj)) by a counting sort on the row owner's gid:
// rows are already sorted by partner gid (R14), so placing each editable's upper entries at the
// exclusive prefix of the per-gid counts yields the sorted list without a comparison sort.
__global__ void k_max_gid(uint32_t E, const float4* __restrict__ posE, unsigned int* __restrict__ mx) {
    uint32_t m = 0u;
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x)
        m = max(m, __float_as_uint(posE[e].w));
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0) atomicMax(mx, m);
}

__global__ void k_count_upper(uint32_t E, const unsigned long long* __restrict__ rowptr,
                              const uint32_t* __restrict__ rows, const float4* __restrict__ posE,
                              uint32_t* __restrict__ cnt) {
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
        uint32_t u = 0;
        for (unsigned long long k = rowptr[e]; k < rowptr[e + 1]; k++) u += (rows[k] & ENT_UPPER) ? 1u : 0u;
        cnt[__float_as_uint(posE[e].w)] = u;
    }
}

__global__ void __launch_bounds__(256)
k_get_pairs_sorted(uint32_t E, const unsigned long long* __restrict__ rowptr, const uint32_t* __restrict__ rows,
                   const float4* __restrict__ posE, const float4* __restrict__ dec4, const uint32_t* __restrict__ slotE,
                   const uint32_t* __restrict__ pos, Th t, int64_t cap, uint32_t* __restrict__ gi,
                   uint32_t* __restrict__ gj, uint8_t* __restrict__ fl) {
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
        const float4 pd = dec4[slotE[e]];
        const uint32_t g0 = __float_as_uint(posE[e].w);
        int64_t q = pos[g0];
        for (unsigned long long k = rowptr[e]; k < rowptr[e + 1]; k++) {
            const uint32_t ent = rows[k];
            if (!(ent & ENT_UPPER)) continue;
            const uint32_t j = ent & ENT_IDX;
            const float4 qd = dec4[slotE[j]];
            if (q < cap) {
                gi[q] = g0;
                gj[q] = __float_as_uint(posE[j].w);
                fl[q] = (uint8_t)(((ent & ENT_OLINK) ? 1 : 0) | (dist2(pd, qd, t) <= t.b2 ? 2 : 0));
            }
            q++;
        }
    }
}

cc_status get_pairs_run(cc_ctx* c, uint32_t* gi, uint32_t* gj, uint8_t* flags, int64_t cap, unsigned long long* n_dev) {
    CC_CUDA(c, cudaMemsetAsync(n_dev, 0, sizeof(unsigned long long), c->stream));
    if (c->E == 0) return CC_OK;
    const int nb = (int)std::min<int64_t>((c->E + 255) / 256, 148 * 8);
    const unsigned long long* rowptr = reinterpret_cast<const unsigned long long*>(c->rowptr.p);
    if (cap <= 0) {  // count only (the total is needed to size the outputs)
        CCL(c, k_get_pairs<<<nb, 256, 0, c->stream>>>((uint32_t)c->E, rowptr, c->rows.p, c->origE.p, c->dec4.p,
                                                       c->slotE.p, c->th, 0, gi, gj, flags, n_dev));
        CC_CUDA(c, cudaGetLastError());
        return CC_OK;
    }
    // largest owner gid -> counting-sort array size
    CC_TRY(cc_ensure(c, c->counters, 16, "counters"));
    unsigned int* mx = reinterpret_cast<unsigned int*>(c->counters.p + 13);
    CC_CUDA(c, cudaMemsetAsync(mx, 0, sizeof(unsigned int), c->stream));
    CCL(c, k_max_gid<<<nb, 256, 0, c->stream>>>((uint32_t)c->E, c->origE.p, mx));
    unsigned int hmx = 0;
    CC_CUDA(c, cudaMemcpyAsync(&hmx, mx, sizeof(hmx), cudaMemcpyDeviceToHost, c->stream));
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    const int64_t G = (int64_t)hmx + 1;
    CC_TRY(cc_ensure(c, c->gp_cnt, (size_t)G, "pair sort counts"));
    CC_TRY(cc_ensure(c, c->gp_pos, (size_t)G, "pair sort offsets"));
    CC_CUDA(c, cudaMemsetAsync(c->gp_cnt.p, 0, (size_t)G * sizeof(uint32_t), c->stream));
    CCL(c, k_count_upper<<<nb, 256, 0, c->stream>>>((uint32_t)c->E, rowptr, c->rows.p, c->origE.p, c->gp_cnt.p));
    CC_CUDA(c, cudaMemsetAsync(n_dev, 0, sizeof(unsigned long long), c->stream));
    CC_TRY(scan_u32_to_u32(c, c->gp_cnt.p, c->gp_pos.p, G, reinterpret_cast<uint64_t*>(n_dev)));
    CCL(c, k_get_pairs_sorted<<<nb, 256, 0, c->stream>>>((uint32_t)c->E, rowptr, c->rows.p, c->origE.p, c->dec4.p,
                                                          c->slotE.p, c->gp_pos.p, c->th, cap, gi, gj, flags));
    CC_CUDA(c, cudaGetLastError());
    return CC_OK;
}

cc_status halo_sizes_run(cc_ctx* c, int64_t min_size, int64_t* sizes_h, int64_t cap, int64_t* n_h) {
    const int64_t n = c->n;
    CC_TRY(cc_ensure(c, c->scratch_u32, (size_t)std::max<int64_t>(n, 1), "halo list"));
    CC_CUDA(c, cudaMemsetAsync(c->counters.p + 9, 0, sizeof(unsigned long long), c->stream));
    if (n > 0)
        CCL(c, k_halo_collect<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(
            n, c->parent.p, c->gsize.p, (uint32_t)std::max<int64_t>(min_size, 1), c->scratch_u32.p, c->counters.p + 9));
    CC_CUDA(c, cudaGetLastError());
    CC_CUDA(c, cudaMemcpyAsync(c->h_counters, c->counters.p + 9, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                               c->stream));
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    const int64_t k = (int64_t)c->h_counters[0];
    std::vector<uint32_t> h((size_t)k);
    if (k > 0) {
        CC_CUDA(c, cudaMemcpyAsync(h.data(), c->scratch_u32.p, (size_t)k * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                                   c->stream));
        CC_CUDA(c, cudaStreamSynchronize(c->stream));
    }
    std::sort(h.begin(), h.end(), [](uint32_t a, uint32_t b) { return a > b; });
    for (int64_t q = 0; q < k && q < cap; q++) sizes_h[q] = h[(size_t)q];
    *n_h = k;
    return CC_OK;
}

}  // namespace cc
