// api.cu -- the C ABI of libcc (include/cc.h): context, S0 parameters, step orchestration,
// memory management and profiling.  Host C++; every step of the path runs in the kernels of
// bin.cu / scan.cu / pairs.cu / pgd.cu / fof.cu.  No CPU fallback exists.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "cc_internal.cuh"

// ------------------------------------------------------------------------------------------
cc_status cc_fail(cc_ctx* c, cc_status st, const std::string& msg) {
    if (c) c->err = msg;
    return st;
}

cc_status cc_cuda_check(cc_ctx* c, cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        return cc_fail(c, CC_E_OOM, std::string("out of device memory: ") + what);
    }
    if (c) c->dead = true;
    return cc_fail(c, CC_E_CUDA, std::string(cudaGetErrorString(e)) + " at " + what);
}

// scratch memory: the caller's allocator when cc_params supplies one (e.g. torch's caching
// allocator, bound to the context's stream by the caller), else stream-ordered cudaMallocAsync
static void scratch_free(cc_ctx* c, void* p) {
    if (!p) return;
    if (c->p.free_fn) c->p.free_fn(p, c->p.alloc_user);
    else cudaFreeAsync(p, c->stream);
}

template <typename T>
cc_status cc_ensure(cc_ctx* c, cc::DBuf<T>& b, size_t n, const char* name) {
    if (n == 0) n = 1;
    if (b.cap >= n) return CC_OK;
    if (b.p) {
        scratch_free(c, b.p);
        b.p = nullptr;
        b.cap = 0;
    }
    void* p = nullptr;
    if (c->p.alloc_fn) {
        p = c->p.alloc_fn(n * sizeof(T), c->p.alloc_user);
        if (!p)
            return cc_fail(c, CC_E_OOM, std::string("allocator callback failed for ") + name + " (" +
                                            std::to_string(n * sizeof(T)) + " bytes)");
        b.p = static_cast<T*>(p);
        b.cap = n;
        return CC_OK;
    }
    cudaError_t e = cudaMallocAsync(&p, n * sizeof(T), c->stream);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return cc_fail(c, CC_E_OOM, std::string("cudaMallocAsync failed for ") + name + " (" +
                                        std::to_string(n * sizeof(T)) + " bytes)");
    }
    b.p = static_cast<T*>(p);
    b.cap = n;
    return CC_OK;
}

template <typename T>
void cc_release(cc_ctx* c, cc::DBuf<T>& b) {
    if (b.p) scratch_free(c, b.p);
    b.p = nullptr;
    b.cap = 0;
}

#define CC_INST(T)                                                                 \
    template cc_status cc_ensure<T>(cc_ctx*, cc::DBuf<T>&, size_t, const char*); \
    template void cc_release<T>(cc_ctx*, cc::DBuf<T>&);
CC_INST(float4)
CC_INST(uint32_t)
CC_INST(uint64_t)
CC_INST(float)
CC_INST(float2)
CC_INST(double)
CC_INST(unsigned long long)
CC_INST(cc::Ctl)
CC_INST(long long)
CC_INST(unsigned char)
CC_INST(uint2)
CC_INST(uint4)

unsigned long long* cc::work_counters(cc_ctx* c) {
    if (!c->k3work.p) {
        if (cc_ensure(c, c->k3work, 8, "work counters") != CC_OK) return nullptr;
        if (cudaMemsetAsync(c->k3work.p, 0, 8 * sizeof(unsigned long long), c->stream) != cudaSuccess) return nullptr;
    }
    return c->k3work.p;
}

// ------------------------------------------------------------------------------------------
// profiling
int cc_prof_begin(cc_ctx* c, const char* cls) {
    if (!c->p.profile) return -1;
    int k = -1;
    for (size_t i = 0; i < c->prof.size(); i++)
        if (c->prof[i].name == cls) k = (int)i;
    if (k < 0) {
        c->prof.push_back({cls, 0.0, 0});
        k = (int)c->prof.size() - 1;
    }
    cudaEvent_t a, b;
    if (c->ev_pool.size() >= 2) {
        a = c->ev_pool.back();
        c->ev_pool.pop_back();
        b = c->ev_pool.back();
        c->ev_pool.pop_back();
    } else {
        cudaEventCreate(&a);
        cudaEventCreate(&b);
    }
    cudaEventRecord(a, c->stream);
    c->pend.push_back({k, a, b});
    return (int)c->pend.size() - 1;
}

void cc_prof_end(cc_ctx* c, int token) {
    if (token < 0) return;
    cudaEventRecord(c->pend[(size_t)token].b, c->stream);
}

static void prof_drain(cc_ctx* c) {
    if (c->pend.empty()) return;
    cudaStreamSynchronize(c->stream);
    for (auto& pe : c->pend) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, pe.a, pe.b) == cudaSuccess) {
            c->prof[(size_t)pe.cls].ms += ms;
            c->prof[(size_t)pe.cls].launches += 1;
        }
        c->ev_pool.push_back(pe.a);
        c->ev_pool.push_back(pe.b);
    }
    c->pend.clear();
}

// ------------------------------------------------------------------------------------------
// S0 -- parameters (Alg. 1 lines 1-3 P:419-421; §III-B; readings R2-R8).
// Evaluated in x87 extended precision (64-bit significand) and rounded once to fp32; the
// -m "not gpu" / -m gpu tests compare every threshold with the paper's formulas evaluated in
// 60-digit decimals (tests/paper_s0.py), so this code is pinned independently of the oracle.
typedef long double ld;

static float f32_nearest(ld v) { return (float)v; }  // one rounding from the 64-bit significand

// largest fp32 <= v
static float f32_down(ld v) {
    float f = (float)v;
    while ((ld)f > v) f = std::nextafter(f, -INFINITY);
    return f;
}
// smallest fp32 >= v
static float f32_up(ld v) {
    float f = (float)v;
    while ((ld)f < v) f = std::nextafter(f, INFINITY);
    return f;
}

static cc_status derive_params(cc_ctx* c, int64_t n_total) {
    const cc_params& p = c->p;
    double b = p.b;
    if (!(b > 0)) {
        if (n_total <= 0) return cc_fail(c, CC_E_ARG, "b <= 0 and no particles to derive it from");
        b = p.eta * std::cbrt(p.box * p.box * p.box / (double)n_total);  // b = eta (V/N)^(1/3)
    }
    c->b = b;
    cc::Th& t = c->th;
    const ld sqrt3 = std::sqrt((ld)3);
    const ld B = (ld)b;
    t.xi_f = (float)p.xi;                                         // R6: the bound is fl32(xi)
    const ld X = (ld)t.xi_f;
    c->xi_d = (double)X;
    const ld two_m = std::ldexp((ld)1, p.m);
    t.xip_f = f32_down(X - X / two_m);                            // Alg. 1 l.2: xi' = xi (1 - 2^-m), rounded down (R8)
    const ld eps_q = (ld)2 * X / (two_m - (ld)1);                 // Alg. 1 l.1: eps_q = 2 xi / (2^m - 1)
    c->eps_q = (double)eps_q;
    const ld mu = (ld)2 * sqrt3 * eps_q;                          // Eq. 3 margin 2 sqrt3 eps_q
    c->mu = (double)mu;
    t.c_b = f32_nearest(B - mu);
    t.c_f = f32_nearest(B + mu);
    const ld half = (ld)2 * sqrt3 * X;                            // Alg. 1 l.3: band half-width 2 sqrt3 xi
    const ld edge_lo = B - half, edge_hi = B + half;
    t.lo2 = edge_lo > 0 ? f32_nearest(edge_lo * edge_lo) : -1.0f; // R2: (b - 2 sqrt3 xi, b + 2 sqrt3 xi]
    t.hi2 = f32_nearest(edge_hi * edge_hi);
    t.b2 = f32_nearest(B * B);                                    // R3: d <= b
    t.Lf = (float)p.box;
    t.hLf = f32_nearest((ld)p.box / 2);
    // largest fp32 s with sqrtf(s) <= c (host sqrtf is the correctly rounded IEEE square root,
    // the same as the device's __fsqrt_rn)
    auto sq_thr = [](float c) -> float {
        if (!(c > 0.0f)) return -1.0f;
        float s2 = c * c;
        while (std::sqrt(s2) > c) s2 = std::nextafter(s2, 0.0f);
        while (std::sqrt(std::nextafter(s2, INFINITY)) <= c) s2 = std::nextafter(s2, INFINITY);
        return s2;
    };
    t.sb2 = sq_thr(t.c_b);
    t.sf2 = sq_thr(t.c_f);
    t.periodic = p.periodic ? 1 : 0;

    // Proven-link shells (cc_internal.cuh Th): every pinned fp32 d2 lies within the relative
    // factors (1 -/+ u)^k of the exact squared distance of its fp32 operands (u = 2^-24; 5
    // roundings interior; 3 + an absolute u (L + 2 xi) per component where the minimum image
    // wrapped), and any position within xi_f of the original moves a distance by <= 2 sqrt3 xi_f.
    const ld u = std::ldexp((ld)1, -24), sl = (ld)1 - (ld)1e-9;   // sl: slack for the ld arithmetic
    const ld b2 = (ld)t.b2, w = sqrt3 * u * ((ld)p.box + (ld)2 * X), dx = (ld)2 * sqrt3 * X;
    const ld up5 = std::pow((ld)1 + u, (ld)5), dn5 = std::pow((ld)1 - u, (ld)5);
    const ld up3 = std::pow((ld)1 + u, (ld)3), dn3 = std::pow((ld)1 - u, (ld)3);
    {
        const ld xi_ = std::sqrt(b2 / up5) - dx;                  // interior, stable
        t.lo2s_i = xi_ > 0 ? f32_down(dn5 * xi_ * xi_ * sl) : -1.0f;
        const ld yi_ = std::sqrt(b2 / dn5) + dx;                  // interior, never linked
        t.hi2s_i = f32_up(up5 * yi_ * yi_ / sl);
        const ld xw = ((ld)1 - u) * ((std::sqrt(b2 / up3) - w) / ((ld)1 + u) - dx) - w;
        t.lo2s_w = xw > 0 ? f32_down(dn3 * xw * xw * sl) : -1.0f;
        const ld yw = ((ld)1 + u) * ((std::sqrt(b2 / dn3) + w) / ((ld)1 - u) + dx) + w;
        t.hi2s_w = f32_up(up3 * yw * yw / sl);
        t.lo2s_i = std::min(t.lo2s_i, t.lo2);
        t.lo2s_w = std::min(t.lo2s_w, t.lo2);
        t.hi2s_i = std::max(t.hi2s_i, t.hi2);
        t.hi2s_w = std::max(t.hi2s_w, t.hi2);
    }
    // ghost / search radius: the largest exact original distance of a pair whose pinned d2 can
    // be <= hi2s_w (vulnerable, near shell, or linked in any position set within xi_f):
    // |A| <= (sqrt(d2 / (1-u)^3) + w) / (1-u); never below b + 2 sqrt3 xi
    c->delta = (double)std::max(edge_hi, (std::sqrt((ld)t.hi2s_w / dn3) + w) / ((ld)1 - u));
    c->r_pair = c->delta * (1.0 + 1e-9);
    // FoF on the original positions: d2 <= b2
    c->r_link = (double)((std::sqrt(b2 / dn3) + w) / ((ld)1 - u)) * (1.0 + 1e-9);
    if (p.periodic && c->delta >= 0.5 * p.box)
        return cc_fail(c, CC_E_ARG, "b + 2 sqrt3 xi must be < box/2 for minimum-image distances");
    return CC_OK;
}

// Search structure (cc_internal.cuh "x-sorted rows"): rows of side >= r_pair = delta (1 + 1e-5)
// in y and z (the margin covers fp32 rounding of d2 and of the coordinates), at most ~N rows;
// each row cut into x-bins of width >= 2 r_pair with at most K * N cells in total (perf knob,
// R25).  FoF on the original positions searches radius r_link = b (1 + 1e-5).
static void choose_grid(cc_ctx* c, int64_t n_local, double x_extent, double x0, int xwrap) {
    const double L = c->p.box;
    const double K = c->p.cells_per_particle > 0 ? c->p.cells_per_particle : 0.03;
    const double nl = (double)std::max<int64_t>(n_local, 1);
    int64_t nyz = std::max<int64_t>(1, (int64_t)std::floor(L / c->r_pair));
    while (nyz > 1 && (double)nyz * (double)nyz > std::max(nl, 9.0)) nyz = std::max<int64_t>(1, (int64_t)(nyz * 0.97));
    const double rows = (double)nyz * (double)nyz;
    int64_t nx_max = std::max<int64_t>(1, (int64_t)std::floor(x_extent / (2.0 * c->r_pair)));
    int64_t nx = std::max<int64_t>(1, (int64_t)std::floor(K * nl / rows));
    nx = std::min(nx, nx_max);
    while ((double)nx * rows > 2147483647.0 && nx > 1) nx /= 2;
    c->g.ny = c->g.nz = (int)nyz;
    c->g.nx = (int)nx;
    c->g.inv_w = (double)nyz / L;
    c->g.margin = 2.5 / c->g.inv_w;
    c->g.inv_wx = (double)nx / x_extent;
    c->g.x0 = x0;
    c->g.L = L;
    c->g.ext_x = x_extent;
    c->g.xwrap = xwrap;
    c->ncell = (int64_t)nx * nyz * nyz;
    // thread-per-cell insertion sort only where cells are tiny (K >= 1); crowded cells by a warp
    const double per_cell = nl / (double)c->ncell;
    c->bin_short_max = per_cell < 1.0 ? 16 : 1;
    if (const char* e = std::getenv("CC_BIN_SHORT")) c->bin_short_max = std::max(1, std::min(16, std::atoi(e)));
}

// ------------------------------------------------------------------------------------------
extern "C" {

void cc_default_params(cc_params* p) {
    std::memset(p, 0, sizeof(*p));
    p->box = 1.0;
    p->periodic = 1;
    p->b = 0.0;
    p->eta = 0.2;
    p->xi = 0.0;
    p->m = 16;
    p->alpha = 1e-3;
    p->beta1 = 0.9;
    p->beta2 = 0.999;
    p->eps_adam = 1e-8;
    p->t_max = 10000;
    p->eps_loss = 1e-10;
    p->stop_mode = CC_STOP_ACTIVE;
    p->optimizer = CC_OPT_ADAM;
    p->vanilla_step = 0.0;
    p->graph_batch = 16;
    p->cells_per_particle = 0.03;  // cells = rows of ~30 particles (measured: K1 37 vs 46 ms at C4)
    p->profile = 0;
    p->frontier = 1;
    p->alloc_fn = nullptr;
    p->free_fn = nullptr;
    p->alloc_user = nullptr;
}

cc_status cc_create(cc_ctx** out, int device, void* stream, const cc_params* p, const cc_dist* dist) {
    if (!out) return CC_E_ARG;
    *out = nullptr;
    if (!p) return CC_E_ARG;
    if (!(p->box > 0) || !(p->xi >= 0) || p->m < 2 || p->m > 52 || p->t_max < 0 || p->stop_mode < 0 ||
        p->stop_mode > 3 || p->optimizer < 0 || p->optimizer > 1)
        return CC_E_ARG;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0 || device < 0 || device >= ndev) {
        cudaGetLastError();
        return CC_E_CUDA;
    }
    if (dist && (dist->nranks < 1 || dist->rank < 0 || dist->rank >= dist->nranks)) return CC_E_ARG;
    if (dist && dist->nranks > 1 && !p->periodic) return CC_E_ARG;  // slabs are periodic in x
    cc_ctx* c = new cc_ctx();
    c->device = device;
    c->p = *p;
    if (cudaSetDevice(device) != cudaSuccess) {
        delete c;
        return CC_E_CUDA;
    }
    if (stream) {
        c->stream = static_cast<cudaStream_t>(stream);
    } else if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete c;
        return CC_E_CUDA;
    }
    // keep freed stream-ordered allocations cached in the pool
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    c->owns_stream = (stream == nullptr);
    if (cudaMallocHost(&c->h_ctl, sizeof(cc::Ctl)) != cudaSuccess ||
        cudaMallocHost(&c->h_counters, 16 * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMallocHost(&c->h_red, cc::LFX_STATS * sizeof(unsigned long long)) != cudaSuccess) {
        cc_destroy(c);
        return CC_E_CUDA;
    }
    if (dist && dist->nranks > 1) {
        cc_status st = cc::dist_init(c, dist);
        if (st != CC_OK) {
            cc_destroy(c);
            return st;
        }
    }
    *out = c;
    return CC_OK;
}

void cc_destroy(cc_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cc_release(c, c->orig4); cc_release(c, c->dec4); cc_release(c, c->cor4); cc_release(c, c->posA);
    cc_release(c, c->posB); cc_release(c, c->origE); cc_release(c, c->xk);
    cc_release(c, c->key); cc_release(c, c->rnk); cc_release(c, c->cell_count); cc_release(c, c->cell_start);
    cc_release(c, c->slot_of); cc_release(c, c->deg); cc_release(c, c->eidx); cc_release(c, c->rows);
    cc_release(c, c->slotE); cc_release(c, c->parent); cc_release(c, c->mingid); cc_release(c, c->gsize);
    cc_release(c, c->scratch_u32); cc_release(c, c->rowptr); cc_release(c, c->scratch_u64);
    cc_release(c, c->mom); cc_release(c, c->bc); 
    cc_release(c, c->counters); cc_release(c, c->ctl); cc_release(c, c->trace_a); cc_release(c, c->trace_l);
    cc_release(c, c->trace_v); cc_release(c, c->trace_s); cc_release(c, c->parent_base); cc_release(c, c->rec32);
    cc_release(c, c->frozen); cc_release(c, c->fbits); cc_release(c, c->lab_s); cc_release(c, c->slist); cc_release(c, c->tlist); cc_release(c, c->k3work);
    cc_release(c, c->tmp_bytes); cc_release(c, c->codec_bsum); cc_release(c, c->in_f); cc_release(c, c->in_gid);
    for (int d = 0; d < 2; d++) {
        cc_release(c, c->dflag[d]); cc_release(c, c->dpos[d]); cc_release(c, c->shell[d]); cc_release(c, c->sbuf7[d]);
        cc_release(c, c->rbuf7[d]); cc_release(c, c->req[d]); cc_release(c, c->recv_e[d]); cc_release(c, c->sreq[d]);
        cc_release(c, c->send_e[d]); cc_release(c, c->lsb[d]); cc_release(c, c->lrb[d]); cc_release(c, c->rsb[d]);
        cc_release(c, c->rrb[d]);
    }
    cc_release(c, c->stage); cc_release(c, c->gath); cc_release(c, c->dcnt); cc_release(c, c->red); cc_release(c, c->red_sum);
    cc_release(c, c->bnd); cc_release(c, c->near); cc_release(c, c->near_n); cc_release(c, c->gp_cnt); cc_release(c, c->gp_pos); cc_release(c, c->codec_status);
    cudaStreamSynchronize(c->stream);
    // the PGD graph holds NCCL work (multi-GPU): release it before the communicator
    if (c->pgd_exec) cudaGraphExecDestroy(c->pgd_exec);
    c->pgd_exec = nullptr;
    cudaDeviceSynchronize();
    cc::dist_destroy(c);
    if (c->h_red) cudaFreeHost(c->h_red);
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    for (auto& pe : c->pend) {
        cudaEventDestroy(pe.a);
        cudaEventDestroy(pe.b);
    }
    for (auto e : c->graph_ev) cudaEventDestroy(e);
    if (c->h_ctl) cudaFreeHost(c->h_ctl);
    if (c->h_counters) cudaFreeHost(c->h_counters);
    if (c->owns_stream) cudaStreamDestroy(c->stream);
    delete c;
}

const char* cc_last_error(const cc_ctx* c) { return c ? c->err.c_str() : "null context"; }

cc_status cc_nccl_unique_id(void* id) {
    if (!id) return CC_E_ARG;
    return cc::dist_unique_id(id);
}

#define CC_GUARD(c)                                                                          \
    do {                                                                                     \
        if (!(c)) return CC_E_ARG;                                                           \
        if ((c)->dead) return cc_fail((c), CC_E_CUDA, "context unusable after a CUDA error"); \
        cudaSetDevice((c)->device);                                                          \
    } while (0)

cc_status cc_build_cells(cc_ctx* c, int64_t n, const float* x, const float* y, const float* z, const float* xh,
                         const float* yh, const float* zh, const uint32_t* gid) {
    CC_GUARD(c);
    if (n < 0) return cc_fail(c, CC_E_ARG, "n < 0");
    if (n > 0 && (!x || !y || !z || !xh || !yh || !zh)) return cc_fail(c, CC_E_ARG, "null input pointer");
    if (n >= cc::MAX_LOCAL) return cc_fail(c, CC_E_DATA, "n beyond the 2^30 local index space");
    c->state = 0;
    c->have_labels[0] = c->have_labels[1] = c->have_labels[2] = 0;
    c->fof_which = -1;
    c->base_valid = false;
    int64_t n_total = n;
    if (c->nranks > 1) {
        if (n > 0 && !gid) return cc_fail(c, CC_E_ARG, "multi-GPU needs global particle ids (gid)");
        CC_TRY(cc_ensure(c, c->counters, 16, "counters"));
        c->h_counters[7] = (unsigned long long)n;
        CC_CUDA(c, cudaMemcpyAsync(c->counters.p + 7, c->h_counters + 7, sizeof(unsigned long long),
                                   cudaMemcpyHostToDevice, c->stream));
        CC_TRY(cc::dist_allreduce_u64(c, c->counters.p + 7, 1));
        CC_CUDA(c, cudaMemcpyAsync(c->h_counters + 7, c->counters.p + 7, sizeof(unsigned long long),
                                   cudaMemcpyDeviceToHost, c->stream));
        CC_CUDA(c, cudaStreamSynchronize(c->stream));
        n_total = (int64_t)c->h_counters[7];
    }
    CC_TRY(derive_params(c, n_total));
    c->n_in = n;
    c->n = n;
    if (c->nranks > 1) {
        const double slab = c->slab_hi - c->slab_lo;
        if (slab < 2.0 * c->r_pair)
            return cc_fail(c, CC_E_ARG, "x slab narrower than two ghost widths (b + 2 sqrt3 xi); use fewer GPUs");
        CC_TRY(cc::dist_exchange_ghosts(c, n, x, y, z, xh, yh, zh, gid));
        const double x0 = std::fmod(c->slab_lo - c->r_pair + c->p.box, c->p.box);
        choose_grid(c, c->n, slab + 2.0 * c->r_pair, x0, 0);
        // owned particles read in place, the ghosts from their 7-word staging (stride stage_cap)
        CC_TRY(cc::bin_particles(c, x, y, z, xh, yh, zh, gid, n, c->stage.p, c->stage_cap, c->n));
        c->in_dec[0] = xh;
        c->in_dec[1] = yh;
        c->in_dec[2] = zh;
    } else {
        choose_grid(c, n, c->p.box, 0.0, c->p.periodic ? 1 : 0);
        CC_TRY(cc::bin_particles(c, x, y, z, xh, yh, zh, gid, n, nullptr, 0, n));
        c->in_dec[0] = xh;
        c->in_dec[1] = yh;
        c->in_dec[2] = zh;
    }
    CC_CUDA(c, cudaMemcpyAsync(c->h_counters, c->counters.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                               c->stream));
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    const unsigned long long bad = c->h_counters[0];
    if (bad & 1ull) return cc_fail(c, CC_E_DATA, "non-finite input coordinate");
    if (bad & 2ull) return cc_fail(c, CC_E_BOUND, "decompressed input violates |x_hat - x| <= xi (P:396)");
    c->state = 1;
    return CC_OK;
}

cc_status cc_find_vulnerable(cc_ctx* c, cc_vp_info* info) {
    CC_GUARD(c);
    if (c->state < 1) return cc_fail(c, CC_E_STATE, "cc_build_cells first");
    const int64_t n = c->n;
    CC_TRY(cc::pairs_count(c));
    CC_TRY(cc_ensure(c, c->eidx, (size_t)std::max<int64_t>(n, 1), "eidx"));
    CC_TRY(cc_ensure(c, c->counters, 16, "counters"));
    CC_TRY(cc_ensure(c, c->key, (size_t)std::max<int64_t>(n, 1), "editable list"));  // key is dead after K1
    // S3: the editable list (slots with deg != 0, one pass over deg), then the class scan over it
    int64_t e_all = 0;
    CC_TRY(cc::editable_list(c, &e_all));
    if (e_all >= cc::MAX_LOCAL) return cc_fail(c, CC_E_DATA, "editable set beyond the 2^30 index space");
    const size_t e1 = (size_t)std::max<int64_t>(e_all, 1);
    CC_TRY(cc_ensure(c, c->slotE, e1, "slotE"));
    CC_TRY(cc_ensure(c, c->rowptr, e1 + 1, "rowptr"));
    CC_TRY(cc_ensure(c, c->origE, e1, "origE"));
    CC_TRY(cc_ensure(c, c->posA, e1, "posA"));
    CC_TRY(cc_ensure(c, c->posB, e1, "posB"));
    unsigned long long* tot = c->counters.p + 2;  // 56-byte VDeg total at counters[2..8]
    CC_TRY(cc::scan_editables(c, e_all, tot));
    CC_CUDA(c, cudaMemcpyAsync(c->h_counters + 2, tot, 7 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                               c->stream));
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    unsigned long long totals[7];
    std::memcpy(totals, c->h_counters + 2, sizeof(totals));
    CC_TRY(cc::rows_resolve(c, totals));
    if (c->E_all != e_all) return cc_fail(c, CC_E_DATA, "editable list and class scan disagree");
    CC_TRY(cc::rows_finish(c));
    if (c->nranks > 1) CC_TRY(cc::dist_setup_refresh(c));
    c->state = 2;
    if (info) {
        unsigned long long* cnt = c->counters.p + 4;
        CC_TRY(cc::mcc_run(c, CC_DECOMP, cnt));
        c->h_counters[8] = (unsigned long long)c->E;
        CC_CUDA(c, cudaMemcpyAsync(c->counters.p + 8, c->h_counters + 8, sizeof(unsigned long long),
                                   cudaMemcpyHostToDevice, c->stream));
        CC_TRY(cc::dist_allreduce_u64(c, cnt, 5));  // tp, tn, fp, fn, |E| summed over ranks
        CC_CUDA(c, cudaMemcpyAsync(c->h_counters + 4, cnt, 5 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                   c->stream));
        CC_CUDA(c, cudaStreamSynchronize(c->stream));
        const unsigned long long* h = c->h_counters + 4;
        info->n_pairs = (int64_t)(h[0] + h[1] + h[2] + h[3]);
        info->n_editable = (int64_t)h[4];
        info->n_linked = (int64_t)(h[0] + h[3]);
        info->n_violated0 = (int64_t)(h[2] + h[3]);
        info->n_local = c->n;
        info->cells_per_axis = c->g.ny;
        info->b = c->b;
    }
    return CC_OK;
}

cc_status cc_get_pairs(cc_ctx* c, uint32_t* gi, uint32_t* gj, uint8_t* flags, int64_t cap, int64_t* n_out) {
    CC_GUARD(c);
    if (c->state < 2) return cc_fail(c, CC_E_STATE, "cc_find_vulnerable first");
    if (cap > 0 && (!gi || !gj || !flags)) return cc_fail(c, CC_E_ARG, "null output");
    unsigned long long* cnt = c->counters.p + 10;
    CC_TRY(cc::get_pairs_run(c, gi, gj, flags, cap, cnt));
    CC_CUDA(c, cudaMemcpyAsync(c->h_counters + 10, cnt, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    if (n_out) *n_out = (int64_t)c->h_counters[10];
    return CC_OK;
}

cc_status cc_correct(cc_ctx* c, float* xo, float* yo, float* zo, cc_corr_info* info) {
    CC_GUARD(c);
    if (c->state < 2) return cc_fail(c, CC_E_STATE, "cc_find_vulnerable first");
    if (c->n_in > 0 && (!xo || !yo || !zo)) return cc_fail(c, CC_E_ARG, "null output");
    if (c->p.optimizer == CC_OPT_VANILLA && !(c->p.vanilla_step > 0))
        return cc_fail(c, CC_E_ARG, "vanilla optimizer needs vanilla_step > 0");
    cc_corr_info local{};
    CC_TRY(cc::pgd_run(c, &local));
    CC_TRY(cc::write_output(c, cc::pgd_result(c), xo, yo, zo));
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    c->state = 3;
    c->have_labels[CC_CORR] = 0;
    if (info) *info = local;
    return local.converged ? CC_OK : CC_NOT_CONVERGED;
}

cc_status cc_get_thresholds(cc_ctx* c, cc_thresholds* out) {
    CC_GUARD(c);
    if (!out) return cc_fail(c, CC_E_ARG, "null output");
    if (c->state < 1) return cc_fail(c, CC_E_STATE, "cc_build_cells first");
    const cc::Th& t = c->th;
    std::memset(out, 0, sizeof(*out));
    out->xi_f = t.xi_f; out->xip_f = t.xip_f; out->b2 = t.b2; out->lo2 = t.lo2; out->hi2 = t.hi2;
    out->c_b = t.c_b; out->c_f = t.c_f; out->Lf = t.Lf; out->hLf = t.hLf;
    out->lo2s_i = t.lo2s_i; out->hi2s_i = t.hi2s_i; out->lo2s_w = t.lo2s_w; out->hi2s_w = t.hi2s_w;
    out->b = c->b; out->eps_q = c->eps_q; out->mu = c->mu; out->r_search = c->r_pair; out->r_link = c->r_link;
    out->near_pairs = (c->state >= 2 && c->base_valid) ? c->near_count : -1;
    return CC_OK;
}

cc_status cc_get_schedule(cc_ctx* c, int64_t* sched_h, int64_t cap, int64_t* n_h) {
    CC_GUARD(c);
    if (c->state < 3) return cc_fail(c, CC_E_STATE, "cc_correct first");
    if (cap > 0 && !sched_h) return cc_fail(c, CC_E_ARG, "null output");
    const int64_t n = std::min<int64_t>((int64_t)c->last_iters, (int64_t)c->p.t_max);
    const int64_t k = std::min(n, cap);
    if (k > 0) {
        CC_CUDA(c, cudaMemcpyAsync(sched_h, c->trace_s.p, (size_t)(6 * k) * sizeof(long long), cudaMemcpyDeviceToHost,
                                   c->stream));
        CC_CUDA(c, cudaStreamSynchronize(c->stream));
    }
    if (n_h) *n_h = n;
    return CC_OK;
}

cc_status cc_get_trace(cc_ctx* c, int64_t* active_h, double* loss_h, int64_t* viol_h, int64_t cap, int64_t* n_h) {
    CC_GUARD(c);
    if (c->state < 3) return cc_fail(c, CC_E_STATE, "cc_correct first");
    if (cap > 0 && (!active_h || !loss_h)) return cc_fail(c, CC_E_ARG, "null output");
    const int64_t n = (int64_t)c->last_iters + 1;
    // trace[t-1] holds the stop check of iteration t; checks ran for t = 1..iters+1 unless the
    // loop ended on T_max (then the last state was checked by the final pass only)
    std::vector<long long> a((size_t)n, 0), v((size_t)n, 0);
    std::vector<double> l((size_t)n, 0.0);
    const int64_t k = std::min<int64_t>(n, (int64_t)c->p.t_max);
    if (k > 0) {
        CC_CUDA(c, cudaMemcpyAsync(a.data(), c->trace_a.p, (size_t)k * sizeof(long long), cudaMemcpyDeviceToHost,
                                   c->stream));
        CC_CUDA(c, cudaMemcpyAsync(l.data(), c->trace_l.p, (size_t)k * sizeof(double), cudaMemcpyDeviceToHost,
                                   c->stream));
        CC_CUDA(c, cudaMemcpyAsync(v.data(), c->trace_v.p, (size_t)k * sizeof(long long), cudaMemcpyDeviceToHost,
                                   c->stream));
    }
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    a[(size_t)n - 1] = (long long)c->final_active;  // final (global) check of the returned state
    l[(size_t)n - 1] = c->final_loss;
    v[(size_t)n - 1] = (long long)c->final_violated;
    for (int64_t q = 0; q < n && q < cap; q++) {
        active_h[q] = a[(size_t)q];
        loss_h[q] = l[(size_t)q];
        if (viol_h) viol_h[q] = v[(size_t)q];
    }
    if (n_h) *n_h = n;
    return CC_OK;
}

cc_status cc_fof_label(cc_ctx* c, int which, uint32_t* labels, int64_t* n_groups) {
    CC_GUARD(c);
    if (which < CC_ORIG || which > CC_CORR) return cc_fail(c, CC_E_ARG, "which");
    if (c->state < 1) return cc_fail(c, CC_E_STATE, "cc_build_cells first");
    if (which == CC_CORR && c->state < 3) return cc_fail(c, CC_E_STATE, "cc_correct first");
    int64_t ng = 0;
    CC_TRY(cc::fof_run(c, which, labels, n_groups ? &ng : nullptr));
    if (n_groups) *n_groups = ng;
    c->fof_which = which;
    return CC_OK;
}

cc_status cc_mcc(cc_ctx* c, int which, cc_mcc_info* out) {
    CC_GUARD(c);
    if (!out) return cc_fail(c, CC_E_ARG, "null output");
    if (c->state < 2) return cc_fail(c, CC_E_STATE, "cc_find_vulnerable first");
    if (which == CC_CORR && c->state < 3) return cc_fail(c, CC_E_STATE, "cc_correct first");
    unsigned long long* cnt = c->counters.p + 4;
    CC_TRY(cc::mcc_run(c, which, cnt));
    CC_TRY(cc::dist_allreduce_u64(c, cnt, 4));  // owned pairs summed over ranks (R17)
    CC_CUDA(c, cudaMemcpyAsync(c->h_counters + 4, cnt, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                               c->stream));
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    const unsigned long long* h = c->h_counters + 4;
    out->tp = h[0];
    out->tn = h[1];
    out->fp = h[2];
    out->fn = h[3];
    // MCC with R21's convention; numerator exact in 128-bit integers
    const unsigned __int128 a = (unsigned __int128)(h[0] + h[2]), b = (unsigned __int128)(h[0] + h[3]),
                            cc_ = (unsigned __int128)(h[1] + h[2]), d = (unsigned __int128)(h[1] + h[3]);
    if (a == 0 || b == 0 || cc_ == 0 || d == 0) {
        out->mcc = (h[2] == 0 && h[3] == 0) ? 1.0 : 0.0;
    } else {
        const __int128 num = (__int128)h[0] * (__int128)h[1] - (__int128)h[2] * (__int128)h[3];
        const unsigned __int128 den2 = a * b * cc_ * d;
        out->mcc = (double)num / std::sqrt((double)den2);
    }
    return CC_OK;
}

cc_status cc_halo_sizes(cc_ctx* c, int which, int64_t min_size, int64_t* sizes_h, int64_t cap, int64_t* n_h) {
    CC_GUARD(c);
    if (!n_h || (cap > 0 && !sizes_h)) return cc_fail(c, CC_E_ARG, "null output");
    if (c->fof_which != which) return cc_fail(c, CC_E_STATE, "cc_fof_label(which) must be the last FoF run");
    if (c->nranks > 1) {
        std::vector<uint32_t> v;
        CC_TRY(cc::dist_halo_sizes(c, min_size, v));
        for (size_t q = 0; q < v.size() && (int64_t)q < cap; q++) sizes_h[q] = v[q];
        *n_h = (int64_t)v.size();
        return CC_OK;
    }
    return cc::halo_sizes_run(c, min_size, sizes_h, cap, n_h);
}

cc_status cc_hmf(const int64_t* sizes, int64_t n, double vol, int n_bins, double lo, double hi, double* edges,
                 double* density) {
    if (n < 0 || n_bins <= 0 || !(vol > 0) || !edges || !density || (n > 0 && !sizes)) return CC_E_ARG;
    std::vector<double> lm((size_t)n);
    double mn = INFINITY, mx = -INFINITY;
    for (int64_t i = 0; i < n; i++) {
        lm[(size_t)i] = std::log10((double)sizes[i]);  // M_i = N_i (unit particle mass)
        mn = std::min(mn, lm[(size_t)i]);
        mx = std::max(mx, lm[(size_t)i]);
    }
    if (!(lo < hi)) {
        lo = n > 0 ? mn : 0.0;
        hi = n > 0 ? mx : 1.0;
        if (!(hi > lo)) hi = lo + 1.0;
    }
    const double w = (hi - lo) / n_bins;
    for (int k = 0; k <= n_bins; k++) edges[k] = lo + w * k;
    std::vector<double> cnt((size_t)n_bins, 0.0);
    for (int64_t i = 0; i < n; i++) {
        const double v = lm[(size_t)i];
        int64_t k = (int64_t)std::floor((v - lo) / w);
        if (v == hi) k = n_bins - 1;
        if (k >= 0 && k < n_bins) cnt[(size_t)k] += 1.0;
    }
    for (int k = 0; k < n_bins; k++) density[k] = cnt[(size_t)k] / (vol * w);
    return CC_OK;
}

cc_status cc_kernel_stats(cc_ctx* c, char* names, int64_t names_cap, double* ms, int64_t* launches, int64_t cap,
                          int64_t* n_h, int reset) {
    CC_GUARD(c);
    prof_drain(c);
    std::string all;
    int64_t k = 0;
    for (auto& pe : c->prof) {
        if (k < cap) {
            if (ms) ms[k] = pe.ms;
            if (launches) launches[k] = pe.launches;
        }
        all += pe.name;
        all += '\n';
        k++;
    }
    // pseudo-class: every kernel launched through this context (profiled or not)
    if (k < cap) {
        if (ms) ms[k] = 0.0;
        if (launches) launches[k] = c->launches;
    }
    all += "total_launches\n";
    k++;
    // pseudo-classes: K3 work actually done (the frontier skips frozen particles)
    unsigned long long wk[5] = {0, 0, 0, 0, 0};
    if (c->k3work.p) {
        CC_CUDA(c, cudaMemcpyAsync(wk, c->k3work.p, sizeof(wk), cudaMemcpyDeviceToHost, c->stream));
        CC_CUDA(c, cudaStreamSynchronize(c->stream));
        if (reset) CC_CUDA(c, cudaMemsetAsync(c->k3work.p, 0, sizeof(wk), c->stream));
    }
    const char* wn[5] = {"K3_work_editables\n", "K3_work_entries\n", "K2_count_tests\n", "K2_fill_tests\n",
                         "K4_link_tests\n"};
    for (int q = 0; q < 5; q++) {
        if (k < cap) {
            if (ms) ms[k] = 0.0;
            if (launches) launches[k] = (int64_t)wk[q];
        }
        all += wn[q];
        k++;
    }
    if (names && names_cap > 0) {
        std::strncpy(names, all.c_str(), (size_t)names_cap - 1);
        names[names_cap - 1] = 0;
    }
    if (n_h) *n_h = k;
    if (reset) {
        for (auto& pe : c->prof) {
            pe.ms = 0;
            pe.launches = 0;
        }
        c->launches = 0;
    }
    return CC_OK;
}

cc_status cc_run(cc_ctx* c, int64_t n, const float* x, const float* y, const float* z, const float* xh,
                 const float* yh, const float* zh, const uint32_t* gid, float* xo, float* yo, float* zo, int flags,
                 cc_run_info* info) {
    CC_GUARD(c);
    if (n < 0) return cc_fail(c, CC_E_ARG, "n < 0");
    const float *dx = x, *dy = y, *dz = z, *dxh = xh, *dyh = yh, *dzh = zh;
    const uint32_t* dg = gid;
    float *ox = xo, *oy = yo, *oz = zo;
    const size_t nn = (size_t)std::max<int64_t>(n, 1);
    if (flags & CC_RUN_HOST) {
        CC_TRY(cc_ensure(c, c->in_f, 9 * nn, "run staging"));
        float* s = c->in_f.p;
        const float* src[6] = {x, y, z, xh, yh, zh};
        for (int k = 0; k < 6; k++)
            if (n > 0)
                CC_CUDA(c, cudaMemcpyAsync(s + k * nn, src[k], (size_t)n * sizeof(float), cudaMemcpyHostToDevice,
                                           c->stream));
        dx = s; dy = s + nn; dz = s + 2 * nn; dxh = s + 3 * nn; dyh = s + 4 * nn; dzh = s + 5 * nn;
        ox = s + 6 * nn; oy = s + 7 * nn; oz = s + 8 * nn;
        if (gid) {
            CC_TRY(cc_ensure(c, c->in_gid, nn, "run gid staging"));
            if (n > 0)
                CC_CUDA(c, cudaMemcpyAsync(c->in_gid.p, gid, (size_t)n * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                           c->stream));
            dg = c->in_gid.p;
        }
    }
    CC_TRY(cc_build_cells(c, n, dx, dy, dz, dxh, dyh, dzh, dg));
    cc_run_info loc{};
    CC_TRY(cc_find_vulnerable(c, &loc.vp));
    cc_status st = cc_correct(c, ox, oy, oz, &loc.corr);
    if (st != CC_OK && st != CC_NOT_CONVERGED) return st;
    if ((flags & CC_RUN_HOST) && n > 0) {
        CC_CUDA(c, cudaMemcpyAsync(xo, ox, (size_t)n * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
        CC_CUDA(c, cudaMemcpyAsync(yo, oy, (size_t)n * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
        CC_CUDA(c, cudaMemcpyAsync(zo, oz, (size_t)n * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
        CC_CUDA(c, cudaStreamSynchronize(c->stream));
    }
    if (info) *info = loc;
    return st;
}

}  // extern "C"
