// pgd.cu -- K3, the fused PGD iteration (S4) with a device-side stop (S5).
//
// Paper: Alg. 1 lines 4-10; §III-B P:444 (gradient step then box projection),
// P:448-451 (tightened loss L_tight, Eq. 3), P:458 (projection onto B(xi') around the original
// positions; Adam), §III-C P:465 (the paper's three kernels: per-pair loss with a shared-memory
// reduction, per-pair gradients accumulated with global atomics, per-particle Adam+projection).
//
// B200 form: ONE kernel per iteration, owner-computes: each editable particle walks its CSR row
// (partners sorted by gid, R14), evaluates every pair's L_tight activity, term and gradient
// contribution from the SAME position buffer, then applies Adam and the directed-rounding box
// projection (R8) and writes the other ping-pong buffer.  No gradient buffer, no atomics,
// bit-reproducible.  Short rows: one thread, partner loads issued in batches of 4 before the
// sequential accumulation (memory-level parallelism without changing the summation order).
// Long rows (> 32 entries, halo cores): one warp, lanes load and evaluate 32 entries at once and
// the gradient is then accumulated in row order through warp shuffles (again the pinned order).
// Each pair's counts/loss are taken at its lower-gid endpoint; block partials are reduced by the
// last block in a fixed order, which decides the stop: if the state this launch READ meets the
// stop rule (R11) the loop is over and the read buffer is the result (the speculative write is
// discarded).  Launches after that return at once: a CUDA graph of k launches needs one host
// poll per k iterations.
// Algorithmic bytes per launch: 104 B per editable (pos r/w 32, orig 16, m,v r/w 48, rowptr 8)
// + 4 B per directed row entry; partner positions are gathers (L2 when local).
#include <cmath>
#include <vector>

#include "cc_internal.cuh"

namespace cc {
namespace {

constexpr int PGD_THREADS = 256;
constexpr int PGD_MAX_BLOCKS = 148 * 8;
constexpr int LONG_ROW = 32;  // rows longer than this take the warp path (rows_finish's long list)
constexpr int BATCH = 4;

struct PgdArgs {
    uint32_t E;  // editable particles with rows (owned)
    const unsigned long long* __restrict__ rowptr;
    const uint32_t* __restrict__ rows;
    const float4* __restrict__ origE;
    const uint32_t* __restrict__ long_list;
    uint32_t n_long;
    float4* pos0;
    float4* pos1;
    float* __restrict__ mom;  // 6 x E SoA
    const float2* __restrict__ bc;
    Th t;
    float alpha, b1, b2, omb1, omb2, eps, vstep;
    int optimizer;
    int t_max;
    int stop_mode;
    double eps_loss;
    Ctl* ctl;
    unsigned long long* part_u;  // 2 per block: active, violated
    double* part_d;
    long long* trace_a;
    double* trace_l;
    long long* trace_v;
    int count_only;
    double* red;  // multi-GPU: local (active, loss, violated) for the allreduce, else nullptr
};

// one pair term, pinned (R4, R13, R14, R15): r = minimg(p - q), d_hat = sqrt_rn(r.r);
// kind 0: inactive, 1: add (px,py,pz) to the gradient, 2: coincident -> add px to g.x only
struct Term {
    float px, py, pz;
    float ee;
    int kind;
    bool viol;
};

__device__ __forceinline__ Term pair_term(const float4& p, const float4& q, uint32_t ent, const Th& th) {
    Term o;
    const float rx = min_image(__fsub_rn(p.x, q.x), th);
    const float ry = min_image(__fsub_rn(p.y, q.y), th);
    const float rz = min_image(__fsub_rn(p.z, q.z), th);
    float s = __fmul_rn(rx, rx);
    s = __fadd_rn(s, __fmul_rn(ry, ry));
    s = __fadd_rn(s, __fmul_rn(rz, rz));
    const float d = __fsqrt_rn(s);
    const bool ol = (ent & ENT_OLINK) != 0;
    o.viol = (s <= th.b2) != ol;  // link status differs from the original (Eq. 1 support)
    // Eq. (3): broken side (orig linked) active iff d_hat > b - 2 sqrt3 eps_q;
    //          false side (orig unlinked) active iff d_hat <= b + 2 sqrt3 eps_q
    const bool act = ol ? (d > th.c_b) : (d <= th.c_f);
    o.kind = 0;
    o.ee = 0.0f;
    o.px = o.py = o.pz = 0.0f;
    if (act) {
        o.ee = __fsub_rn(d, ol ? th.c_b : th.c_f);
        const float two_e = __fmul_rn(2.0f, o.ee);
        if (d > 0.0f) {
            const float kk = __fdiv_rn(two_e, d);  // grad = 2 (d_hat - c) r / d_hat
            o.px = __fmul_rn(kk, rx);
            o.py = __fmul_rn(kk, ry);
            o.pz = __fmul_rn(kk, rz);
            o.kind = 1;
        } else {  // coincident: +x for the lower-gid endpoint (ENT_UPPER set), -x for the other
            o.px = (ent & ENT_UPPER) ? two_e : -two_e;
            o.kind = 2;
        }
    }
    return o;
}

__device__ __forceinline__ void accumulate(float& gx, float& gy, float& gz, const Term& tm) {
    if (tm.kind == 1) {
        gx = __fadd_rn(gx, tm.px);
        gy = __fadd_rn(gy, tm.py);
        gz = __fadd_rn(gz, tm.pz);
    } else if (tm.kind == 2) {
        gx = __fadd_rn(gx, tm.px);
    }
}

__device__ __forceinline__ float adam_coord(float x, float g, float* __restrict__ m, float* __restrict__ v,
                                            const PgdArgs& a, float bc1, float bc2) {
    const float mm = __fadd_rn(__fmul_rn(a.b1, *m), __fmul_rn(a.omb1, g));
    const float vv = __fadd_rn(__fmul_rn(a.b2, *v), __fmul_rn(a.omb2, __fmul_rn(g, g)));
    *m = mm;
    *v = vv;
    const float mh = __fdiv_rn(mm, bc1);
    const float vh = __fdiv_rn(vv, bc2);
    const float den = __fadd_rn(__fsqrt_rn(vh), a.eps);
    const float step = __fmul_rn(a.alpha, __fdiv_rn(mh, den));
    return __fsub_rn(x, step);
}

__device__ __forceinline__ float project(float x, float o, float xip) {
    const float lo = __fsub_ru(o, xip);
    const float hi = __fadd_rd(o, xip);
    if (x < lo) x = lo;
    if (x > hi) x = hi;
    return x;
}

// Adam (or vanilla) step + projection of editable e, written to dst
__device__ __forceinline__ void update(const PgdArgs& a, uint32_t e, const float4& p, float gx, float gy, float gz,
                                       float bc1, float bc2, float4* __restrict__ dst) {
    const float4 o = a.origE[e];
    float x = p.x, y = p.y, z = p.z;
    if (a.optimizer == CC_OPT_ADAM) {
        float* m = a.mom;
        const size_t E = a.E;
        x = adam_coord(x, gx, m + e, m + 3 * E + e, a, bc1, bc2);
        y = adam_coord(y, gy, m + E + e, m + 4 * E + e, a, bc1, bc2);
        z = adam_coord(z, gz, m + 2 * E + e, m + 5 * E + e, a, bc1, bc2);
    } else {
        x = __fsub_rn(x, __fmul_rn(a.vstep, gx));
        y = __fsub_rn(y, __fmul_rn(a.vstep, gy));
        z = __fsub_rn(z, __fmul_rn(a.vstep, gz));
    }
    x = project(x, o.x, a.t.xip_f);
    y = project(y, o.y, a.t.xip_f);
    z = project(z, o.z, a.t.xip_f);
    dst[e] = make_float4(x, y, z, p.w);
}

__global__ void __launch_bounds__(PGD_THREADS) k_pgd(PgdArgs a) {
    Ctl* ctl = a.ctl;
    if (!a.count_only && *((volatile int*)&ctl->done)) return;
    const int t = a.count_only ? 0 : ctl->t + 1;
    const float4* __restrict__ src;
    float4* __restrict__ dst;
    if (a.count_only) {
        src = (ctl->t_res & 1) ? a.pos1 : a.pos0;
        dst = nullptr;
    } else {
        src = ((t - 1) & 1) ? a.pos1 : a.pos0;
        dst = (t & 1) ? a.pos1 : a.pos0;
    }
    float bc1 = 1.0f, bc2 = 1.0f;
    if (!a.count_only && a.optimizer == CC_OPT_ADAM) {
        const float2 bcv = a.bc[t - 1];
        bc1 = bcv.x;
        bc2 = bcv.y;
    }
    const Th th = a.t;
    unsigned int cnt = 0, nviol = 0;
    double loss = 0.0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;

    // ---- long rows: one warp per row, 32 entries per round, row-order accumulation via shuffles
    const uint32_t gw = blockIdx.x * (PGD_THREADS / 32) + w, nw = gridDim.x * (PGD_THREADS / 32);
    for (uint32_t q = gw; q < a.n_long; q += nw) {
        const uint32_t e = a.long_list[q];
        const float4 p = src[e];
        const unsigned long long k0 = a.rowptr[e], k1 = a.rowptr[e + 1];
        float gx = 0.0f, gy = 0.0f, gz = 0.0f;
        for (unsigned long long kb = k0; kb < k1; kb += 32) {
            const unsigned long long k = kb + lane;
            Term tm;
            tm.kind = 0;
            if (k < k1) {
                const uint32_t ent = a.rows[k];
                tm = pair_term(p, src[ent & ENT_IDX], ent, th);
                if (ent & ENT_UPPER) {
                    if (tm.kind) {
                        cnt++;
                        loss += (double)tm.ee * (double)tm.ee;
                    }
                    nviol += tm.viol;
                }
            }
            const int m = (int)min((unsigned long long)32, k1 - kb);
            for (int i = 0; i < m; i++) {  // the pinned sequential order, identical on all lanes
                Term u;
                u.kind = __shfl_sync(0xffffffffu, tm.kind, i);
                u.px = __shfl_sync(0xffffffffu, tm.px, i);
                u.py = __shfl_sync(0xffffffffu, tm.py, i);
                u.pz = __shfl_sync(0xffffffffu, tm.pz, i);
                accumulate(gx, gy, gz, u);
            }
        }
        if (!a.count_only && lane == 0) update(a, e, p, gx, gy, gz, bc1, bc2, dst);
    }

    // ---- short rows: one thread each, partner loads batched ahead of the sequential sum
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < a.E; e += stride) {
        const unsigned long long k0 = a.rowptr[e], k1 = a.rowptr[e + 1];
        if (k1 - k0 > (unsigned long long)LONG_ROW) continue;  // warp path
        const float4 p = src[e];
        float gx = 0.0f, gy = 0.0f, gz = 0.0f;
        for (unsigned long long kb = k0; kb < k1; kb += BATCH) {
            uint32_t ent[BATCH];
            float4 qq[BATCH];
#pragma unroll
            for (int i = 0; i < BATCH; i++) ent[i] = (kb + i < k1) ? a.rows[kb + i] : 0u;
#pragma unroll
            for (int i = 0; i < BATCH; i++)
                if (kb + i < k1) qq[i] = src[ent[i] & ENT_IDX];
#pragma unroll
            for (int i = 0; i < BATCH; i++) {
                if (kb + i < k1) {
                    const Term tm = pair_term(p, qq[i], ent[i], th);
                    if (ent[i] & ENT_UPPER) {
                        if (tm.kind) {
                            cnt++;
                            loss += (double)tm.ee * (double)tm.ee;
                        }
                        nviol += tm.viol;
                    }
                    accumulate(gx, gy, gz, tm);
                }
            }
        }
        if (!a.count_only) update(a, e, p, gx, gy, gz, bc1, bc2, dst);
    }

    // ---- deterministic block reduction (fixed shuffle tree + fixed warp order)
    __shared__ unsigned long long sh_u[PGD_THREADS / 32], sh_v[PGD_THREADS / 32];
    __shared__ double sh_d[PGD_THREADS / 32];
    __shared__ bool am_last;
    unsigned long long cu = cnt, cv = nviol;
    for (int o = 16; o > 0; o >>= 1) {
        cu += __shfl_down_sync(0xffffffffu, cu, o);
        cv += __shfl_down_sync(0xffffffffu, cv, o);
        loss += __shfl_down_sync(0xffffffffu, loss, o);
    }
    if (lane == 0) {
        sh_u[w] = cu;
        sh_v[w] = cv;
        sh_d[w] = loss;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long bu = 0, bv = 0;
        double bd = 0.0;
        for (int k = 0; k < PGD_THREADS / 32; k++) {
            bu += sh_u[k];
            bv += sh_v[k];
            bd += sh_d[k];
        }
        a.part_u[2 * blockIdx.x] = bu;
        a.part_u[2 * blockIdx.x + 1] = bv;
        a.part_d[blockIdx.x] = bd;
        __threadfence();
        const unsigned int tk = atomicAdd(&ctl->ticket, 1u);
        am_last = (tk == gridDim.x - 1);
    }
    __syncthreads();
    if (!am_last) return;
    // last block: fixed-order sum of the block partials
    __threadfence();
    unsigned long long su = 0, sv = 0;
    double sd = 0.0;
    for (uint32_t b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
        su += ((volatile unsigned long long*)a.part_u)[2 * b];
        sv += ((volatile unsigned long long*)a.part_u)[2 * b + 1];
        sd += ((volatile double*)a.part_d)[b];
    }
    for (int o = 16; o > 0; o >>= 1) {
        su += __shfl_down_sync(0xffffffffu, su, o);
        sv += __shfl_down_sync(0xffffffffu, sv, o);
        sd += __shfl_down_sync(0xffffffffu, sd, o);
    }
    __syncthreads();
    if (lane == 0) {
        sh_u[w] = su;
        sh_v[w] = sv;
        sh_d[w] = sd;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long tu = 0, tv = 0;
        double td = 0.0;
        for (int k = 0; k < PGD_THREADS / 32; k++) {
            tu += sh_u[k];
            tv += sh_v[k];
            td += sh_d[k];
        }
        ctl->active = tu;
        ctl->violated = tv;
        ctl->loss = td;
        ctl->ticket = 0;
        if (a.red) {  // multi-GPU: the decision waits for the allreduce (dist.cu k_decide)
            a.red[0] = (double)tu;
            a.red[1] = td;
            a.red[2] = (double)tv;
        } else if (!a.count_only) {
            if (a.trace_a) {
                a.trace_a[t - 1] = (long long)tu;
                a.trace_l[t - 1] = td;
                a.trace_v[t - 1] = (long long)tv;
            }
            if (stop_rule(a.stop_mode, tu, td, tv, a.eps_loss)) {
                ctl->done = 1;
                ctl->t_res = t - 1;  // the state this launch read
                ctl->converged = 1;
            } else if (t >= a.t_max) {
                ctl->done = 1;
                ctl->t_res = t;      // the state this launch wrote
            }
            ctl->t = t;
        }
        __threadfence();
    }
}

__global__ void k_ctl_reset(Ctl* ctl) {
    ctl->done = 0;
    ctl->t = 0;
    ctl->t_res = 0;
    ctl->converged = 0;
    ctl->ticket = 0;
    ctl->active = 0;
    ctl->violated = 0;
    ctl->loss = 0.0;
}

__global__ void k_reset_pos(int64_t Ea, const uint32_t* __restrict__ slotE, const float4* __restrict__ dec4,
                            const float4* __restrict__ origE, float4* __restrict__ posA) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= Ea) return;
    const float4 d = dec4[slotE[e]];
    posA[e] = make_float4(d.x, d.y, d.z, origE[e].w);
}

// corrected positions in slot order: editable -> result buffer, others -> decompressed
__global__ void k_cor4(int64_t n, const float4* __restrict__ dec4, const uint32_t* __restrict__ eidx,
                       uint32_t e_own, const float4* __restrict__ res, float4* __restrict__ cor4) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const uint32_t e0 = eidx[s];
    float4 d = dec4[s];
    if (e0 != 0xFFFFFFFFu) {
        const uint32_t e = (e0 & 0x80000000u) ? e_own + (e0 & 0x7FFFFFFFu) : e0;
        const float4 r = res[e];
        d.x = r.x;
        d.y = r.y;
        d.z = r.z;
    }
    cor4[s] = d;
}

// outputs in input order (owned particles)
__global__ void k_output(int64_t n_in, const uint32_t* __restrict__ slot_of, const float4* __restrict__ cor4,
                         float* __restrict__ xo, float* __restrict__ yo, float* __restrict__ zo) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_in) return;
    const float4 v = cor4[slot_of[i]];
    xo[i] = v.x;
    yo[i] = v.y;
    zo[i] = v.z;
}

PgdArgs make_args(cc_ctx* c, int count_only) {
    PgdArgs a{};
    a.E = (uint32_t)c->E;
    a.rowptr = reinterpret_cast<const unsigned long long*>(c->rowptr.p);
    a.rows = c->rows.p;
    a.origE = c->origE.p;
    a.long_list = c->longrow.p;
    a.n_long = (uint32_t)c->n_long;
    a.pos0 = c->posA.p;
    a.pos1 = c->posB.p;
    a.mom = c->mom.p;
    a.bc = c->bc.p;
    a.t = c->th;
    a.alpha = (float)c->p.alpha;
    a.b1 = (float)c->p.beta1;
    a.b2 = (float)c->p.beta2;
    a.omb1 = (float)(1.0 - c->p.beta1);
    a.omb2 = (float)(1.0 - c->p.beta2);
    a.eps = (float)c->p.eps_adam;
    a.vstep = (float)c->p.vanilla_step;
    a.optimizer = c->p.optimizer;
    a.t_max = c->p.t_max;
    a.stop_mode = c->p.stop_mode;
    a.eps_loss = c->p.eps_loss;
    a.ctl = c->ctl.p;
    a.part_u = c->partial_u.p;
    a.part_d = c->partial_d.p;
    a.trace_a = c->trace_a.p;
    a.trace_l = c->trace_l.p;
    a.trace_v = c->trace_v.p;
    a.count_only = count_only;
    a.red = c->nranks > 1 ? c->red.p : nullptr;
    return a;
}

int pgd_blocks(int64_t E) {
    int64_t b = (E + PGD_THREADS - 1) / PGD_THREADS;
    if (b > PGD_MAX_BLOCKS) b = PGD_MAX_BLOCKS;
    if (b < 1) b = 1;
    return (int)b;
}

}  // namespace

const float4* pgd_result(cc_ctx* c) { return (c->last_iters & 1) ? c->posB.p : c->posA.p; }

// (active, loss, violated) of the count-only pass just enqueued, summed over ranks (synchronising)
static cc_status global_check(cc_ctx* c, double* al) {
    if (c->nranks > 1) {
        CC_TRY(dist_allreduce_f64(c, c->red.p, 3));
        CC_CUDA(c, cudaMemcpyAsync(c->h_red, c->red.p, 3 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CC_CUDA(c, cudaStreamSynchronize(c->stream));
        for (int k = 0; k < 3; k++) al[k] = c->h_red[k];
    } else {
        CC_CUDA(c, cudaMemcpyAsync(c->h_ctl, c->ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, c->stream));
        CC_CUDA(c, cudaStreamSynchronize(c->stream));
        al[0] = (double)c->h_ctl->active;
        al[1] = c->h_ctl->loss;
        al[2] = (double)c->h_ctl->violated;
    }
    return CC_OK;
}

cc_status pgd_run(cc_ctx* c, cc_corr_info* info) {
    const int64_t E = c->E, Ea = c->E_all;
    const int tmax = c->p.t_max;
    CC_TRY(cc_ensure(c, c->mom, (size_t)std::max<int64_t>(6 * E, 1), "adam moments"));
    CC_TRY(cc_ensure(c, c->bc, (size_t)std::max(tmax, 1), "bias corrections"));
    CC_TRY(cc_ensure(c, c->partial_u, 2 * PGD_MAX_BLOCKS, "partials"));
    CC_TRY(cc_ensure(c, c->partial_d, PGD_MAX_BLOCKS, "partials"));
    CC_TRY(cc_ensure(c, c->ctl, 1, "ctl"));
    CC_TRY(cc_ensure(c, c->trace_a, (size_t)tmax + 1, "trace"));
    CC_TRY(cc_ensure(c, c->trace_l, (size_t)tmax + 1, "trace"));
    CC_TRY(cc_ensure(c, c->trace_v, (size_t)tmax + 1, "trace"));
    if (c->nranks > 1) CC_TRY(cc_ensure(c, c->red, 4, "allreduce buffer"));
    // restart from P_hat^(0) (a previous cc_correct may have overwritten posA)
    if (Ea > 0)
        CCL(c, k_reset_pos<<<(unsigned)((Ea + 255) / 256), 256, 0, c->stream>>>(Ea, c->slotE.p, c->dec4.p,
                                                                                c->origE.p, c->posA.p));
    CC_CUDA(c, cudaMemsetAsync(c->mom.p, 0, (size_t)std::max<int64_t>(6 * E, 1) * sizeof(float), c->stream));
    if (Ea > E)  // ghost partner positions also live in posB (refreshed each iteration, multi-GPU)
        CC_CUDA(c, cudaMemcpyAsync(c->posB.p + E, c->posA.p + E, (size_t)(Ea - E) * sizeof(float4),
                                   cudaMemcpyDeviceToDevice, c->stream));
    // Adam bias corrections: beta^t as an fp64 running product (R9), rounded once
    {
        std::vector<float2> h((size_t)std::max(tmax, 1));
        double p1 = 1.0, p2 = 1.0;
        for (int t = 0; t < tmax; t++) {
            p1 = p1 * c->p.beta1;
            p2 = p2 * c->p.beta2;
            h[t] = make_float2((float)(1.0 - p1), (float)(1.0 - p2));
        }
        CC_CUDA(c, cudaMemcpyAsync(c->bc.p, h.data(), h.size() * sizeof(float2), cudaMemcpyHostToDevice, c->stream));
        CC_CUDA(c, cudaStreamSynchronize(c->stream));  // h goes out of scope
    }
    CCL(c, k_ctl_reset<<<1, 1, 0, c->stream>>>(c->ctl.p));
    const int nb = pgd_blocks(std::max<int64_t>(E, (int64_t)c->n_long * 32));
    const int batch = c->p.graph_batch > 0 ? c->p.graph_batch : 16;
    PgdArgs a = make_args(c, 0);
    // initial statistics of P_hat^(0) for the report
    PgdArgs a0 = make_args(c, 1);
    CCL(c, k_pgd<<<nb, PGD_THREADS, 0, c->stream>>>(a0));
    CC_CUDA(c, cudaGetLastError());
    {
        double al[3];
        CC_TRY(global_check(c, al));
        info->active0 = (int64_t)al[0];
        info->loss0 = al[1];
        info->violated0 = (int64_t)al[2];
    }
    CCL(c, k_ctl_reset<<<1, 1, 0, c->stream>>>(c->ctl.p));

    int iters = 0;
    if (tmax > 0) {
        // (re)capture a graph of `batch` iterations, each bracketed by event records
        const void* key[5] = {c->posA.p, c->rows.p, c->mom.p, c->ctl.p, c->longrow.p};
        bool same = c->pgd_exec && c->pgd_batch == batch && c->pgd_E == E && c->pgd_nlong == c->n_long;
        for (int k = 0; k < 5; k++) same = same && key[k] == c->pgd_key[k];
        if (!same) {
            if (c->pgd_exec) cudaGraphExecDestroy(c->pgd_exec);
            c->pgd_exec = nullptr;
            if (c->p.profile) {
                while ((int)c->graph_ev.size() < 2 * batch) {
                    cudaEvent_t ev;
                    CC_CUDA(c, cudaEventCreate(&ev));
                    c->graph_ev.push_back(ev);
                }
            }
            cudaGraph_t graph;
            CC_CUDA(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
            for (int k = 0; k < batch; k++) {
                if (c->p.profile) cudaEventRecordWithFlags(c->graph_ev[2 * k], c->stream, cudaEventRecordExternal);
                CCL(c, k_pgd<<<nb, PGD_THREADS, 0, c->stream>>>(a));
                if (c->p.profile)
                    cudaEventRecordWithFlags(c->graph_ev[2 * k + 1], c->stream, cudaEventRecordExternal);
                if (c->nranks > 1) {
                    const int64_t l0 = c->launches;
                    cc_status st = dist_iter_tail(c, c->posA.p, c->posB.p);
                    if (st != CC_OK) {
                        cudaGraph_t g2 = nullptr;
                        cudaStreamEndCapture(c->stream, &g2);
                        if (g2) cudaGraphDestroy(g2);
                        return st;
                    }
                    c->launches_per_iter_tail = c->launches - l0;
                    c->launches = l0;
                }
            }
            c->launches -= batch;  // captured, not launched
            cudaError_t ce = cudaStreamEndCapture(c->stream, &graph);
            CC_CUDA(c, ce);
            CC_CUDA(c, cudaGraphInstantiate(&c->pgd_exec, graph, 0));
            cudaGraphDestroy(graph);
            for (int k = 0; k < 5; k++) c->pgd_key[k] = key[k];
            c->pgd_batch = batch;
            c->pgd_E = E;
            c->pgd_nlong = c->n_long;
        }
        int t_before = 0;
        for (;;) {
            CC_CUDA(c, cudaGraphLaunch(c->pgd_exec, c->stream));
            c->launches += batch * (1 + c->launches_per_iter_tail);
            CC_CUDA(c, cudaMemcpyAsync(c->h_ctl, c->ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, c->stream));
            CC_CUDA(c, cudaStreamSynchronize(c->stream));
            const Ctl h = *c->h_ctl;
            if (c->p.profile) {
                // launches that did work: iterations t_before+1 .. h.t
                const int worked = h.t - t_before;
                for (int k = 0; k < worked && k < batch; k++) {
                    float ms = 0.f;
                    if (cudaEventElapsedTime(&ms, c->graph_ev[2 * k], c->graph_ev[2 * k + 1]) == cudaSuccess) {
                        bool found = false;
                        for (auto& pe : c->prof)
                            if (pe.name == "K3_pgd") {
                                pe.ms += ms;
                                pe.launches += 1;
                                found = true;
                            }
                        if (!found) c->prof.push_back({"K3_pgd", (double)ms, 1});
                    }
                }
            }
            t_before = h.t;
            if (h.done) {
                iters = h.t_res;
                break;
            }
        }
    }
    c->last_iters = iters;
    // final evaluation of the returned state
    c->h_ctl->t_res = iters;
    CC_CUDA(c, cudaMemcpyAsync(&c->ctl.p->t_res, &c->h_ctl->t_res, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    PgdArgs af = make_args(c, 1);
    int tok = cc_prof_begin(c, "K3_final_check");
    CCL(c, k_pgd<<<nb, PGD_THREADS, 0, c->stream>>>(af));
    cc_prof_end(c, tok);
    CC_CUDA(c, cudaGetLastError());
    double al[3];
    CC_TRY(global_check(c, al));
    info->iterations = iters;
    info->active_final = (int64_t)al[0];
    info->loss_final = al[1];
    info->violated_final = (int64_t)al[2];
    info->converged = stop_rule(c->p.stop_mode, (unsigned long long)al[0], al[1], (unsigned long long)al[2],
                                c->p.eps_loss) ||
                      (c->p.stop_mode == CC_STOP_NONE && al[0] == 0.0);
    c->final_active = (unsigned long long)al[0];
    c->final_loss = al[1];
    c->final_violated = (unsigned long long)al[2];
    return CC_OK;
}

cc_status write_output(cc_ctx* c, const float4* res, float* xo, float* yo, float* zo) {
    const int64_t n = c->n;
    CC_TRY(cc_ensure(c, c->cor4, (size_t)std::max<int64_t>(n, 1), "cor4"));
    int tok = cc_prof_begin(c, "K3_output");
    if (n > 0)
        CCL(c, k_cor4<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(n, c->dec4.p, c->eidx.p, (uint32_t)c->E,
                                                                          res, c->cor4.p));
    if (c->n_in > 0 && xo)
        CCL(c, k_output<<<(unsigned)((c->n_in + 255) / 256), 256, 0, c->stream>>>(c->n_in, c->slot_of.p, c->cor4.p,
                                                                                  xo, yo, zo));
    cc_prof_end(c, tok);
    CC_CUDA(c, cudaGetLastError());
    return CC_OK;
}

}  // namespace cc
