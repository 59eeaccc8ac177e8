// dist.cu -- multi-GPU form of the hot path (§III-D; §IV-D): x-slab spatial
// decomposition, ghost shells of width delta = b + 2 sqrt3 xi exchanged with NCCL (the paper's
// MPI_Isend/Irecv), a per-iteration refresh of editable ghost positions (R19) and a global
// allreduce of the L_tight-active count that drives the stop (the paper's MPI_Allreduce of the
// loss), FoF label merging across slabs, and reductions of MCC counts and halo sizes.
//
// Rank r owns original x in [r L/R, (r+1) L/R); its neighbours are r-1 and r+1 (periodic).  The
// local particle set is [owned | ghosts from the left | ghosts from the right]; the local search
// structure spans x in [lo - gw, hi + gw) without wrap.  Every pair with an owned endpoint is
// found locally; the pair belongs to the owner of its min-gid endpoint (R17).  Results are
// bit-identical to one GPU: rows are summed in gid order and ghost positions are the owners'.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <unordered_map>
#include <vector>

#include "cc_internal.cuh"

namespace cc {
namespace {

constexpr int DT = 256;



// both shell lists in ONE pass over x (decoupled look-back, cc_internal.cuh lookback_warp0):
// list0 = owned particles within the ghost width of the lower face, list1 = of the upper face,
// each in ascending input order; a thread owns SL_I consecutive particles.  Replaces a flag pass,
// two device-wide scans and two compactions.  The two running counts share one
// look-back word (31 bits each: counts < 2^30).
constexpr int SL_T = 256, SL_I = 16, SL_TILE = SL_T * SL_I;

__global__ void __launch_bounds__(SL_T)
k_shell_lists(int64_t n, const float* __restrict__ x, double lo, double hi, double gw, uint32_t* __restrict__ list0,
              uint32_t* __restrict__ list1, unsigned long long* __restrict__ status, unsigned int* __restrict__ ticket,
              unsigned long long* __restrict__ out /* [0] error bits, [1] n0, [2] n1 */) {
    __shared__ unsigned int tile_sh;
    __shared__ unsigned long long base_sh;
    __shared__ unsigned long long wsum[SL_T / 32];
    if (threadIdx.x == 0) tile_sh = atomicAdd(ticket, 1u);
    __syncthreads();
    const unsigned int tile = tile_sh;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t i0 = (int64_t)tile * SL_TILE + (int64_t)threadIdx.x * SL_I;
    uint32_t m0 = 0u, m1 = 0u;
    bool bad = false;
#pragma unroll
    for (int k = 0; k < SL_I; k++) {
        const int64_t i = i0 + k;
        if (i < n) {
            const double xv = (double)x[i];
            bad |= !(xv >= lo && xv < hi);  // not in this rank's slab
            m0 |= (xv < lo + gw ? 1u : 0u) << k;
            m1 |= (xv >= hi - gw ? 1u : 0u) << k;
        }
    }
    if (bad) atomicOr(&out[0], 4ull);
    const unsigned long long cnt = (unsigned long long)__popc(m0) | ((unsigned long long)__popc(m1) << 32);
    unsigned long long inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    unsigned long long wex = 0ull, tot = 0ull;
#pragma unroll
    for (int k = 0; k < SL_T / 32; k++) {
        wex += k < w ? wsum[k] : 0ull;
        tot += wsum[k];
    }
    const unsigned long long M31 = (1ull << 31) - 1ull;
    if (threadIdx.x < 32) {
        const unsigned long long packed = (tot & 0xFFFFFFFFull) | ((tot >> 32) << 31);
        const unsigned long long ex = lookback_warp0(status, tile, packed);
        if (lane == 0) {
            base_sh = ex;
            if ((int64_t)(tile + 1) * SL_TILE >= n) {  // the last tile
                out[1] = (ex & M31) + (tot & 0xFFFFFFFFull);
                out[2] = (ex >> 31) + (tot >> 32);
            }
        }
    }
    __syncthreads();
    const unsigned long long my = wex + inc - cnt;
    unsigned long long q0 = (base_sh & M31) + (my & 0xFFFFFFFFull);
    unsigned long long q1 = (base_sh >> 31) + (my >> 32);
    while (m0) {
        const int k = __ffs(m0) - 1;
        m0 &= m0 - 1u;
        list0[q0++] = (uint32_t)(i0 + k);
    }
    while (m1) {
        const int k = __ffs(m1) - 1;
        m1 &= m1 - 1u;
        list1[q1++] = (uint32_t)(i0 + k);
    }
}


// pack particles of a list as 7 SoA words (x, y, z, xh, yh, zh, gid)
__global__ void k_pack7(int64_t m, const uint32_t* __restrict__ list, const float* __restrict__ x,
                        const float* __restrict__ y, const float* __restrict__ z, const float* __restrict__ xh,
                        const float* __restrict__ yh, const float* __restrict__ zh, const uint32_t* __restrict__ gid,
                        uint32_t* __restrict__ buf) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    const uint32_t i = list[k];
    buf[0 * m + k] = __float_as_uint(x[i]);
    buf[1 * m + k] = __float_as_uint(y[i]);
    buf[2 * m + k] = __float_as_uint(z[i]);
    buf[3 * m + k] = __float_as_uint(xh[i]);
    buf[4 * m + k] = __float_as_uint(yh[i]);
    buf[5 * m + k] = __float_as_uint(zh[i]);
    buf[6 * m + k] = gid ? gid[i] : i;
}


// received block of m particles -> staging rows [off, off + m)
__global__ void k_unstage(int64_t m, int64_t cap, int64_t off, const uint32_t* __restrict__ buf,
                          uint32_t* __restrict__ st) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    for (int w = 0; w < 7; w++) st[w * cap + off + k] = buf[w * m + k];
}

// ghost editables: (source dir, index in the source's shell list) for each ghost editable
__global__ void k_ghost_requests(int64_t n, const uint32_t* __restrict__ eidx, const float4* __restrict__ dec4,
                                 uint32_t n_own, uint32_t n_from_left, uint32_t e_own, uint32_t* __restrict__ req_left,
                                 uint32_t* __restrict__ req_left_e, unsigned long long* __restrict__ cnt_left,
                                 uint32_t* __restrict__ req_right, uint32_t* __restrict__ req_right_e,
                                 unsigned long long* __restrict__ cnt_right) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const uint32_t eg = eidx[s];
    if (eg == 0xFFFFFFFFu || eg < e_own) return;  // ghost editables are numbered after all owned ones
    const uint32_t i = __float_as_uint(dec4[s].w);
    if (i - n_own < n_from_left) {
        const unsigned long long q = atomicAdd(cnt_left, 1ull);
        req_left[q] = i - n_own;
        req_left_e[q] = eg;
    } else {
        const unsigned long long q = atomicAdd(cnt_right, 1ull);
        req_right[q] = i - n_own - n_from_left;
        req_right_e[q] = eg;
    }
}

// owner side: requested shell-list index -> owned editable index
// slot_of may still hold provisional slots (bin.cu ensure_slot_of: completed on first use); the
// few shell particles asked for here take the two-step lookup fin[slot_of[i]] instead of
// completing the whole map inside S2-S3
__global__ void k_map_requests(int64_t m, const uint32_t* __restrict__ req, const uint32_t* __restrict__ shell,
                               const uint32_t* __restrict__ slot_of, const uint32_t* __restrict__ fin, int fixed,
                               const uint32_t* __restrict__ eidx, uint32_t e_own, uint32_t* __restrict__ send_e,
                               unsigned long long* errs) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    uint32_t sl = slot_of[shell[req[k]]];
    if (!fixed) sl = fin[sl];
    const uint32_t e = eidx[sl];
    if (e >= e_own) atomicOr(errs, 8ull);  // must be an owned editable
    send_e[k] = e;
}

// per-iteration refresh: pack the updated owned positions / unpack into ghost slots
__global__ void k_refresh_pack(int64_t m, const uint32_t* __restrict__ send_e, const Ctl* __restrict__ ctl,
                               const float4* __restrict__ p0, const float4* __restrict__ p1, float4* __restrict__ buf) {
    if (ctl->done) return;
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    const int t = ctl->t + 1;  // the iteration whose update was just written (t not yet advanced)
    const float4* dst = (t & 1) ? p1 : p0;
    buf[k] = dst[send_e[k]];
}

__global__ void k_refresh_unpack(int64_t m, const uint32_t* __restrict__ recv_e, const Ctl* __restrict__ ctl,
                                 float4* __restrict__ p0, float4* __restrict__ p1, const float4* __restrict__ buf) {
    if (ctl->done) return;
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    const int t = ctl->t + 1;
    float4* dst = (t & 1) ? p1 : p0;
    dst[recv_e[k]] = buf[k];
}


// ---- per-iteration exchange over NVLink peer memory (X3, replaces NCCL send/recv + allreduce)
// Block layout (bytes): [0, 64) flags u32[16] (rank r's epoch at index r); [64, 1088) stop
// statistics u64 [2 parities][8 ranks][LFX_STATS]; [1088, 1092) local ticket; [1280, ...) the two
// receive areas (0: from the left rank, 1: from the right rank), each 2 parities x cap float4.
constexpr size_t PM_STATS = 64, PM_TICKET = 1088, PM_AREAS = 1280;
__host__ __device__ inline size_t pm_area_off(int d, const int64_t cap[2]) {
    return PM_AREAS + (d ? 2 * (size_t)cap[0] * sizeof(float4) : 0);
}

struct PeerArgs {
    Ctl* ctl;
    const float4* p0;
    const float4* p1;
    const uint32_t* send_e[2];
    int64_t ns[2];
    float4* dst[2];       // send dir 0 -> the left rank's area 1, dir 1 -> the right rank's area 0
    int64_t dstride[2];   // their capacity per parity
    const unsigned long long* red;  // this rank's statistics (k_pgd's last block)
    unsigned long long* red_sum;    // the global sums (k_decide's input)
    unsigned char* blk[8];          // every rank's block (mine included), mapped here
    int rank, nranks;
};

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// push the updated owned positions the neighbours hold as ghosts straight into their receive
// areas (P2P stores over NVLink), then the last block publishes this rank's statistics and epoch
// flag in every rank's block, waits for every rank's flag and sums the statistics (integer sums:
// the same value on every rank, in any order)
__global__ void __launch_bounds__(256) k_peer_exchange(PeerArgs a) {
    Ctl* ctl = a.ctl;
    if (ctl->done) return;
    const int t = ctl->t + 1;  // the iteration whose update was just written
    const int par = t & 1;
    const float4* src = par ? a.p1 : a.p0;
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gs = (int64_t)gridDim.x * blockDim.x;
    for (int d = 0; d < 2; d++) {
        float4* dst = a.dst[d] + (size_t)par * a.dstride[d];
        for (int64_t k = gt; k < a.ns[d]; k += gs) dst[k] = src[a.send_e[d][k]];
    }
    __threadfence_system();
    __syncthreads();
    __shared__ bool last;
    unsigned* ticket = reinterpret_cast<unsigned*>(a.blk[a.rank] + PM_TICKET);
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    *ticket = 0u;
    __threadfence_system();
    const unsigned epoch = ctl->ep_base + (unsigned)t;
    for (int r = 0; r < a.nranks; r++) {
        unsigned long long* st = reinterpret_cast<unsigned long long*>(a.blk[r] + PM_STATS) +
                                 ((size_t)par * 8 + a.rank) * LFX_STATS;
        for (int w = 0; w < LFX_STATS; w++) st[w] = a.red[w];
    }
    __threadfence_system();
    for (int r = 0; r < a.nranks; r++) st_release_sys(reinterpret_cast<unsigned*>(a.blk[r]) + a.rank, epoch);
    const unsigned* fl = reinterpret_cast<const unsigned*>(a.blk[a.rank]);
    for (int r = 0; r < a.nranks; r++)
        while ((int)(ld_acquire_sys(fl + r) - epoch) < 0) __nanosleep(64);
    const volatile unsigned long long* mine =
        reinterpret_cast<const volatile unsigned long long*>(a.blk[a.rank] + PM_STATS) + (size_t)par * 8 * LFX_STATS;
    for (int w = 0; w < LFX_STATS; w++) {
        unsigned long long v = 0ull;
        for (int r = 0; r < a.nranks; r++) v += mine[(size_t)r * LFX_STATS + w];
        a.red_sum[w] = v;
    }
    __threadfence();
}

// global stop decision after the allreduce of (active, loss)
__global__ void k_decide(Ctl* ctl, const unsigned long long* __restrict__ red, int stop_mode, double eps_loss,
                         int t_max, long long* trace_a, double* trace_l, long long* trace_v) {
    if (ctl->done) return;
    const int t = ctl->t + 1;
    const unsigned long long tu = red[0];
    const double td = lfx_value(red + 2);  // exact integer sums over ranks: rank-count invariant
    const unsigned long long tv = red[1];
    ctl->active = tu;
    ctl->loss = td;
    ctl->violated = tv;
    if (trace_a) {
        trace_a[t - 1] = (long long)tu;
        trace_l[t - 1] = td;
        trace_v[t - 1] = (long long)tv;
    }
    if (stop_rule(stop_mode, tu, lfx_le(red + 2, eps_loss), tv)) {
        ctl->done = 1;
        ctl->t_res = t - 1;
        ctl->converged = 1;
    } else if (t >= t_max) {
        ctl->done = 1;
        ctl->t_res = t;
    }
    ctl->t = t;
}

// the peer path's per-iteration tail after k_peer_exchange in ONE launch: unpack both receive
// areas into the ghost slots, then the last block (ticket) applies the stop rule like k_decide.
// Two graph nodes fewer per PGD iteration (C5 at R = 4: 662 iterations).  ctl->ticket is free
// here: k_pgd's last block left it at 0, and this kernel's last block resets it.
__global__ void __launch_bounds__(256)
k_peer_finish(int64_t m0, int64_t m1, const uint32_t* __restrict__ recv0, const uint32_t* __restrict__ recv1, Ctl* ctl,
              float4* __restrict__ p0, float4* __restrict__ p1, const float4* __restrict__ area0, int64_t cap0,
              const float4* __restrict__ area1, int64_t cap1, const unsigned long long* __restrict__ red,
              int stop_mode, double eps_loss, int t_max, long long* trace_a, double* trace_l, long long* trace_v) {
    if (ctl->done) return;
    const int t = ctl->t + 1;
    float4* dst = (t & 1) ? p1 : p0;
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < m0) dst[recv0[k]] = __ldcv(area0 + (size_t)(t & 1) * cap0 + k);
    else if (k < m0 + m1) dst[recv1[k - m0]] = __ldcv(area1 + (size_t)(t & 1) * cap1 + (k - m0));
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&ctl->ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    ctl->ticket = 0u;
    const unsigned long long tu = red[0];
    const double td = lfx_value(red + 2);  // exact integer sums over ranks: rank-count invariant
    const unsigned long long tv = red[1];
    ctl->active = tu;
    ctl->loss = td;
    ctl->violated = tv;
    if (trace_a) {
        trace_a[t - 1] = (long long)tu;
        trace_l[t - 1] = td;
        trace_v[t - 1] = (long long)tv;
    }
    if (stop_rule(stop_mode, tu, lfx_le(red + 2, eps_loss), tv)) {
        ctl->done = 1;
        ctl->t_res = t - 1;
        ctl->converged = 1;
    } else if (t >= t_max) {
        ctl->done = 1;
        ctl->t_res = t;
    }
    ctl->t = t;
    __threadfence();
}

// FoF label exchange: labels of the shell lists (owner side) ...
__global__ void k_label_pack(int64_t m, const uint32_t* __restrict__ shell, const uint32_t* __restrict__ slot_of,
                             const uint32_t* __restrict__ par, const uint32_t* __restrict__ mingid,
                             uint32_t* __restrict__ buf) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    buf[k] = mingid[par[slot_of[shell[k]]]];
}
// ... lower the local component of each ghost to the owner's label
__global__ void k_label_merge(int64_t m, uint32_t first_local, const uint32_t* __restrict__ slot_of,
                              const uint32_t* __restrict__ par, uint32_t* __restrict__ mingid,
                              const uint32_t* __restrict__ buf, unsigned long long* changed) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    const uint32_t r = par[slot_of[first_local + k]];
    const uint32_t old = atomicMin(&mingid[r], buf[k]);
    if (buf[k] < old) atomicAdd(changed, 1ull);
}

// owned particles whose label equals their own gid = one per global component
__global__ void k_count_label_roots(int64_t n_own, const uint32_t* __restrict__ slot_of,
                                    const uint32_t* __restrict__ par, const uint32_t* __restrict__ mingid,
                                    const float4* __restrict__ orig4, unsigned long long* __restrict__ cnt) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned int v = 0;
    if (i < n_own) {
        const uint32_t s = slot_of[i];
        v = mingid[par[s]] == __float_as_uint(orig4[s].w);
    }
    const unsigned int tot = __syncthreads_count(v);
    if (threadIdx.x == 0 && tot) atomicAdd(cnt, (unsigned long long)tot);
}

// owned members per local root, and whether the local component touches a ghost
__global__ void k_root_counts(int64_t n, uint32_t n_own, const uint32_t* __restrict__ par,
                              const float4* __restrict__ dec4, uint32_t* __restrict__ owned_cnt,
                              uint32_t* __restrict__ has_ghost) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const uint32_t r = par[s];
    if (__float_as_uint(dec4[s].w) < n_own) atomicAdd(&owned_cnt[r], 1u);
    else has_ghost[r] = 1u;
}

__global__ void k_root_collect(int64_t n, const uint32_t* __restrict__ par, const uint32_t* __restrict__ owned_cnt,
                               const uint32_t* __restrict__ has_ghost, const uint32_t* __restrict__ mingid,
                               uint32_t min_size, uint32_t* __restrict__ interior, unsigned long long* n_interior,
                               uint2* __restrict__ boundary, unsigned long long* n_boundary) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    if (par[s] != (uint32_t)s || owned_cnt[s] == 0) return;
    if (has_ghost[s]) {
        const unsigned long long q = atomicAdd(n_boundary, 1ull);
        boundary[q] = make_uint2(mingid[s], owned_cnt[s]);
    } else if (owned_cnt[s] >= min_size) {
        const unsigned long long q = atomicAdd(n_interior, 1ull);
        interior[q] = owned_cnt[s];
    }
}

}  // namespace

// ------------------------------------------------------------------------------------------
cc_status dist_init(cc_ctx* c, const cc_dist* d) {
    c->rank = d->rank;
    c->nranks = d->nranks;
    if (d->nranks <= 1) return CC_OK;
    if ((!d->nccl_id_h && !d->vgroup) || d->rank < 0 || d->rank >= d->nranks) return cc_fail(c, CC_E_ARG, "bad cc_dist");
    CC_TRY(comm_init(c, d));
    c->left = (d->rank + d->nranks - 1) % d->nranks;
    c->right = (d->rank + 1) % d->nranks;
    c->slab_lo = c->p.box * (double)d->rank / d->nranks;
    c->slab_hi = c->p.box * (double)(d->rank + 1) / d->nranks;
    return CC_OK;
}

void dist_destroy(cc_ctx* c) {
    for (int r = 0; r < 8; r++)
        if (c->pm_peer[r] && c->pm_peer[r] != c->pm_local) cudaIpcCloseMemHandle(c->pm_peer[r]);
    if (c->pm_local) cudaFree(c->pm_local);
    c->pm_local = nullptr;
    for (int r = 0; r < 8; r++) c->pm_peer[r] = nullptr;
    if (c->nranks > 1) comm_destroy(c);
}

// in-place global sums of small device arrays (synchronising)
cc_status dist_allreduce_u64(cc_ctx* c, unsigned long long* dev, size_t count) {
    if (c->nranks <= 1) return CC_OK;
    CC_TRY(comm_allreduce(c, dev, count, CT_U64, CO_SUM));
    return CC_OK;
}
cc_status dist_allreduce_f64(cc_ctx* c, double* dev, size_t count) {
    if (c->nranks <= 1) return CC_OK;
    CC_TRY(comm_allreduce(c, dev, count, CT_F64, CO_SUM));
    return CC_OK;
}

// one-time ghost exchange (X1): local staging = [owned | from left | from right]
cc_status dist_exchange_ghosts(cc_ctx* c, int64_t n, const float* x, const float* y, const float* z, const float* xh,
                               const float* yh, const float* zh, const uint32_t* gid) {
    const double gw = c->r_pair;  // ghost width delta (1 + 1e-5)
    const size_t n1 = (size_t)std::max<int64_t>(n, 1);
    CC_TRY(cc_ensure(c, c->shell[0], n1, "shell list"));
    CC_TRY(cc_ensure(c, c->shell[1], n1, "shell list"));
    CC_TRY(cc_ensure(c, c->counters, 16, "counters"));
    CC_CUDA(c, cudaMemsetAsync(c->counters.p, 0, 16 * sizeof(unsigned long long), c->stream));
    if (n > 0) {
        const int64_t nt = (n + SL_TILE - 1) / SL_TILE;
        CC_TRY(cc_ensure(c, c->codec_status, (size_t)nt + 2, "look-back status"));
        unsigned long long* st = c->codec_status.p;
        CC_CUDA(c, cudaMemsetAsync(st, 0, (size_t)(nt + 1) * sizeof(unsigned long long), c->stream));
        CCL(c, k_shell_lists<<<(unsigned)nt, SL_T, 0, c->stream>>>(n, x, c->slab_lo, c->slab_hi, gw, c->shell[0].p,
                                                                   c->shell[1].p, st,
                                                                   reinterpret_cast<unsigned int*>(st + nt),
                                                                   c->counters.p));
    }
    CC_CUDA(c, cudaMemcpyAsync(c->h_counters, c->counters.p, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                               c->stream));
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    if (c->h_counters[0] & 4ull) return cc_fail(c, CC_E_DATA, "an owned particle lies outside this rank's x slab");
    int64_t ns[2] = {(int64_t)c->h_counters[1], (int64_t)c->h_counters[2]};
    for (int d = 0; d < 2; d++) c->n_shell[d] = ns[d];
    // counts: send dir0 -> left, dir1 -> right; receive from right (their dir0), from left (their dir1)
    CC_TRY(cc_ensure(c, c->dcnt, 4, "dist counts"));
    {
        long long h[4] = {ns[0], ns[1], 0, 0};
        CC_CUDA(c, cudaMemcpyAsync(c->dcnt.p, h, 2 * sizeof(long long), cudaMemcpyHostToDevice, c->stream));
        CC_TRY(comm_group_start(c));
        CC_TRY(comm_send(c, c->dcnt.p + 0, 1, CT_I64, c->left));
        CC_TRY(comm_send(c, c->dcnt.p + 1, 1, CT_I64, c->right));
        CC_TRY(comm_recv(c, c->dcnt.p + 2, 1, CT_I64, c->right));
        CC_TRY(comm_recv(c, c->dcnt.p + 3, 1, CT_I64, c->left));
        CC_TRY(comm_group_end(c));
        CC_CUDA(c, cudaMemcpyAsync(h, c->dcnt.p, 4 * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
        CC_CUDA(c, cudaStreamSynchronize(c->stream));
        c->n_from_right = h[2];
        c->n_from_left = h[3];
    }
    const int64_t nl = n + c->n_from_left + c->n_from_right;
    if (nl >= MAX_LOCAL) return cc_fail(c, CC_E_DATA, "local particles beyond the 2^30 index space");
    // ghost staging only (7 SoA words, stride cap = ghost count): binning reads the owned
    // particles from the caller's arrays in place
    const int64_t cap = std::max<int64_t>(c->n_from_left + c->n_from_right, 1);
    CC_TRY(cc_ensure(c, c->stage, (size_t)(7 * cap), "ghost staging"));
    for (int d = 0; d < 2; d++)
        CC_TRY(cc_ensure(c, c->sbuf7[d], (size_t)std::max<int64_t>(7 * ns[d], 1), "ghost send buffer"));
    CC_TRY(cc_ensure(c, c->rbuf7[0], (size_t)std::max<int64_t>(7 * c->n_from_left, 1), "ghost recv buffer"));
    CC_TRY(cc_ensure(c, c->rbuf7[1], (size_t)std::max<int64_t>(7 * c->n_from_right, 1), "ghost recv buffer"));
    for (int d = 0; d < 2; d++)
        if (ns[d] > 0)
            CCL(c, k_pack7<<<(unsigned)((ns[d] + DT - 1) / DT), DT, 0, c->stream>>>(ns[d], c->shell[d].p, x, y, z, xh, yh,
                                                                                  zh, gid, c->sbuf7[d].p));
    CC_TRY(comm_group_start(c));
    if (ns[0] > 0) CC_TRY(comm_send(c, c->sbuf7[0].p, (size_t)(7 * ns[0]), CT_U32, c->left));
    if (ns[1] > 0) CC_TRY(comm_send(c, c->sbuf7[1].p, (size_t)(7 * ns[1]), CT_U32, c->right));
    if (c->n_from_right > 0)
        CC_TRY(comm_recv(c, c->rbuf7[1].p, (size_t)(7 * c->n_from_right), CT_U32, c->right));
    if (c->n_from_left > 0)
        CC_TRY(comm_recv(c, c->rbuf7[0].p, (size_t)(7 * c->n_from_left), CT_U32, c->left));
    CC_TRY(comm_group_end(c));
    if (c->n_from_left > 0)
        CCL(c, k_unstage<<<(unsigned)((c->n_from_left + DT - 1) / DT), DT, 0, c->stream>>>(c->n_from_left, cap, 0,
                                                                                          c->rbuf7[0].p, c->stage.p));
    if (c->n_from_right > 0)
        CCL(c, k_unstage<<<(unsigned)((c->n_from_right + DT - 1) / DT), DT, 0, c->stream>>>(
                   c->n_from_right, cap, c->n_from_left, c->rbuf7[1].p, c->stage.p));
    CC_CUDA(c, cudaGetLastError());
    c->stage_cap = cap;
    c->n = nl;
    return CC_OK;
}

// refresh lists of ghost editables (X2), after the rows exist

// map every rank's peer block (X3 over NVLink): (re)allocate mine if the receive areas grew,
// exchange IPC handles with an allgather, open the peers' blocks that changed
static cc_status dist_setup_peer(cc_ctx* c) {
    // Every rank takes part in the same collectives whatever its environment says; the peer
    // path is used only if EVERY rank wants it and mapped every peer (one allgather of the
    // wishes + handles, one MIN allreduce of the outcome) -- a rank falling back alone to the
    // NCCL path while the others spin on epoch flags would hang.
    c->pm_ok = false;
    if (c->vgroup) return CC_OK;  // virtual ranks share one GPU: the copy transport, no peer mapping
    const char* env = std::getenv("CC_PEER");
    const int want = !((env && env[0] == '0') || c->nranks > 8);
    if (want) {
        const int64_t need0 = std::max<int64_t>(c->n_ref_recv[0], 1), need1 = std::max<int64_t>(c->n_ref_recv[1], 1);
        if (!c->pm_local || need0 > c->pm_cap[0] || need1 > c->pm_cap[1]) {
            if (c->pm_local) cudaFree(c->pm_local);
            c->pm_local = nullptr;
            c->pm_cap[0] = need0 + need0 / 4 + 64;
            c->pm_cap[1] = need1 + need1 / 4 + 64;
            c->pm_bytes = pm_area_off(1, c->pm_cap) + 2 * (size_t)c->pm_cap[1] * sizeof(float4);
            CC_CUDA(c, cudaMalloc(&c->pm_local, c->pm_bytes));
            CC_CUDA(c, cudaMemsetAsync(c->pm_local, 0, c->pm_bytes, c->stream));
        }
    }
    struct Rec {
        cudaIpcMemHandle_t h;
        int64_t cap[2];
        int32_t want;
        unsigned char pad[128 - sizeof(cudaIpcMemHandle_t) - 20];
    };
    static_assert(sizeof(Rec) == 128, "");
    Rec mine;
    std::memset(&mine, 0, sizeof(mine));
    if (want) CC_CUDA(c, cudaIpcGetMemHandle(&mine.h, c->pm_local));
    mine.cap[0] = c->pm_cap[0];
    mine.cap[1] = c->pm_cap[1];
    mine.want = want;
    unsigned char* dbuf = nullptr;
    CC_CUDA(c, cudaMalloc(&dbuf, 128 * (size_t)(c->nranks + 1)));
    CC_CUDA(c, cudaMemcpyAsync(dbuf, &mine, 128, cudaMemcpyHostToDevice, c->stream));
    CC_TRY(comm_allgather(c, dbuf, dbuf + 128, 128, CT_U8));
    std::vector<Rec> all((size_t)c->nranks);
    CC_CUDA(c, cudaMemcpyAsync(all.data(), dbuf + 128, 128 * (size_t)c->nranks, cudaMemcpyDeviceToHost, c->stream));
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    bool all_want = true;
    for (int r = 0; r < c->nranks; r++) all_want = all_want && all[(size_t)r].want != 0;
    int ok = all_want ? 1 : 0;
    for (int r = 0; r < c->nranks && ok; r++) {
        c->pm_peer_cap[r][0] = all[(size_t)r].cap[0];
        c->pm_peer_cap[r][1] = all[(size_t)r].cap[1];
        if (r == c->rank) {
            c->pm_peer[r] = c->pm_local;
            continue;
        }
        if (c->pm_peer[r] && std::memcmp(c->pm_handle[r], &all[(size_t)r].h, 64) == 0) continue;
        if (c->pm_peer[r]) cudaIpcCloseMemHandle(c->pm_peer[r]);
        c->pm_peer[r] = nullptr;
        void* ptr = nullptr;
        if (cudaIpcOpenMemHandle(&ptr, all[(size_t)r].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            cudaGetLastError();
            ok = 0;  // no peer mapping here: every rank must stay on the NCCL path
            break;
        }
        c->pm_peer[r] = ptr;
        std::memcpy(c->pm_handle[r], &all[(size_t)r].h, 64);
    }
    // agreement: the peer path only if every rank succeeded
    int* dok = reinterpret_cast<int*>(dbuf);
    CC_CUDA(c, cudaMemcpyAsync(dok, &ok, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    CC_TRY(comm_allreduce(c, dok, 1, CT_I32, CO_MIN));
    int all_ok = 0;
    CC_CUDA(c, cudaMemcpyAsync(&all_ok, dok, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    cudaFree(dbuf);
    if (!all_ok) return CC_OK;
    CC_TRY(cc_ensure(c, c->red_sum, LFX_STATS, "peer statistics"));
    c->pm_ok = true;
    return CC_OK;
}

cc_status dist_setup_refresh(cc_ctx* c) {
    const int64_t n = c->n;
    CC_TRY(cc_ensure(c, c->counters, 16, "counters"));
    const int64_t ng = std::max<int64_t>(c->E_all - c->E, 1);
    for (int d = 0; d < 2; d++) {
        CC_TRY(cc_ensure(c, c->req[d], (size_t)ng, "ghost requests"));
        CC_TRY(cc_ensure(c, c->recv_e[d], (size_t)ng, "ghost refresh targets"));
    }
    CC_CUDA(c, cudaMemsetAsync(c->counters.p + 12, 0, 3 * sizeof(unsigned long long), c->stream));
    if (n > 0)
        CCL(c, k_ghost_requests<<<(unsigned)((n + DT - 1) / DT), DT, 0, c->stream>>>(
                   n, c->eidx.p, c->dec4.p, (uint32_t)c->n_in, (uint32_t)c->n_from_left, (uint32_t)c->E, c->req[0].p,
                   c->recv_e[0].p, c->counters.p + 12, c->req[1].p, c->recv_e[1].p, c->counters.p + 13));
    CC_CUDA(c, cudaMemcpyAsync(c->h_counters + 12, c->counters.p + 12, 2 * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, c->stream));
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    int64_t nreq[2] = {(int64_t)c->h_counters[12], (int64_t)c->h_counters[13]};  // to left, to right
    // exchange request counts: my dir-0 requests concern the left rank's dir-1 shell, etc.
    {
        long long h[4] = {nreq[0], nreq[1], 0, 0};
        CC_CUDA(c, cudaMemcpyAsync(c->dcnt.p, h, 2 * sizeof(long long), cudaMemcpyHostToDevice, c->stream));
        CC_TRY(comm_group_start(c));
        CC_TRY(comm_send(c, c->dcnt.p + 0, 1, CT_I64, c->left));
        CC_TRY(comm_send(c, c->dcnt.p + 1, 1, CT_I64, c->right));
        CC_TRY(comm_recv(c, c->dcnt.p + 2, 1, CT_I64, c->right));
        CC_TRY(comm_recv(c, c->dcnt.p + 3, 1, CT_I64, c->left));
        CC_TRY(comm_group_end(c));
        CC_CUDA(c, cudaMemcpyAsync(h, c->dcnt.p, 4 * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
        CC_CUDA(c, cudaStreamSynchronize(c->stream));
        // from the right: requests about my dir-1 shell (sent to the right); from the left: dir-0
        c->n_ref_send[1] = h[2];
        c->n_ref_send[0] = h[3];
    }
    c->n_ref_recv[0] = nreq[0];
    c->n_ref_recv[1] = nreq[1];
    for (int d = 0; d < 2; d++) {
        CC_TRY(cc_ensure(c, c->sreq[d], (size_t)std::max<int64_t>(c->n_ref_send[d], 1), "incoming requests"));
        CC_TRY(cc_ensure(c, c->send_e[d], (size_t)std::max<int64_t>(c->n_ref_send[d], 1), "refresh sources"));
        CC_TRY(cc_ensure(c, c->rsb[d], (size_t)std::max<int64_t>(c->n_ref_send[d], 1), "refresh send buffer"));
        CC_TRY(cc_ensure(c, c->rrb[d], (size_t)std::max<int64_t>(c->n_ref_recv[d], 1), "refresh recv buffer"));
    }
    CC_TRY(comm_group_start(c));
    if (nreq[0] > 0) CC_TRY(comm_send(c, c->req[0].p, (size_t)nreq[0], CT_U32, c->left));
    if (nreq[1] > 0) CC_TRY(comm_send(c, c->req[1].p, (size_t)nreq[1], CT_U32, c->right));
    if (c->n_ref_send[1] > 0)
        CC_TRY(comm_recv(c, c->sreq[1].p, (size_t)c->n_ref_send[1], CT_U32, c->right));
    if (c->n_ref_send[0] > 0)
        CC_TRY(comm_recv(c, c->sreq[0].p, (size_t)c->n_ref_send[0], CT_U32, c->left));
    CC_TRY(comm_group_end(c));
    for (int d = 0; d < 2; d++)
        if (c->n_ref_send[d] > 0)
            CCL(c, k_map_requests<<<(unsigned)((c->n_ref_send[d] + DT - 1) / DT), DT, 0, c->stream>>>(
                       c->n_ref_send[d], c->sreq[d].p, c->shell[d].p, c->slot_of.p, c->rnk.p, c->slot_of_valid ? 1 : 0,
                       c->eidx.p, (uint32_t)c->E, c->send_e[d].p, c->counters.p + 14));
    CC_CUDA(c, cudaMemcpyAsync(c->h_counters + 14, c->counters.p + 14, sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, c->stream));
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    if (c->h_counters[14] & 8ull) return cc_fail(c, CC_E_DATA, "ghost editable is not editable on its owner");
    CC_TRY(cc_ensure(c, c->red, LFX_STATS, "allreduce buffer"));
    return dist_setup_peer(c);
}

// per-iteration tail (X3): refresh ghosts, allreduce the stop statistics, decide
cc_status dist_iter_tail(cc_ctx* c, const float4* p0, const float4* p1) {
    if (c->pm_ok) {
        PeerArgs a;
        std::memset(&a, 0, sizeof(a));
        a.ctl = c->ctl.p;
        a.p0 = p0;
        a.p1 = p1;
        for (int d = 0; d < 2; d++) {
            a.send_e[d] = c->send_e[d].p;
            a.ns[d] = c->n_ref_send[d];
        }
        // my dir-0 sends land in the left rank's area 1 (its "from the right"), dir 1 in the
        // right rank's area 0
        a.dst[0] = reinterpret_cast<float4*>(static_cast<unsigned char*>(c->pm_peer[c->left]) +
                                             pm_area_off(1, c->pm_peer_cap[c->left]));
        a.dstride[0] = c->pm_peer_cap[c->left][1];
        a.dst[1] = reinterpret_cast<float4*>(static_cast<unsigned char*>(c->pm_peer[c->right]) +
                                             pm_area_off(0, c->pm_peer_cap[c->right]));
        a.dstride[1] = c->pm_peer_cap[c->right][0];
        a.red = c->red.p;
        a.red_sum = c->red_sum.p;
        for (int r = 0; r < c->nranks; r++) a.blk[r] = static_cast<unsigned char*>(c->pm_peer[r]);
        a.rank = c->rank;
        a.nranks = c->nranks;
        const int64_t ns = std::max(c->n_ref_send[0], c->n_ref_send[1]);
        const unsigned nb = (unsigned)std::min<int64_t>(std::max<int64_t>((ns + 255) / 256, 1), 148);
        CCL(c, k_peer_exchange<<<nb, 256, 0, c->stream>>>(a));
        const int64_t mr = c->n_ref_recv[0] + c->n_ref_recv[1];
        const float4* ar[2];
        for (int d = 0; d < 2; d++)
            ar[d] = reinterpret_cast<const float4*>(static_cast<unsigned char*>(c->pm_local) + pm_area_off(d, c->pm_cap));
        CCL(c, k_peer_finish<<<(unsigned)std::max<int64_t>((mr + 255) / 256, 1), 256, 0, c->stream>>>(
                   c->n_ref_recv[0], c->n_ref_recv[1], c->recv_e[0].p, c->recv_e[1].p, c->ctl.p,
                   const_cast<float4*>(p0), const_cast<float4*>(p1), ar[0], c->pm_cap[0], ar[1], c->pm_cap[1],
                   c->red_sum.p, c->p.stop_mode, c->p.eps_loss, c->p.t_max, c->trace_a.p, c->trace_l.p,
                   c->trace_v.p));
        return CC_OK;
    }
    for (int d = 0; d < 2; d++)
        if (c->n_ref_send[d] > 0)
            CCL(c, k_refresh_pack<<<(unsigned)((c->n_ref_send[d] + DT - 1) / DT), DT, 0, c->stream>>>(
                       c->n_ref_send[d], c->send_e[d].p, c->ctl.p, p0, p1, c->rsb[d].p));
    CC_TRY(comm_group_start(c));
    if (c->n_ref_send[0] > 0)
        CC_TRY(comm_send(c, c->rsb[0].p, (size_t)(4 * c->n_ref_send[0]), CT_F32, c->left));
    if (c->n_ref_send[1] > 0)
        CC_TRY(comm_send(c, c->rsb[1].p, (size_t)(4 * c->n_ref_send[1]), CT_F32, c->right));
    if (c->n_ref_recv[1] > 0)
        CC_TRY(comm_recv(c, c->rrb[1].p, (size_t)(4 * c->n_ref_recv[1]), CT_F32, c->right));
    if (c->n_ref_recv[0] > 0)
        CC_TRY(comm_recv(c, c->rrb[0].p, (size_t)(4 * c->n_ref_recv[0]), CT_F32, c->left));
    // the stop statistics travel in the same NCCL group as the ghost refresh (one launch)
    CC_TRY(comm_allreduce(c, c->red.p, LFX_STATS, CT_U64, CO_SUM));
    CC_TRY(comm_group_end(c));
    for (int d = 0; d < 2; d++)
        if (c->n_ref_recv[d] > 0)
            CCL(c, k_refresh_unpack<<<(unsigned)((c->n_ref_recv[d] + DT - 1) / DT), DT, 0, c->stream>>>(
                       c->n_ref_recv[d], c->recv_e[d].p, c->ctl.p, const_cast<float4*>(p0), const_cast<float4*>(p1),
                       c->rrb[d].p));
    CCL(c, k_decide<<<1, 1, 0, c->stream>>>(c->ctl.p, c->red.p, c->p.stop_mode, c->p.eps_loss, c->p.t_max,
                                            c->trace_a.p, c->trace_l.p, c->trace_v.p));
    return CC_OK;
}

// FoF label merge across slabs (X4): owners send their shell particles' labels; receivers lower
// the ghosts' local components; repeat until no label changes anywhere.
cc_status dist_fof_merge(cc_ctx* c, int64_t* n_groups) {
    CC_TRY(ensure_slot_of(c));
    const int64_t ns0 = c->n_shell[0], ns1 = c->n_shell[1], nfl = c->n_from_left, nfr = c->n_from_right;
    for (int d = 0; d < 2; d++) {
        CC_TRY(cc_ensure(c, c->lsb[d], (size_t)std::max<int64_t>(c->n_shell[d], 1), "label send"));
    }
    CC_TRY(cc_ensure(c, c->lrb[0], (size_t)std::max<int64_t>(nfl, 1), "label recv"));
    CC_TRY(cc_ensure(c, c->lrb[1], (size_t)std::max<int64_t>(nfr, 1), "label recv"));
    CC_TRY(cc_ensure(c, c->counters, 16, "counters"));
    for (int round = 0; round < 4 * c->nranks + 8; round++) {
        CC_CUDA(c, cudaMemsetAsync(c->counters.p + 15, 0, sizeof(unsigned long long), c->stream));
        if (ns0 > 0)
            CCL(c, k_label_pack<<<(unsigned)((ns0 + DT - 1) / DT), DT, 0, c->stream>>>(ns0, c->shell[0].p, c->slot_of.p,
                                                                                     c->parent.p, c->mingid.p,
                                                                                     c->lsb[0].p));
        if (ns1 > 0)
            CCL(c, k_label_pack<<<(unsigned)((ns1 + DT - 1) / DT), DT, 0, c->stream>>>(ns1, c->shell[1].p, c->slot_of.p,
                                                                                     c->parent.p, c->mingid.p,
                                                                                     c->lsb[1].p));
        CC_TRY(comm_group_start(c));
        if (ns0 > 0) CC_TRY(comm_send(c, c->lsb[0].p, (size_t)ns0, CT_U32, c->left));
        if (ns1 > 0) CC_TRY(comm_send(c, c->lsb[1].p, (size_t)ns1, CT_U32, c->right));
        if (nfr > 0) CC_TRY(comm_recv(c, c->lrb[1].p, (size_t)nfr, CT_U32, c->right));
        if (nfl > 0) CC_TRY(comm_recv(c, c->lrb[0].p, (size_t)nfl, CT_U32, c->left));
        CC_TRY(comm_group_end(c));
        if (nfl > 0)
            CCL(c, k_label_merge<<<(unsigned)((nfl + DT - 1) / DT), DT, 0, c->stream>>>(
                       nfl, (uint32_t)c->n_in, c->slot_of.p, c->parent.p, c->mingid.p, c->lrb[0].p,
                       c->counters.p + 15));
        if (nfr > 0)
            CCL(c, k_label_merge<<<(unsigned)((nfr + DT - 1) / DT), DT, 0, c->stream>>>(
                       nfr, (uint32_t)(c->n_in + nfl), c->slot_of.p, c->parent.p, c->mingid.p, c->lrb[1].p,
                       c->counters.p + 15));
        CC_TRY(dist_allreduce_u64(c, c->counters.p + 15, 1));
        CC_CUDA(c, cudaMemcpyAsync(c->h_counters + 15, c->counters.p + 15, sizeof(unsigned long long),
                                   cudaMemcpyDeviceToHost, c->stream));
        CC_CUDA(c, cudaStreamSynchronize(c->stream));
        if (c->h_counters[15] == 0) break;
    }
    if (n_groups) {
        CC_CUDA(c, cudaMemsetAsync(c->counters.p + 8, 0, sizeof(unsigned long long), c->stream));
        if (c->n_in > 0)
            CCL(c, k_count_label_roots<<<(unsigned)((c->n_in + DT - 1) / DT), DT, 0, c->stream>>>(
                       c->n_in, c->slot_of.p, c->parent.p, c->mingid.p, c->orig4.p, c->counters.p + 8));
        CC_TRY(dist_allreduce_u64(c, c->counters.p + 8, 1));
        CC_CUDA(c, cudaMemcpyAsync(c->h_counters + 8, c->counters.p + 8, sizeof(unsigned long long),
                                   cudaMemcpyDeviceToHost, c->stream));
        CC_CUDA(c, cudaStreamSynchronize(c->stream));
        *n_groups = (int64_t)c->h_counters[8];
    }
    return CC_OK;
}

// global halo catalogue (X5): interior components are complete locally; boundary components
// are merged by label across ranks on the host after an allgather.
cc_status dist_halo_sizes(cc_ctx* c, int64_t min_size, std::vector<uint32_t>& out) {
    const int64_t n = c->n;
    const size_t n1 = (size_t)std::max<int64_t>(n, 1);
    CC_TRY(cc_ensure(c, c->gsize, n1, "owned counts"));
    CC_TRY(cc_ensure(c, c->dflag[0], n1, "ghost flags"));
    CC_TRY(cc_ensure(c, c->scratch_u32, n1, "interior sizes"));
    CC_TRY(cc_ensure(c, c->bnd, n1, "boundary components"));
    CC_CUDA(c, cudaMemsetAsync(c->gsize.p, 0, n1 * sizeof(uint32_t), c->stream));
    CC_CUDA(c, cudaMemsetAsync(c->dflag[0].p, 0, n1 * sizeof(uint32_t), c->stream));
    CC_CUDA(c, cudaMemsetAsync(c->counters.p + 10, 0, 2 * sizeof(unsigned long long), c->stream));
    const unsigned nb = (unsigned)((n + DT - 1) / DT);
    if (n > 0) {
        CCL(c, k_root_counts<<<nb, DT, 0, c->stream>>>(n, (uint32_t)c->n_in, c->parent.p, c->dec4.p, c->gsize.p,
                                                       c->dflag[0].p));
        CCL(c, k_root_collect<<<nb, DT, 0, c->stream>>>(n, c->parent.p, c->gsize.p, c->dflag[0].p, c->mingid.p,
                                                        (uint32_t)std::max<int64_t>(min_size, 1), c->scratch_u32.p,
                                                        c->counters.p + 10, c->bnd.p, c->counters.p + 11));
    }
    CC_CUDA(c, cudaMemcpyAsync(c->h_counters + 10, c->counters.p + 10, 2 * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, c->stream));
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    const int64_t ni = (int64_t)c->h_counters[10], nbnd = (int64_t)c->h_counters[11];
    std::vector<uint32_t> interior((size_t)ni);
    if (ni > 0)
        CC_CUDA(c, cudaMemcpyAsync(interior.data(), c->scratch_u32.p, (size_t)ni * sizeof(uint32_t),
                                   cudaMemcpyDeviceToHost, c->stream));
    // allgather the interior sizes and the boundary (label, count) pairs
    CC_TRY(cc_ensure(c, c->dcnt, 4 + 2 * (size_t)c->nranks, "gather counts"));
    long long mine[2] = {ni, nbnd};
    CC_CUDA(c, cudaMemcpyAsync(c->dcnt.p + 4 + 2 * c->rank, mine, 2 * sizeof(long long), cudaMemcpyHostToDevice,
                               c->stream));
    CC_TRY(comm_allgather(c, c->dcnt.p + 4 + 2 * c->rank, c->dcnt.p + 4, 2, CT_I64));
    std::vector<long long> all((size_t)2 * c->nranks);
    CC_CUDA(c, cudaMemcpyAsync(all.data(), c->dcnt.p + 4, all.size() * sizeof(long long), cudaMemcpyDeviceToHost,
                               c->stream));
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    long long mi = 0, mb = 0;
    for (int r = 0; r < c->nranks; r++) {
        mi = std::max(mi, all[2 * r]);
        mb = std::max(mb, all[2 * r + 1]);
    }
    // padded allgather: [interior sizes (mi) | boundary pairs (2 mb)] per rank
    const size_t per = (size_t)(mi + 2 * mb);
    CC_TRY(cc_ensure(c, c->gath, std::max<size_t>(per * (size_t)(c->nranks + 1), 1), "gather buffer"));
    uint32_t* mineb = c->gath.p + per * (size_t)c->nranks;
    CC_CUDA(c, cudaMemsetAsync(mineb, 0, std::max<size_t>(per, 1) * sizeof(uint32_t), c->stream));
    if (ni > 0)
        CC_CUDA(c, cudaMemcpyAsync(mineb, c->scratch_u32.p, (size_t)ni * sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                                   c->stream));
    if (nbnd > 0)
        CC_CUDA(c, cudaMemcpyAsync(mineb + mi, c->bnd.p, (size_t)nbnd * sizeof(uint2), cudaMemcpyDeviceToDevice,
                                   c->stream));
    if (per > 0) CC_TRY(comm_allgather(c, mineb, c->gath.p, per, CT_U32));
    std::vector<uint32_t> h(per * (size_t)c->nranks);
    if (!h.empty())
        CC_CUDA(c, cudaMemcpyAsync(h.data(), c->gath.p, h.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                                   c->stream));
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    out.clear();
    std::unordered_map<uint32_t, uint64_t> merged;
    for (int r = 0; r < c->nranks; r++) {
        const uint32_t* b = h.data() + per * (size_t)r;
        for (long long k = 0; k < all[2 * r]; k++) out.push_back(b[k]);
        for (long long k = 0; k < all[2 * r + 1]; k++) merged[b[mi + 2 * k]] += b[mi + 2 * k + 1];
    }
    for (auto& kv : merged)
        if ((int64_t)kv.second >= min_size) out.push_back((uint32_t)kv.second);
    std::sort(out.begin(), out.end(), [](uint32_t a, uint32_t b) { return a > b; });
    return CC_OK;
}

cc_status dist_unique_id(void* out) {
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return CC_E_NCCL;
    std::memcpy(out, &id, sizeof(id));
    return CC_OK;
}

}  // namespace cc
