// cc_internal.cuh -- shared internals of libcc (the CUDA path).  Independent of oracle/.
//
// Data layout in HBM:
//   per local particle, cell-sorted "slot" order s:
//     orig4[s] = (x, y, z, gid bits)          float4, original P           (S1)
//     dec4[s]  = (xh, yh, zh, input index i)  float4, decompressed P_hat^(0)
//     cell_start[c]  u32 (n_cell + 1), slot_of[i] u32 (input index -> slot)
//     deg[s] u32 (band partners), eidx[s] u32 (editable index or 0xFFFFFFFF)
//   per editable particle e (class-major, slot order within a class, S3):
//     posA/posB[e] float4 (x, y, z, gid bits) ping-pong, origE[e] float4, slotE[e] u32,
//     rowptr[e] u64, Adam moments m,v as 6 float SoA arrays
//   rows[k] u32 (2|V| directed entries, sorted by partner gid within a row):
//     bits 0..29 partner editable index, bit 30 partner gid > own gid, bit 31 original link
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <string>
#include <vector>

#include "../../include/cc.h"

namespace cc {

constexpr uint32_t ENT_IDX = 0x3FFFFFFFu;
constexpr uint32_t ENT_UPPER = 0x40000000u;
constexpr uint32_t ENT_OLINK = 0x80000000u;
constexpr int64_t MAX_LOCAL = (int64_t)1 << 30;

// fp32 thresholds of S0 (computed on the host in fp64, rounded once; R2-R8)
struct Th {
    float Lf, hLf;     // fl32(L), fl32(L/2)
    float xi_f;        // fl32(xi)
    float xip_f;       // RD32(xi_f (1 - 2^-m))
    float b2;          // fl32(b^2)
    float lo2, hi2;    // fl32((b -/+ 2 sqrt3 xi)^2); lo2 = -1 if b - 2 sqrt3 xi <= 0
    float c_b, c_f;    // fl32(b -/+ 2 sqrt3 eps_q)
    int periodic;
    // Proven link status under ANY positions within xi_f of the originals (DESIGN.md §5,
    // "stable and near shells"): original d2 <= lo2s  =>  linked in every such position set;
    // d2 > hi2s  =>  unlinked in every one -- rigorous bounds through the fp32 rounding of the
    // pinned expression.  _i: interior pairs (no minimum-image wrap; relative rounding only),
    // _w: pairs near a periodic face (the wrap adds an absolute error u (L + 2 xi)).  Pairs in
    // (lo2s, lo2] or (hi2, hi2s] form the near-shell list re-tested on the positions.
    float lo2s_i, hi2s_i, lo2s_w, hi2s_w;
    // Eq. 3 activity on the squared distance (K3 skips the square root of inactive pairs):
    // sqrt_rn(s) > c_b  <=>  s > sb2,  sqrt_rn(s) <= c_f  <=>  s <= sf2 (sqrt_rn is monotone;
    // sb2/sf2 = the largest fp32 s with sqrt_rn(s) <= c_b / c_f, found on the host)
    float sb2, sf2;
};

// Search structure on ORIGINAL positions ("x-sorted rows"): the (y,z) plane is cut into
// ny x nz rows of side >= r_max = (b + 2 sqrt3 xi)(1 + 1e-5); each row is cut along x into nx
// bins; particles are counting-sorted by (z-row, y-row, x-bin) and sorted by x inside every bin,
// so every row is one x-sorted slot range.  A radius-r search from a particle visits the 9
// neighbouring rows and, in each, only the x-window [u - r, u + r] (binary search on the x keys xk[]).
// Coordinates: u = x - x0 wrapped once into [0, L) (x0 = 0 on one GPU; the slab's lower ghost
// edge on several); all window arithmetic in fp64.
struct Grid {
    int nx, ny, nz;
    double inv_w;      // rows per unit length in y and z
    double margin;     // 2.5 row widths: interior() (host-computed: no fp64 division in kernels)
    double inv_wx;     // x-bins per unit length
    double x0;         // lower x edge of the local grid
    double L;          // box
    double ext_x;      // x extent of the local grid (L on one GPU)
    int xwrap;         // 1: x axis periodic inside this grid (single GPU)
};

// per-iteration control block of the PGD loop (device resident)
struct Ctl {
    int done;          // 1 once the loop has ended (later launches return immediately)
    int t;             // iterations whose stop check has run
    int t_res;         // updates contained in the result buffer
    int converged;
    unsigned int ticket;
    int sel;           // K3: this launch processes only the bitmap-selected editables (pgd.cu)
    int bld;           // K3: this launch builds the awake/touched bitmaps
    unsigned int nsel; // K3: short-row editables selected for the next k_pgd (k_select)
    unsigned int nsel_l;  // K3: long-row editables selected (stored from slist[e_short])
    unsigned long long active;   // L_tight-active pairs at the last check
    unsigned long long violated; // pairs whose link status differs from the original (Eq. 1)
    double loss;
    int loss_le;                 // L_tight <= eps_L at the last check, decided exactly (lfx_le)
    unsigned long long acc[14];  // K3 launch statistics being summed (LFX layout + schedule counts)
    unsigned int tail_nn;        // k_tail: length of the list being built
    unsigned int tail_ncur;      // k_tail: length of the list of the next iteration
    int tail_go;                 // k_tail: 1 while the tail loop continues
    unsigned int bar_count, bar_gen;  // k_tail's grid barrier
    unsigned int ep_base;        // multi-GPU peer exchange: epoch of iteration t is ep_base + t
};

// ---------------------------------------------------------------------------------------
// exact, order-independent L_tight sum (R28).  Every term ee^2 (ee fp32, so ee^2 is
// exact in fp64) is truncated to a multiple of 2^-LFX_UNIT and added as 32-bit digits into
// 64-bit limbs: integer sums, so any summation order -- threads, blocks, ranks -- gives the
// same loss, and the stop decision (R11) is bit-identical for any grid or rank count.
// Statistics words: [0] active pairs, [1] violated pairs, [2..7] loss limbs (limb k weighs
// 2^(32k - LFX_UNIT)); range [2^-140, 2^52).
constexpr int LFX_UNIT = 140;
constexpr int LFX_STATS = 8;

template <int STRIDE = 1>
__device__ __forceinline__ void lfx_add(unsigned long long* l, double d) {
    if (!(d > 0.0)) return;
    const unsigned long long bits = (unsigned long long)__double_as_longlong(d);
    const int ex = (int)((bits >> 52) & 0x7FF);
    unsigned long long m = (bits & 0xFFFFFFFFFFFFFull) | (ex ? (1ull << 52) : 0ull);
    int s = (ex ? ex : 1) - 1075 + LFX_UNIT;  // d = m * 2^(s - LFX_UNIT)
    if (s < 0) {
        if (s <= -64) return;
        m >>= -s;
        s = 0;
    }
    const int k0 = s >> 5, off = s & 31;
#pragma unroll
    for (int k = 0; k < 6; k++) {
        unsigned long long part = 0ull;
        if (k == k0) part = (m << off) & 0xFFFFFFFFull;
        else if (k == k0 + 1) part = (m >> (32 - off)) & 0xFFFFFFFFull;
        else if (k == k0 + 2 && off) part = (m >> (64 - off)) & 0xFFFFFFFFull;
        if (part) l[k * STRIDE] += part;
    }
}

// value of the limbs: carries normalised, then summed from the top in fp64 (fixed order)
__host__ __device__ inline double lfx_value(const unsigned long long* l) {
    unsigned long long d[6], carry = 0ull;
    for (int k = 0; k < 6; k++) {
        const unsigned long long v = l[k] + carry;  // < 2^64: carry < 2^32 and l[k] < 2^63
        d[k] = v & 0xFFFFFFFFull;
        carry = v >> 32;
    }
    double r = (double)carry;
    for (int k = 5; k >= 0; k--) r = r * 4294967296.0 + (double)d[k];
    // scale by 2^-LFX_UNIT in two exact steps
    const double s70 = 8.470329472543003e-22;  // 2^-70
    return r * s70 * s70;
}

// Exact stop test of Alg. 1 line 6: sum(limbs) <= v, decided on the exact integer
// digits (never on the rounded lfx_value).  Every L_tight term e^2 is a multiple of
// (ulp(c)/2)^2 (e = fl(d_hat - c) is a multiple of ulp(c)/2 for c = c_b or c_f), so for
// c >= 2^-46 the truncation to 2^-LFX_UNIT in lfx_add drops nothing and the limbs hold the
// real number L_tight exactly; the sum is then a multiple of 2^-LFX_UNIT and
// sum <= v  <=>  sum <= floor(v 2^LFX_UNIT) 2^-LFX_UNIT.
__host__ __device__ inline bool lfx_le(const unsigned long long* l, double v) {
    if (!(v >= 0.0)) return false;  // the sum is >= 0; NaN never holds
    unsigned long long sd[7], vd[7] = {0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull}, carry = 0ull;
    for (int k = 0; k < 6; k++) {
        const unsigned long long x = l[k] + carry;
        sd[k] = x & 0xFFFFFFFFull;
        carry = x >> 32;
    }
    sd[6] = carry;
    const double two52 = 4503599627370496.0;
    if (v >= two52) return true;  // beyond the limbs' range [2^-140, 2^52)
    // v = mant 2^(ex - 1075), digits of floor(v 2^LFX_UNIT)
    unsigned long long bits;
    memcpy(&bits, &v, sizeof(bits));
    const int ex = (int)((bits >> 52) & 0x7FF);
    unsigned long long m = (bits & 0xFFFFFFFFFFFFFull) | (ex ? (1ull << 52) : 0ull);
    int s = (ex ? ex : 1) - 1075 + LFX_UNIT;
    if (s < 0) {
        m = s <= -64 ? 0ull : (m >> -s);
        s = 0;
    }
    const int k0 = s >> 5, off = s & 31;
    for (int k = 0; k < 7; k++) {
        if (k == k0) vd[k] = (m << off) & 0xFFFFFFFFull;
        else if (k == k0 + 1) vd[k] = (m >> (32 - off)) & 0xFFFFFFFFull;
        else if (k == k0 + 2 && off) vd[k] = (m >> (64 - off)) & 0xFFFFFFFFull;
    }
    for (int k = 6; k >= 0; k--)
        if (sd[k] != vd[k]) return sd[k] < vd[k];
    return true;
}

template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t cap = 0;  // elements
};

struct ProfEntry {
    std::string name;
    double ms = 0.0;
    int64_t launches = 0;
};

struct PendingEv {
    int cls;
    cudaEvent_t a, b;
};

}  // namespace cc

struct cc_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cc_params p{};
    int rank = 0, nranks = 1;
    void* nccl_comm = nullptr;
    void* vgroup = nullptr;  // in-process virtual ranks (comm.cu) instead of NCCL
    int comm_depth = 0;      // open comm groups (virtual ranks)
    std::string err;
    int state = 0;  // 0 created, 1 cells, 2 pairs, 3 corrected
    bool dead = false;
    bool owns_stream = false;
    int64_t launches = 0;  // kernels launched by this context (incl. graph-launched ones)

    // S0
    cc::Th th{};
    double b = 0, xi_d = 0, eps_q = 0, mu = 0, delta = 0;
    cc::Grid g{};
    int64_t ncell = 0;
    int bin_short_max = 16;  // K1 finish: cells up to this size sorted by one thread, larger by a warp / block

    // sizes
    int64_t n_in = 0;      // particles given by the caller (owned)
    int64_t n = 0;         // local particles (owned + ghost)
    int64_t E = 0;         // editable (owned rows)
    int64_t E_all = 0;     // editable incl. ghost partners (multi-GPU)
    int64_t nent = 0;      // directed row entries

    // device buffers
    cc::DBuf<float4> orig4, dec4, cor4, posA, posB, origE;
    bool cor4_valid = false;  // cor4 matches the last cc_correct (built on demand)
    bool slot_of_valid = false;  // slot_of completed since the last build (ensure_slot_of)
    const float* in_dec[3] = {nullptr, nullptr, nullptr};  // decompressed inputs of the last build (input order)
    cc::DBuf<uint32_t> key, rnk, cell_count, cell_start, slot_of, deg, eidx, rows, slotE, parent, mingid,
        gsize, scratch_u32;
    cc::DBuf<uint64_t> rowptr, scratch_u64;
    cc::DBuf<uint32_t> xk;       // x_sort_key of the original x per slot (the in-row search key)
    cc::DBuf<uint4> rec32;       // K1 binning records, 2 x uint4 = 32 B per particle
    cc::DBuf<uint32_t> parent_base;  // FoF forest of the stable links (d2 <= lo2), per build
    bool base_valid = false;
    cc::DBuf<uint32_t> gp_cnt, gp_pos;  // cc_get_pairs: counting sort by owner gid
    cc::DBuf<uint2> near;        // near-shell pairs (slot, slot | bit 31 = linked in the original), K2 count
    cc::DBuf<unsigned long long> near_n;  // their count (may exceed near.cap: then FoF searches directly)
    int64_t near_count = 0;      // host copy after cc_find_vulnerable
    double r_pair = 0, r_link = 0;   // search radii: vulnerable band / FoF on original positions
    cc::DBuf<float> mom;         // 6 * E floats: mx, my, mz, vx, vy, vz
    cc::DBuf<float2> bc;         // Adam bias corrections per iteration
    cc::DBuf<unsigned long long> counters;
    cc::DBuf<cc::Ctl> ctl;
    cc::DBuf<long long> trace_a, trace_v, trace_s;
    cc::DBuf<uint32_t> lab_s;     // FoF labels in slot order (fof.cu)
    cc::DBuf<uint32_t> frozen, fbits, slist, tlist;  // K3 frontier: last-processed iteration, awake/touched bitmaps (pgd.cu)
    cc::DBuf<unsigned long long> k3work;  // work totals: K3 editables updated, entries evaluated; K2 count / fill and K4 pair tests
    int64_t E_cls[4] = {0, 0, 0, 0};  // editables per K3 work class (row_class), numbered class-major
    cc::DBuf<double> trace_l;
    cc::DBuf<unsigned char> tmp_bytes;  // scan scratch
    cc::DBuf<unsigned long long> codec_bsum;  // f1 edit log: block sums + total + error flag
    cc::DBuf<unsigned long long> codec_status;  // f1 single-pass encode: per-tile look-back status, ticket, total
    cc::DBuf<float> in_f;        // cc_run host staging: 6 n floats
    cc::DBuf<uint32_t> in_gid;

    // multi-GPU (dist.cu)
    int left = 0, right = 0;
    double slab_lo = 0, slab_hi = 0;
    cc::DBuf<uint32_t> dflag[2], dpos[2], shell[2], stage, sbuf7[2], rbuf7[2], req[2], recv_e[2], sreq[2], send_e[2],
        lsb[2], lrb[2], gath;
    cc::DBuf<long long> dcnt;
    cc::DBuf<float4> rsb[2], rrb[2];
    cc::DBuf<unsigned long long> red;  // K3 stop statistics (LFX_STATS words) for the allreduce
    cc::DBuf<uint2> bnd;
    int64_t n_shell[2] = {0, 0}, n_from_left = 0, n_from_right = 0, stage_cap = 0;
    int64_t n_ref_send[2] = {0, 0}, n_ref_recv[2] = {0, 0};
    int64_t launches_per_iter_tail = 0;
    // per-iteration exchange over NVLink peer memory (dist.cu): one cudaMalloc'd block per rank
    // (flags, stop statistics, two parities of the two ghost-refresh receive areas), mapped by
    // every peer through CUDA IPC
    void* pm_local = nullptr;
    size_t pm_bytes = 0;
    int64_t pm_cap[2] = {0, 0};
    void* pm_peer[8] = {};
    unsigned char pm_handle[8][64] = {};
    int64_t pm_peer_cap[8][2] = {};
    bool pm_ok = false;
    unsigned int epoch_base = 0;
    cc::DBuf<unsigned long long> red_sum;
    unsigned long long* h_red = nullptr;
    unsigned long long final_active = 0;
    double final_loss = 0.0;
    unsigned long long final_violated = 0;

    // pinned host mirrors
    cc::Ctl* h_ctl = nullptr;
    unsigned long long* h_counters = nullptr;

    // PGD graph cache
    cudaGraphExec_t pgd_exec = nullptr;
    std::vector<unsigned char> pgd_sig;  // arguments baked into pgd_exec (re-capture on change)
    int last_iters = 0;
    int fof_which = -1;
    int have_labels[3] = {0, 0, 0};

    // profiling
    std::vector<cc::ProfEntry> prof;
    std::vector<cc::PendingEv> pend;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<cudaEvent_t> graph_ev;    // 2*batch events recorded inside the PGD graph
};

namespace cc {

// K3 work classes by row length (editables are numbered class-major, slot order inside a
// class): 0: 1..4 entries (thread, one batch), 1: 5..16, 2: 17..32 (thread, uniform trip
// counts per warp), 3: > 32 (one warp per row)
__host__ __device__ inline int row_class(uint32_t len) { return len <= 4u ? 0 : (len <= 16u ? 1 : (len <= 32u ? 2 : 3)); }

// Alg. 1 line 6 stop test per stop mode (R11): ACTIVE: no L_tight-active pair;
// EPS: L_tight <= eps_L; RESTORED: L_tight <= eps_L and every link status restored (MCC = 1)
// loss_le: L_tight <= eps_L decided exactly (lfx_le)
__host__ __device__ inline bool stop_rule(int mode, unsigned long long active, bool loss_le,
                                          unsigned long long violated) {
    if (mode == CC_STOP_ACTIVE) return active == 0ull;
    if (mode == CC_STOP_EPS) return loss_le;
    if (mode == CC_STOP_RESTORED) return violated == 0ull && loss_le;
    return false;
}

// ---------------------------------------------------------------------------------------
// pinned fp32 distance arithmetic (R4): explicit round-to-nearest intrinsics, no
// FMA contraction (the library is also compiled with -fmad=false).
__device__ __forceinline__ float min_image(float d, const Th& t) {
    if (t.periodic) {
        if (d > t.hLf) d = __fsub_rn(d, t.Lf);
        else if (d < -t.hLf) d = __fadd_rn(d, t.Lf);
    }
    return d;
}

// squared distance from particle a to particle b: dx = fl(b.x - a.x) ...
__device__ __forceinline__ float dist2(const float4& a, const float4& b, const Th& t) {
    float dx = min_image(__fsub_rn(b.x, a.x), t);
    float dy = min_image(__fsub_rn(b.y, a.y), t);
    float dz = min_image(__fsub_rn(b.z, a.z), t);
    float s = __fmul_rn(dx, dx);
    s = __fadd_rn(s, __fmul_rn(dy, dy));
    s = __fadd_rn(s, __fmul_rn(dz, dz));
    return s;
}

// lock-free union-find (FoF, K2's stable links): roots are hooked larger-under-smaller with
// atomicCAS, finds path-halve (every write replaces a parent by one of its ancestors)
// relaxed GPU-scope accesses of the union-find forest (every writer is on this GPU; `volatile`
// compiled to system-scope strong loads, ~2x the latency on the stable-forest unions of K2)
__device__ __forceinline__ uint32_t ld_rlx(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rlx(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t uf_find(uint32_t* par, uint32_t x) {
    for (;;) {
        const uint32_t p = ld_rlx(par + x);
        if (p == x) return x;
        const uint32_t gp = ld_rlx(par + p);
        if (gp != p) st_rlx(par + x, gp);
        x = gp;
    }
}

// returns a root the two sets shared when the call ended (an ancestor of both from then on)
__device__ __forceinline__ uint32_t uf_unite(uint32_t* par, uint32_t a, uint32_t b) {
    a = uf_find(par, a);
    b = uf_find(par, b);
    while (a != b) {
        if (a < b) {
            const uint32_t t = a;
            a = b;
            b = t;
        }
        const uint32_t old = atomicCAS(&par[a], a, b);  // hook root a (larger) under b
        if (old == a) return b;
        a = uf_find(par, old);
        b = uf_find(par, b);
    }
    return a;
}

// Link s with j unless they are visibly in one set already: rs is a cached ancestor of s (sets
// only merge, so a stale parent/grandparent of j equal to rs proves it); dense halo cores meet
// mostly redundant links, which this filter turns from two L2 root walks into L1 loads.
__device__ __forceinline__ void uf_link(uint32_t* par, uint32_t s, uint32_t j, uint32_t& rs) {
    const uint32_t pj = par[j];
    if (pj == rs) return;
    if (par[pj] == rs) return;
    rs = uf_unite(par, s, j);
}

__device__ __forceinline__ int cell_coord(double x, double x0, double inv_w, int n) {
    double f = floor((x - x0) * inv_w);
    int c = (f < 0.0) ? 0 : (f > (double)(n - 1) ? n - 1 : (int)f);
    return c;
}

// local x coordinate: x - x0 wrapped once into [0, L) (identity on one GPU)
__device__ __forceinline__ double local_u(double x, const Grid& g) {
    double u = x - g.x0;
    if (u < 0.0) u += g.L;
    else if (u >= g.L) u -= g.L;
    return u;
}

// the (x-bin, y-row, z-row) of an ORIGINAL position; u = its local x coordinate
__device__ __forceinline__ void cell_of(float x, float y, float z, const Grid& g, double& u, int& cx, int& cy,
                                        int& cz) {
    u = local_u((double)x, g);
    cx = cell_coord(u, 0.0, g.inv_wx, g.nx);
    cy = cell_coord((double)y, 0.0, g.inv_w, g.ny);
    cz = cell_coord((double)z, 0.0, g.inv_w, g.nz);
}

// 32-bit in-row sort key of an original x: order of u = (x < x0 ? 1 : 0, x) (x >= 0 assumed,
// -0 folded into +0), exact -- no rounding of u is involved.
__device__ __forceinline__ uint32_t x_sort_key(float x, const Grid& g) {
    const float xp = __fadd_rn(x, 0.0f);
    const uint32_t wrapped = ((double)x < g.x0) ? 0x80000000u : 0u;
    return __float_as_uint(xp) | wrapped;
}

__device__ __forceinline__ int wrapi(int a, int n) { return a < 0 ? a + n : (a >= n ? a - n : a); }

// in-row key bounds of a local-x window [a, b] (0 <= a, b <= L): every slot with a <= u <= b
// has key_lo(a) <= key <= key_hi(b) (directed fp32 rounding widens, never narrows; the exact
// distance test filters the candidates afterwards)
__device__ __forceinline__ uint32_t key_lo(double a, const Grid& g) {
    double x = a + g.x0;
    uint32_t w = 0u;
    if (x >= g.L) {
        x -= g.L;
        w = 0x80000000u;
    }
    return __float_as_uint(__fadd_rn(__double2float_rd(fmax(x, 0.0)), 0.0f)) | w;
}
__device__ __forceinline__ uint32_t key_hi(double b, const Grid& g) {
    double x = b + g.x0;
    uint32_t w = 0u;
    if (x >= g.L) {
        x -= g.L;
        w = 0x80000000u;
    }
    return __float_as_uint(__fadd_rn(__double2float_ru(fmax(x, 0.0)), 0.0f)) | w;
}

// first slot j in [j0, j1) with xk[j] >= k (keys non-decreasing over the range)
__device__ __forceinline__ uint32_t lower_bound_key(const uint32_t* __restrict__ xk, uint32_t j0, uint32_t j1,
                                                    uint32_t k) {
    while (j0 < j1) {
        const uint32_t m = (j0 + j1) >> 1;
        if (xk[m] < k) j0 = m + 1;
        else j1 = m;
    }
    return j0;
}

// visit every slot j of the row starting at cell index `rowbase` with a <= u_j <= b
template <class F>
__device__ __forceinline__ void scan_row_window(const Grid& g, const uint32_t* __restrict__ cs,
                                                const uint32_t* __restrict__ xk, int64_t rowbase, double a, double b,
                                                F& f) {
    const int ca = cell_coord(a, 0.0, g.inv_wx, g.nx), cb = cell_coord(b, 0.0, g.inv_wx, g.nx);
    const uint32_t j1 = cs[rowbase + cb + 1];
    const uint32_t khi = key_hi(b, g);
    uint32_t j = lower_bound_key(xk, cs[rowbase + ca], j1, key_lo(a, g));
    for (; j < j1; j++) {
        if (xk[j] > khi) break;
        f(j);
    }
}

// visit the x-window [u - r, u + r] (periodic in x when g.xwrap) of one row
template <class F>
__device__ __forceinline__ void scan_row(const Grid& g, const uint32_t* __restrict__ cs, const uint32_t* __restrict__ xk,
                                         int64_t rowbase, double u, double r, F& f) {
    double a = u - r, b = u + r;
    double sa[3], sb[3];
    int ns = 0;
    if (g.xwrap) {
        if (a < 0.0) {
            sa[ns] = a + g.L;
            sb[ns++] = g.L;
            a = 0.0;
        }
        if (b >= g.L) {
            sa[ns] = 0.0;
            sb[ns++] = b - g.L;
            b = g.L;
        }
    } else {
        if (a < 0.0) a = 0.0;
        if (b > g.ext_x) b = g.ext_x;
    }
    sa[ns] = a;
    sb[ns++] = b;
#pragma unroll 1
    for (int k = 0; k < ns; k++) scan_row_window(g, cs, xk, rowbase, sa[k], sb[k], f);
}

// Radius-r candidates of a particle at local x u in row (cy, cz): the 9 neighbouring rows
// (offsets de-duplicated when an axis has fewer than 3 rows, R1), x-window per row.  f(j).
template <class F>
__device__ __forceinline__ void for_each_candidate(const Grid& g, const uint32_t* __restrict__ cs,
                                                   const uint32_t* __restrict__ xk, double u, int cy, int cz, double r,
                                                   bool periodic_yz, F&& f) {
    const int ny_off = g.ny >= 3 ? 3 : g.ny, nz_off = g.nz >= 3 ? 3 : g.nz;
    const int offs[3] = {0, 1, -1};
#pragma unroll 1
    for (int kz = 0; kz < nz_off; kz++) {
        int zz = cz + offs[kz];
        if (periodic_yz) zz = wrapi(zz, g.nz);
        else if (zz < 0 || zz >= g.nz) continue;
#pragma unroll 1
        for (int ky = 0; ky < ny_off; ky++) {
            int yy = cy + offs[ky];
            if (periodic_yz) yy = wrapi(yy, g.ny);
            else if (yy < 0 || yy >= g.ny) continue;
            scan_row(g, cs, xk, ((int64_t)zz * g.ny + yy) * g.nx, u, r, f);
        }
    }
}

// x-window of one search (identical for every row it visits): at most two segments of local x
// (the periodic seam splits it on one GPU), each as (first x-bin, last x-bin, key bounds).  The
// window math (fp64 floor, directed key rounding) is done once per particle, not once per row.
struct XWin {
    int n;            // segments (1 or 2)
    bool up;          // segment 1 is the part above the seam, [0, u + r - L]
    int ca[2], cb[2]; // first / last x-bin of each segment
    uint32_t klo[2], khi[2];
};

__device__ __forceinline__ XWin make_xwin(const Grid& g, double u, double r) {
    XWin w;
    double a = u - r, b = u + r, a1 = 0.0, b1 = -1.0;
    w.up = false;
    if (g.xwrap) {
        if (a < 0.0) {
            a1 = a + g.L;
            b1 = g.L;
            a = 0.0;
        } else if (b >= g.L) {
            a1 = 0.0;
            b1 = b - g.L;
            b = g.L;
            w.up = true;
        }
    } else {
        if (a < 0.0) a = 0.0;
        if (b > g.ext_x) b = g.ext_x;
    }
    w.n = b1 >= a1 ? 2 : 1;
    w.ca[0] = cell_coord(a, 0.0, g.inv_wx, g.nx);
    w.cb[0] = cell_coord(b, 0.0, g.inv_wx, g.nx);
    w.klo[0] = key_lo(a, g);
    w.khi[0] = key_hi(b, g);
    w.ca[1] = cell_coord(a1, 0.0, g.inv_wx, g.nx);
    w.cb[1] = cell_coord(fmax(b1, a1), 0.0, g.inv_wx, g.nx);
    w.klo[1] = key_lo(a1, g);
    w.khi[1] = key_hi(fmax(b1, a1), g);
    return w;
}

// visit the slots of one row inside window segment k (j0/j1 = the bin range's slots)
template <class F>
__device__ __forceinline__ void scan_seg(const uint32_t* __restrict__ xk, uint32_t j0, uint32_t j1, uint32_t klo,
                                         uint32_t khi, F& f) {
    uint32_t j = lower_bound_key(xk, j0, j1, klo);
    for (; j < j1; j++) {
        if (xk[j] > khi) break;
        f(j);
    }
}

// Every unordered pair {s, j} within radius r, visited once over all s: the half-shell of rows
// (own row forward in slot = x order plus the periodic wrap at the row start, then rows
// (dz=0,dy=+1) and (dz=+1,dy=-1..1)); with fewer than 3 periodic rows on an axis, all 9 rows
// with j > s.  f(j) for each candidate j (the caller tests the distance).
template <class F>
__device__ __forceinline__ void for_each_pair_forward(const Grid& g, const uint32_t* __restrict__ cs,
                                                      const uint32_t* __restrict__ xk, uint32_t s, double u, int cy,
                                                      int cz, double r, bool periodic_yz, F&& f) {
    const bool half = !periodic_yz || (g.ny >= 3 && g.nz >= 3);
    if (!half) {
        auto fwd = [&](uint32_t j) {
            if (j > s) f(j);
        };
        for_each_candidate(g, cs, xk, u, cy, cz, r, periodic_yz, fwd);
        return;
    }
    if (g.nx == 1) {
        // cells are whole rows (the default grid): the x-window's key bounds are the same for
        // all 5 rows -- computed once; each row is one slot range searched by its keys
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
        {   // own row: forward in slot (= x) order, then the part above the seam at the row start
            const int64_t row = (int64_t)cz * g.ny + cy;
            const uint32_t row_end = cs[row + 1];
            for (uint32_t j = s + 1; j < row_end; j++) {
                if (xk[j] > khi0) break;
                f(j);
            }
            if (two && up) {
                for (uint32_t j = cs[row]; j < s; j++) {
                    if (xk[j] > khi1) break;
                    f(j);
                }
            }
        }
        const int rows_dz[4] = {0, 1, 1, 1};
        const int rows_dy[4] = {1, -1, 0, 1};
#pragma unroll 1
        for (int k = 0; k < 4; k++) {
            int zz = cz + rows_dz[k], yy = cy + rows_dy[k];
            if (periodic_yz) {
                zz = wrapi(zz, g.nz);
                yy = wrapi(yy, g.ny);
            } else if (zz < 0 || zz >= g.nz || yy < 0 || yy >= g.ny) {
                continue;
            }
            const int64_t row = (int64_t)zz * g.ny + yy;
            const uint32_t j0 = cs[row], j1 = cs[row + 1];
            for (uint32_t j = lower_bound_key(xk, j0, j1, klo0); j < j1; j++) {
                if (xk[j] > khi0) break;
                f(j);
            }
            if (two)
                for (uint32_t j = lower_bound_key(xk, j0, j1, klo1); j < j1; j++) {
                    if (xk[j] > khi1) break;
                    f(j);
                }
        }
        return;
    }
    {
        const int64_t rowbase = ((int64_t)cz * g.ny + cy) * g.nx;
        const double b = u + r;
        const uint32_t row_end = cs[rowbase + g.nx];
        const uint32_t khi = key_hi(fmin(b, g.xwrap ? g.L : g.ext_x), g);
        for (uint32_t j = s + 1; j < row_end; j++) {
            if (xk[j] > khi) break;
            f(j);
        }
        if (g.xwrap && b >= g.L) scan_row_window(g, cs, xk, rowbase, 0.0, b - g.L, f);
    }
    const int rows_dz[4] = {0, 1, 1, 1};
    const int rows_dy[4] = {1, -1, 0, 1};
#pragma unroll 1
    for (int k = 0; k < 4; k++) {
        int zz = cz + rows_dz[k], yy = cy + rows_dy[k];
        if (periodic_yz) {
            zz = wrapi(zz, g.nz);
            yy = wrapi(yy, g.ny);
        } else if (zz < 0 || zz >= g.nz || yy < 0 || yy >= g.ny) {
            continue;
        }
        scan_row(g, cs, xk, ((int64_t)zz * g.ny + yy) * g.nx, u, r, f);
    }
}

// per-warp sum of a per-thread counter into a global total (one atomic per warp; callable after
// an early return of some lanes)
// ascending in-place sort of v[0..len) in global memory by one block, for the rare rows too long
// for shared memory (K1 rows, K2 rows): bitonic network in its all-ascending form (each merge
// phase opens with the mirror comparator i <-> i ^ (kk-1), then half-cleaners i <-> i | j), so
// every comparator puts the minimum at the lower index and the virtual +inf padding beyond len
// never moves: comparators reaching past len are skipped.  key(x) = a unique sort key.
// O(len log^2 len) comparators, block-synchronised per step.
template <class T, class K>
__device__ void block_sort_global(T* v, int64_t len, const K& key) {
    int64_t p2 = 1;
    while (p2 < len) p2 <<= 1;
    for (int64_t kk = 2; kk <= p2; kk <<= 1) {
        for (int64_t j = kk >> 1; j > 0; j >>= 1) {
            for (int64_t t = threadIdx.x; t < (p2 >> 1); t += blockDim.x) {
                const int64_t i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
                const int64_t q = (j == (kk >> 1)) ? (i ^ (kk - 1)) : (i | j);
                if (q < len) {
                    const T a = v[i], b = v[q];
                    if (key(a) > key(b)) {
                        v[i] = b;
                        v[q] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// decoupled look-back of the single-pass scans (K2's editable list, f1's encode).  A tile's
// status word = 2 flag bits (aggregate published / inclusive prefix published) | 62-bit value.
// Called by warp 0 of the block owning `tile` with the tile's aggregate: publishes it, sums the
// predecessors' values (32 per step) back to the nearest published inclusive prefix, publishes
// its own inclusive prefix and returns the exclusive prefix (on every lane).  Tiles are taken in
// ticket order, so every predecessor is running or done: the spin terminates.
constexpr unsigned long long LB_AGG = 1ull << 62, LB_PRE = 2ull << 62, LB_VAL = (1ull << 62) - 1ull;

__device__ __forceinline__ unsigned long long lookback_warp0(unsigned long long* status, unsigned tile,
                                                             unsigned long long tot) {
    const int lane = threadIdx.x & 31;
    volatile unsigned long long* st = status;
    if (tile == 0) {
        if (lane == 0) st[0] = LB_PRE | tot;
        return 0ull;
    }
    if (lane == 0) {
        st[tile] = LB_AGG | tot;
        __threadfence();
    }
    __syncwarp();
    unsigned long long acc = 0ull;
    long long top = (long long)tile - 1;  // predecessors top, top-1, ... in this window
    for (;;) {
        const long long pi = top - lane;
        unsigned long long v = 0ull;
        bool ready;
        do {
            v = pi >= 0 ? st[pi] : (LB_PRE | 0ull);
            ready = (v >> 62) != 0ull;
        } while (!__all_sync(0xffffffffu, ready));
        const unsigned pre = __ballot_sync(0xffffffffu, (v >> 62) == 2ull);
        const int stop = pre ? __ffs(pre) - 1 : 32;  // nearest predecessor with a prefix
        unsigned long long add = lane <= stop ? (v & LB_VAL) : 0ull;
        for (int o = 16; o > 0; o >>= 1) add += __shfl_xor_sync(0xffffffffu, add, o);
        acc += add;
        if (pre) break;
        top -= 32;
    }
    if (lane == 0) {
        __threadfence();
        st[tile] = LB_PRE | (acc + tot);
    }
    return acc;
}

__device__ __forceinline__ void warp_count(unsigned long long* dst, unsigned v) {
    const unsigned m = __activemask();
    const unsigned x = __reduce_add_sync(m, v);
    if ((threadIdx.x & 31) == (unsigned)(__ffs(m) - 1) && x) atomicAdd(dst, (unsigned long long)x);
}

// pinned d2 without the minimum image: identical to dist2 whenever no coordinate difference
// can exceed L/2, i.e. for particles away from the periodic faces (interior below)
__device__ __forceinline__ float dist2_nw(const float4& a, const float4& b) {
    const float dx = __fsub_rn(b.x, a.x), dy = __fsub_rn(b.y, a.y), dz = __fsub_rn(b.z, a.z);
    float s = __fmul_rn(dx, dx);
    s = __fadd_rn(s, __fmul_rn(dy, dy));
    s = __fadd_rn(s, __fmul_rn(dz, dz));
    return s;
}

// true if every candidate of a search around this ORIGINAL position (rows +-1 of width w >= r,
// x-window r; positions within xi of the originals) has |difference| far below L/2 on every axis,
// so min_image is the identity: the particle keeps >= 2.5 w from the periodic faces
__device__ __forceinline__ bool interior(float x, float y, float z, const Grid& g, const Th& t) {
    if (!t.periodic) return true;
    const double m = g.margin;
    return 4.0 * m < g.L && (double)x >= m && (double)x <= g.L - m && (double)y >= m && (double)y <= g.L - m &&
           (double)z >= m && (double)z <= g.L - m;
}

}  // namespace cc

// ---------------------------------------------------------------------------------------
// host-side helpers shared by the .cu files of libcc
cc_status cc_fail(cc_ctx* c, cc_status st, const std::string& msg);
cc_status cc_cuda_check(cc_ctx* c, cudaError_t e, const char* what);
#define CC_CUDA(ctx, expr)                                                   \
    do {                                                                     \
        cudaError_t e_ = (expr);                                             \
        if (e_ != cudaSuccess) return cc_cuda_check((ctx), e_, #expr);       \
    } while (0)
// every kernel launch goes through CCL so the context can report how many it issued
#define CCL(c, ...)             \
    do {                        \
        __VA_ARGS__;            \
        (c)->launches++;        \
    } while (0)
#define CC_TRY(expr)                                                       \
    do {                                                                     \
        cc_status s_ = (expr);                                               \
        if (s_ != CC_OK) return s_;                                          \
    } while (0)

template <typename T>
cc_status cc_ensure(cc_ctx* c, cc::DBuf<T>& b, size_t n, const char* name);
template <typename T>
void cc_release(cc_ctx* c, cc::DBuf<T>& b);

// profiling: bracket a launch; cls = kernel class name
int cc_prof_begin(cc_ctx* c, const char* cls);
void cc_prof_end(cc_ctx* c, int token);

// launch wrappers (each .cu file)
namespace cc {
cc_status scan_u32_to_u32(cc_ctx* c, const uint32_t* in, uint32_t* out, int64_t n, uint64_t* total_dev);
cc_status editable_list(cc_ctx* c, int64_t* e_all);
cc_status scan_editables(cc_ctx* c, int64_t e_all, unsigned long long* totals_dev);
cc_status rows_resolve(cc_ctx* c, const unsigned long long* totals_h);
cc_status bin_particles(cc_ctx* c, const float* x, const float* y, const float* z, const float* xh,
                        const float* yh, const float* zh, const uint32_t* gid, int64_t n_own, const uint32_t* g7,
                        int64_t gm, int64_t n);
cc_status pairs_count(cc_ctx* c);
cc_status fof_base_build(cc_ctx* c);
cc_status read_near_count(cc_ctx* c);
cc_status ensure_slot_of(cc_ctx* c);
cc_status pairs_fill(cc_ctx* c);
cc_status rows_finish(cc_ctx* c);
cc_status pgd_run(cc_ctx* c, cc_corr_info* info);
cc_status write_output(cc_ctx* c, const float4* pos_res, float* xo, float* yo, float* zo);
cc_status ensure_cor4(cc_ctx* c);
cc_status fof_run(cc_ctx* c, int which, uint32_t* labels, int64_t* n_groups);
cc_status mcc_run(cc_ctx* c, int which, unsigned long long* counts_dev);
cc_status get_pairs_run(cc_ctx* c, uint32_t* gi, uint32_t* gj, uint8_t* flags, int64_t cap,
                        unsigned long long* n_dev);
cc_status halo_sizes_run(cc_ctx* c, int64_t min_size, int64_t* sizes_h, int64_t cap, int64_t* n_h);
const float4* pgd_result(cc_ctx* c);
cc_status fof_base_begin(cc_ctx* c);
cc_status fof_base_end(cc_ctx* c);
cc_status union_near(cc_ctx* c, const float4* P, uint32_t* par);
unsigned long long* work_counters(cc_ctx* c);  // k3work, allocated and zeroed on first use
// comm.cu: the exchange layer (NCCL or in-process virtual ranks)
enum { CT_U8, CT_I32, CT_U32, CT_I64, CT_U64, CT_F32, CT_F64 };
enum { CO_SUM, CO_MIN };
cc_status comm_init(cc_ctx* c, const cc_dist* d);
void comm_destroy(cc_ctx* c);
cc_status comm_group_start(cc_ctx* c);
cc_status comm_group_end(cc_ctx* c);
cc_status comm_send(cc_ctx* c, const void* buf, size_t count, int type, int peer);
cc_status comm_recv(cc_ctx* c, void* buf, size_t count, int type, int peer);
cc_status comm_allreduce(cc_ctx* c, void* buf, size_t count, int type, int op);
cc_status comm_allgather(cc_ctx* c, const void* send, void* recv, size_t count, int type);
// dist.cu
cc_status dist_init(cc_ctx* c, const cc_dist* d);
void dist_destroy(cc_ctx* c);
cc_status dist_unique_id(void* out);
cc_status dist_allreduce_u64(cc_ctx* c, unsigned long long* dev, size_t count);
cc_status dist_allreduce_f64(cc_ctx* c, double* dev, size_t count);
cc_status dist_exchange_ghosts(cc_ctx* c, int64_t n, const float* x, const float* y, const float* z, const float* xh,
                               const float* yh, const float* zh, const uint32_t* gid);
cc_status dist_setup_refresh(cc_ctx* c);
cc_status dist_iter_tail(cc_ctx* c, const float4* p0, const float4* p1);
cc_status dist_fof_merge(cc_ctx* c, int64_t* n_groups);
cc_status dist_halo_sizes(cc_ctx* c, int64_t min_size, std::vector<uint32_t>& out);
}  // namespace cc
