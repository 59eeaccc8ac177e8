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
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>

#include "cc_internal.cuh"

namespace cg = cooperative_groups;

namespace cc {
namespace {

constexpr int PGD_THREADS = 256;
constexpr int PGD_MAX_BLOCKS = 148 * 8;
constexpr int NSTAT = LFX_STATS + 5;
constexpr int NB = 4;         // row entries per lane per chunk
constexpr int CH = 32 * NB;   // flattened row entries per warp chunk
constexpr uint32_t TAIL_ENTER = 32768;  // k_tail takes over when a selected list is this small
constexpr uint32_t TAIL_CAP = 131072;  // ... and hands back when a list would exceed this
constexpr int TAIL_BLOCKS = 148;       // k_tail's co-resident blocks

struct WarpSh {               // per-warp staging of K3's flattened row evaluation
    float4 t[CH];             // term (px, py, pz, kind bits) of each chunk entry
    float4 p[32];             // positions of the warp's 32 editables
    unsigned char inner[32];  // the editable is interior (its row never needs the minimum image)
    unsigned long long k0[32];
    uint32_t off[32];         // exclusive scan of the row lengths
    uint32_t ent[CH];         // partner editable of each chunk entry (the movers' touches)
    unsigned char seg[CH];    // owning lane of each chunk entry
};

struct PgdArgs {
    uint32_t E;  // editable particles with rows (owned)
    const unsigned long long* __restrict__ rowptr;
    const uint32_t* __restrict__ rows;
    const float4* __restrict__ origE;
    uint32_t e_short;  // editables are numbered class-major by row length (pairs.cu): [0, e_short)
                       // have <= 16 entries (k_pgd<0>), [e_short, E) more (k_pgd<1>)
    float4* pos0;
    float4* pos1;
    float* __restrict__ mom;  // 6 x E SoA
    const float2* __restrict__ bc;
    Th t;
    float imin, imax;  // a row whose owner lies in [imin, imax]^3 never wraps (min_image = identity)
    float alpha, b1, b2, omb1, omb2, eps, vstep;
    int optimizer;
    int t_max;
    int stop_mode;
    double eps_loss;
    Ctl* ctl;
    long long* trace_a;
    double* trace_l;
    long long* trace_v;
    long long* trace_s;  // schedule per iteration: items, awake, moved entries
    int count_only;
    unsigned long long* red;  // multi-GPU: local statistics (LFX_STATS words) for the allreduce, else nullptr
    // frontier (exact active-set skipping): frozen[e] = 0 awake, FZ_NEVER never frozen (has a
    // ghost partner), else the last iteration e was processed.  Iteration t (>= 3) processes
    // only its work list: the editables awake after t-1 and the partners of those that moved
    // at t-1 (built by t-1); errs counts unsafe freezes
    int frontier;
    uint32_t* frozen;
    uint32_t* abits;  // 2 bitmaps of nwords words: editables awake after an iteration
    uint32_t* ubits;  // 3 bitmaps: editables touched (a partner moved) in an iteration
    uint32_t nwords;
    uint32_t* slist;  // editables selected for the current iteration, k_select's output
    uint32_t* tlist;  // k_tail: 2 lists of TAIL_CAP editables (ping-pong)
    uint32_t* tbits;  // k_tail: 2 membership bitmaps of nwords words (kept all-zero outside k_tail)
    unsigned long long* errs;
    unsigned long long* work;  // running totals: [0] editables updated, [1] row entries evaluated
};

constexpr uint32_t FZ_NEVER = 0xFFFFFFFFu;

// one pair term, pinned (R4, R13, R14, R15): r = minimg(p - q), d_hat = sqrt_rn(r.r);
// kind 0: inactive, 1: add (px,py,pz) to the gradient, 2: coincident -> add px to g.x only
struct Term {
    float px, py, pz;
    float ee;
    int kind;
    bool viol;
};

template <bool INNER = false>
__device__ __forceinline__ Term pair_term(const float4& p, const float4& q, uint32_t ent, const Th& th) {
    Term o;
    // INNER: the row's owner is far from the periodic faces (interior()), min_image is the identity
    const float rx = INNER ? __fsub_rn(p.x, q.x) : min_image(__fsub_rn(p.x, q.x), th);
    const float ry = INNER ? __fsub_rn(p.y, q.y) : min_image(__fsub_rn(p.y, q.y), th);
    const float rz = INNER ? __fsub_rn(p.z, q.z) : min_image(__fsub_rn(p.z, q.z), th);
    float s = __fmul_rn(rx, rx);
    s = __fadd_rn(s, __fmul_rn(ry, ry));
    s = __fadd_rn(s, __fmul_rn(rz, rz));
    const bool ol = (ent & ENT_OLINK) != 0;
    o.viol = (s <= th.b2) != ol;  // link status differs from the original (Eq. 1 support)
    // Eq. (3): broken side (orig linked) active iff d_hat > b - 2 sqrt3 eps_q;
    //          false side (orig unlinked) active iff d_hat <= b + 2 sqrt3 eps_q
    // decided on s = d_hat^2 against sb2 / sf2 (identical decisions, Th); d_hat only if active
    const bool act = ol ? (s > th.sb2) : (s <= th.sf2);
    o.kind = 0;
    o.ee = 0.0f;
    o.px = o.py = o.pz = 0.0f;
    if (act) {
        const float d = __fsqrt_rn(s);
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


__device__ __forceinline__ float project(float x, float o, float xip) {
    const float lo = __fsub_ru(o, xip);
    const float hi = __fadd_rd(o, xip);
    if (x < lo) x = lo;
    if (x > hi) x = hi;
    return x;
}

// IEEE a / b (round to nearest) with the zero-dividend case answered directly: the exact
// result is a signed zero, and __fdiv_rn would take its slow path for it (frequent here: the
// Adam moments of particles without active pairs are exactly 0).  b is finite and non-zero.
__device__ __forceinline__ float div_rn(float a, float b) {
    if (a == 0.0f) return __int_as_float((__float_as_int(a) ^ __float_as_int(b)) & 0x80000000);
    return __fdiv_rn(a, b);
}

__device__ __forceinline__ bool k3_inner(const float4& p, const PgdArgs& a) {
    return p.x >= a.imin && p.x <= a.imax && p.y >= a.imin && p.y <= a.imax && p.z >= a.imin && p.z <= a.imax;
}

// per-editable state loads: plain, or through L2 only (k_tail: blocks read what other blocks
// wrote an iteration earlier)
template <bool CG, typename T>
__device__ __forceinline__ T ldst(const T* p) {
    if (CG) return __ldcg(p);
    return *p;
}

// one coordinate's Adam step in registers (R9); returns the new coordinate, sets |step|
__device__ __forceinline__ float adam_reg(float x, float g, float& m, float& v, const PgdArgs& a, float bc1, float bc2,
                                          float& step_abs) {
    m = __fadd_rn(__fmul_rn(a.b1, m), __fmul_rn(a.omb1, g));
    v = __fadd_rn(__fmul_rn(a.b2, v), __fmul_rn(a.omb2, __fmul_rn(g, g)));
    const float mh = div_rn(m, bc1);
    const float vh = div_rn(v, bc2);
    const float den = __fadd_rn(vh == 0.0f ? vh : __fsqrt_rn(vh), a.eps);
    const float step = __fmul_rn(a.alpha, div_rn(mh, den));
    step_abs = fabsf(step);
    return __fsub_rn(x, step);
}

// |step| far below the coordinate's ulp: the particle cannot move while its gradient stays 0
// (the Adam step then shrinks by ~10% per iteration), the frontier's freeze condition
__device__ __forceinline__ bool negligible(float step_abs, float x) { return step_abs <= fabsf(x) * 1.4901161e-8f; }

// True if any number of zero-gradient Adam steps from state (m, v) provably leaves coordinate x
// unchanged.  With g = 0, step k has |m_k| <= |m| (b1 (1+d))^k, v_k >= v (b2 (1-d))^k,
// bc1_k >= bc1a and bc2_k <= bc2z (the last replayed step's), so |step_k| <= alpha |m| b1^k /
// (bc1a (sqrt(v b2^k / bc2z) + eps)) up to rounding factors; since b1 < sqrt(b2) the bound is
// largest at k = 1.  If that bound is below half an
// ulp of x, x - step rounds back to x at every step and the projection (x is already inside the
// box) is the identity.  Factors 0.999 / 1.001 and the 1e-44 terms dominate every fp32
// rounding (relative 2^-24, absolute 2^-149 for subnormals) and exp/sqrt error by far.
__device__ __forceinline__ bool replay_still(float x, float m, float v, float bc1a, float bc2z, const PgdArgs& a) {
    const float ax = fabsf(x);
    if (!(ax >= 1e-30f) || !(a.b1 < sqrtf(a.b2) * 0.999f)) return false;
    const float mh = fabsf(m) * a.b1 / bc1a * 1.001f + 1e-44f;
    const float den = (sqrtf(v * a.b2 / bc2z) * 0.999f + a.eps) * 0.999f;
    const float bound = a.alpha * mh / den * 1.001f + 1e-44f;
    return bound < ax * 2.98023224e-8f;  // 2^-25 |x| <= half an ulp of x
}

// True if coordinate x sits on the face of its box B(xi') (project's directed-rounding bounds)
// toward which every zero-gradient Adam step from moment m pushes: with g = 0 the moment keeps
// its sign (m_k = fl(b1 m_{k-1}), possibly +-0), the step alpha m_hat / (sqrt(v_hat) + eps) has
// that sign or is 0, so x - step_k never rounds to the inside of the face and the projection
// returns the face, i.e. x, at every step.  Particles pressed against their box by leftover
// momentum (no active pair) are the bulk of the awake set at small xi (C4 xi_rel = 1e-6: ~1.86M
// editables processed per iteration for 60 iterations) -- they can freeze.
__device__ __forceinline__ bool clamp_still(float x, float m, float o, float xip) {
    return (x == __fsub_ru(o, xip) && m >= 0.0f) || (x == __fadd_rd(o, xip) && m <= 0.0f);
}

// Adam (or vanilla) step + projection of editable e, written to dst.  `replay` zero-gradient
// iterations missed while e was frozen (frontier) are first re-run exactly, in order.
// Returns bit0 = moved, bit1 = freeze-eligible step (negligible on all coordinates).
template <bool CG>
__device__ __forceinline__ int update(const PgdArgs& a, uint32_t e, const float4& p, float gx, float gy, float gz,
                                      int t, int replay_from, float4* __restrict__ dst) {
    const float4 o = a.origE[e];
    float x = p.x, y = p.y, z = p.z;
    int flags = 0;
    if (a.optimizer == CC_OPT_ADAM) {
        float* M = a.mom;
        const size_t E = a.E;
        float mx = ldst<CG>(M + e), my = ldst<CG>(M + E + e), mz = ldst<CG>(M + 2 * E + e);
        float vx = ldst<CG>(M + 3 * E + e), vy = ldst<CG>(M + 4 * E + e), vz = ldst<CG>(M + 5 * E + e);
        float sx, sy, sz;
        // zero-gradient iterations missed while frozen, in order: steps that provably cannot
        // move the coordinates only advance the moments; the others are recomputed in full and
        // checked (a move would mean the freeze was unsafe).  The proof is retried every 8 full
        // steps (the bound shrinks as the moments decay), so a particle frozen for thousands of
        // iterations replays a few dozen steps in full, not all of them.
        if (replay_from < t) {
            const float bc2z = a.bc[t - 2].y;
            int tt = replay_from;
            for (;;) {
                const float bc1a = a.bc[tt - 1].x;
                if ((replay_still(x, mx, vx, bc1a, bc2z, a) || clamp_still(x, mx, o.x, a.t.xip_f)) &&
                    (replay_still(y, my, vy, bc1a, bc2z, a) || clamp_still(y, my, o.y, a.t.xip_f)) &&
                    (replay_still(z, mz, vz, bc1a, bc2z, a) || clamp_still(z, mz, o.z, a.t.xip_f))) {
                    for (; tt < t; tt++) {  // provably no move (same expressions as adam_reg, g = 0)
                        mx = __fadd_rn(__fmul_rn(a.b1, mx), __fmul_rn(a.omb1, 0.0f));
                        my = __fadd_rn(__fmul_rn(a.b1, my), __fmul_rn(a.omb1, 0.0f));
                        mz = __fadd_rn(__fmul_rn(a.b1, mz), __fmul_rn(a.omb1, 0.0f));
                        vx = __fadd_rn(__fmul_rn(a.b2, vx), __fmul_rn(a.omb2, __fmul_rn(0.0f, 0.0f)));
                        vy = __fadd_rn(__fmul_rn(a.b2, vy), __fmul_rn(a.omb2, __fmul_rn(0.0f, 0.0f)));
                        vz = __fadd_rn(__fmul_rn(a.b2, vz), __fmul_rn(a.omb2, __fmul_rn(0.0f, 0.0f)));
                    }
                    break;
                }
                flags |= 4;  // full replay steps (reported in the schedule trace)
                const int t8 = min(t, tt + 8);  // retry the proof every 8 full steps (the bound decays)
                for (; tt < t8; tt++) {
                    const float2 b = a.bc[tt - 1];
                    const float nx = project(adam_reg(x, 0.0f, mx, vx, a, b.x, b.y, sx), o.x, a.t.xip_f);
                    const float ny = project(adam_reg(y, 0.0f, my, vy, a, b.x, b.y, sy), o.y, a.t.xip_f);
                    const float nz = project(adam_reg(z, 0.0f, mz, vz, a, b.x, b.y, sz), o.z, a.t.xip_f);
                    if (nx != x || ny != y || nz != z) atomicAdd(a.errs, 1ull);  // freeze was unsafe
                    x = nx;
                    y = ny;
                    z = nz;
                }
                if (tt >= t) break;
            }
        }
        const float2 b = a.bc[t - 1];
        // freeze-eligible: every coordinate's step negligible, or the coordinate held on its box
        // face by the momentum's direction (checked on the new state)
        const float nx = project(adam_reg(x, gx, mx, vx, a, b.x, b.y, sx), o.x, a.t.xip_f);
        bool still = negligible(sx, x) || clamp_still(nx, mx, o.x, a.t.xip_f);
        M[e] = mx;
        M[3 * E + e] = vx;
        const float ny = project(adam_reg(y, gy, my, vy, a, b.x, b.y, sy), o.y, a.t.xip_f);
        still = still && (negligible(sy, y) || clamp_still(ny, my, o.y, a.t.xip_f));
        M[E + e] = my;
        M[4 * E + e] = vy;
        const float nz = project(adam_reg(z, gz, mz, vz, a, b.x, b.y, sz), o.z, a.t.xip_f);
        still = still && (negligible(sz, z) || clamp_still(nz, mz, o.z, a.t.xip_f));
        M[2 * E + e] = mz;
        M[5 * E + e] = vz;
        if (still) flags |= 2;
        x = nx;
        y = ny;
        z = nz;
    } else {
        const float sx = __fmul_rn(a.vstep, gx), sy = __fmul_rn(a.vstep, gy), sz = __fmul_rn(a.vstep, gz);
        if (sx == 0.0f && sy == 0.0f && sz == 0.0f) flags |= 2;
        x = project(__fsub_rn(x, sx), o.x, a.t.xip_f);
        y = project(__fsub_rn(y, sy), o.y, a.t.xip_f);
        z = project(__fsub_rn(z, sz), o.z, a.t.xip_f);
    }
    if (x != p.x || y != p.y || z != p.z) flags |= 1;
    dst[e] = make_float4(x, y, z, p.w);
    return flags;
}

// frontier bookkeeping after e was processed at iteration t; returns whether e stays awake.
// any_active: some pair of e's row was L_tight-active OR violated -- when the margin 2 sqrt3 eps_q
// is below fp32 resolution (tiny xi) a pair can be violated yet inactive; freezing e then would
// hide a violated pair from the stop statistics (found on C3 at xi_rel = 1e-6)
__device__ __forceinline__ bool frontier_after(const PgdArgs& a, uint32_t e, int t, int flags, bool any_active,
                                               uint32_t fz) {
    if (fz == FZ_NEVER) return true;
    const bool freeze = !(flags & 1) && (flags & 2) && !any_active;
    a.frozen[e] = freeze ? (uint32_t)t : 0u;
    return !freeze;
}


// per-block K3 working state, shared by k_pgd (one iteration over the grid) and k_tail (one
// block, many iterations)
struct K3Ctx {
    int t;
    const float4* src;        // positions read (state t-1)
    float4* dst;              // positions written (state t)
    bool front, build;
    uint32_t* unext;          // k_pgd build: touched bitmap for t+1
    uint32_t* tbn;            // k_tail: membership bitmap of the list for t+1
    uint32_t* tnext;          // k_tail: the list for t+1
    uint32_t* n_next;         // k_tail: its length (shared memory)
    uint32_t* cn;             // this thread's counters, stride PGD_THREADS
    unsigned long long* lim;  // this thread's loss limbs, stride PGD_THREADS
    WarpSh* ws;
    int lane;
    unsigned long long wk_e, wk_n;  // work done: editables updated, row entries evaluated
};

// positions: plain loads in k_pgd (measured faster than the non-coherent path for these
// gathers); k_tail reads what other blocks wrote an iteration earlier (through L2)
template <bool TAIL>
__device__ __forceinline__ float4 ldpos(const float4* p) {
    if (TAIL) return __ldcg(p);
    return *p;
}

// k_tail: put editable j on the list for t+1 (once: the membership bitmap dedups)
__device__ __forceinline__ void tail_push(K3Ctx& k, uint32_t j) {
    const uint32_t bit = 1u << (j & 31);
    if (atomicOr(&k.tbn[j >> 5], bit) & bit) return;
    const uint32_t i = atomicAdd(k.n_next, 1u);
    if (i < TAIL_CAP) k.tnext[i] = j;
}

// ---- one batch: up to 32 editables (one per lane, `valid`).
// Gradient summation order (R14): the row's terms in ascending partner gid (inactive = +0), in
// chunks of GC = 16 consecutive terms summed left to right; the chunk sums of each group of 32
// chunks (512 terms) combined by the adjacent-pairwise tree; the group results summed left to
// right.  A row of <= GC entries (classes 0-1, most rows) is one chunk: a plain left-to-right sum.
// Short rows: the concatenation of the batch's short rows is evaluated flattened across the
// lanes (CH entries per chunk, NB independent row/partner loads per lane in flight, terms parked
// in shared memory), then every lane sums its own row from shared memory.  Longer rows: every
// lane walks its own row (below).
// Returns whether the lane's editable stays awake.
constexpr int GC = 16;            // terms per chunk of the summation order (R14)
constexpr uint32_t SHORT = GC;    // rows of one chunk take the flattened path (classes 0-1)

template <bool TAIL>
__device__ __forceinline__ void add_term(const Term& tm, uint32_t ent, K3Ctx& k, float& cx, float& cy, float& cz,
                                         bool& act) {
    if (ent & ENT_UPPER) {  // each pair counted once, at its lower-gid endpoint
        if (tm.kind) {
            k.cn[0]++;
            lfx_add<PGD_THREADS>(k.lim, (double)tm.ee * (double)tm.ee);
        }
        if (tm.viol) k.cn[PGD_THREADS]++;
    }
    act |= tm.kind != 0 || tm.viol;  // keeps the editable awake (frontier): active OR violated
    cx = __fadd_rn(cx, tm.px);
    cy = __fadd_rn(cy, tm.py);
    cz = __fadd_rn(cz, tm.pz);
}

// KIND: 0 = every item has a short row (k_pgd<0>), 1 = every item a long row (k_pgd<1>), 2 = mixed
// (k_tail) -- the two grid kernels keep their own register budgets
template <bool TAIL, int KIND>
__device__ __forceinline__ bool process_batch(const PgdArgs& a, K3Ctx& k, const uint32_t e, const bool valid) {
    const Th& th = a.t;
    WarpSh& ws = *k.ws;
    const int lane = k.lane;
    unsigned long long k0 = 0ull;
    uint32_t len = 0u, fz = 0u;
    float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
    if (valid) {
        k0 = a.rowptr[e];
        len = (uint32_t)(a.rowptr[e + 1] - k0);
        p = ldpos<TAIL>(k.src + e);
        if (k.front) fz = ldst<TAIL>(a.frozen + e);
        k.wk_e++;
        k.wk_n += len;
        k.cn[4 * PGD_THREADS]++;
    }
    const bool lng = KIND == 1 ? true : (KIND == 0 ? false : len > SHORT);
    const unsigned lmask = __ballot_sync(0xffffffffu, lng);
    const uint32_t slen = lng ? 0u : len;
    uint32_t off = slen;  // exclusive scan of the short row lengths over the warp
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, off, o);
        if (lane >= o) off += v;
    }
    const uint32_t T = __shfl_sync(0xffffffffu, off, 31);
    off -= slen;
    ws.off[lane] = off;
    ws.k0[lane] = k0;
    ws.p[lane] = p;
    const bool inner = k3_inner(p, a);
    ws.inner[lane] = inner ? 1 : 0;
    __syncwarp();
    bool any_active = false;
    float gx = 0.0f, gy = 0.0f, gz = 0.0f;
    const uint32_t tflat = KIND == 1 ? 0u : T;  // KIND 1 walks every row per lane (below)
#pragma nv_diag_suppress 186  // c < 0u for KIND 1: the loop is meant to vanish there
    for (uint32_t c = 0; c < tflat; c += CH) {
#pragma nv_diag_default 186
        // which lane owns each position of this chunk
        const uint32_t f0 = max(off, c), f1 = min(off + slen, c + CH);
        for (uint32_t f = f0; f < f1; f++) ws.seg[f - c] = (unsigned char)lane;
        __syncwarp();
        uint32_t ent[NB];
        int sg[NB];
#pragma unroll
        for (int j = 0; j < NB; j++) {
            const uint32_t f = c + lane + 32u * j;
            sg[j] = -1;
            ent[j] = 0u;
            if (f < T) {
                const int o = ws.seg[f - c];
                sg[j] = o;
                ent[j] = a.rows[ws.k0[o] + (f - ws.off[o])];
            }
        }
        float4 q[NB];
#pragma unroll
        for (int j = 0; j < NB; j++)
            if (sg[j] >= 0) q[j] = ldpos<TAIL>(k.src + (ent[j] & ENT_IDX));
#pragma unroll
        for (int j = 0; j < NB; j++) {
            if (sg[j] >= 0) {
                ws.ent[lane + 32 * j] = ent[j] & ENT_IDX;
                const Term tm = ws.inner[sg[j]] ? pair_term<true>(ws.p[sg[j]], q[j], ent[j], th)
                                                : pair_term<false>(ws.p[sg[j]], q[j], ent[j], th);
                if (ent[j] & ENT_UPPER) {  // each pair counted once, at its lower-gid endpoint
                    if (tm.kind) {
                        k.cn[0]++;
                        lfx_add<PGD_THREADS>(k.lim, (double)tm.ee * (double)tm.ee);
                    }
                    if (tm.viol) k.cn[PGD_THREADS]++;
                }
                ws.t[lane + 32 * j] = make_float4(tm.px, tm.py, tm.pz, __int_as_float(tm.kind | (tm.viol ? 4 : 0)));
            }
        }
        __syncwarp();
        // own row, in row order (R14; a short row is one chunk).  Branch-free: an inactive term
        // is (+0, +0, +0) and a coincident one (+-2e, +0, +0); g + 0 == g exactly since g is
        // never -0.  Loads of 4 terms are issued ahead of the sums.
        uint32_t f = f0;
        for (; f + 4 <= f1; f += 4) {
            float4 u[4];
#pragma unroll
            for (int i = 0; i < 4; i++) u[i] = ws.t[f + i - c];
#pragma unroll
            for (int i = 0; i < 4; i++) {
                any_active |= __float_as_int(u[i].w) != 0;
                gx = __fadd_rn(gx, u[i].x);
                gy = __fadd_rn(gy, u[i].y);
                gz = __fadd_rn(gz, u[i].z);
            }
        }
        for (; f < f1; f++) {
            const float4 u = ws.t[f - c];
            any_active |= __float_as_int(u.w) != 0;
            gx = __fadd_rn(gx, u.x);
            gy = __fadd_rn(gy, u.y);
            gz = __fadd_rn(gz, u.z);
        }
        __syncwarp();
    }

    // long rows (> SHORT entries, halo cores): every lane walks its OWN row (a class-3 batch has
    // 32 rows of similar length), 4 row/partner loads in flight, terms accumulated in registers:
    // chunk sums of GC terms, the adjacent-pairwise tree over each group of 32 chunk sums kept
    // as a binary counter (pending left operands by level), group results summed in order.
    if (KIND != 0 && lng) {
        float Gx = 0.0f, Gy = 0.0f, Gz = 0.0f;
        float px[5], py[5], pz[5];  // pending left operands of the tree, by level
        bool act = false;
        for (uint32_t g0 = 0; g0 < len; g0 += 32u * GC) {
            const uint32_t g1 = min(len, g0 + 32u * GC);
            uint32_t m = 0;  // chunks of this group completed
            for (uint32_t c0 = g0; c0 < g1; c0 += GC, m++) {
                const uint32_t c1 = min(c0 + GC, g1);
                float cx = 0.0f, cy = 0.0f, cz = 0.0f;
                // row entries as aligned 16-byte vectors (the lanes walk different rows: one L1
                // wavefront per 4 entries instead of per entry); mis = misalignment of the chunk
                // start, entries assembled from the previous and the next vector (the row buffer
                // is padded so the last vector read stays inside it)
                const unsigned long long A = k0 + c0;
                const int mis = (int)(A & 3ull);
                const uint4* R4 = reinterpret_cast<const uint4*>(a.rows) + (A >> 2);
                uint4 bv = R4[0];
                for (uint32_t f = c0; f < c1; f += 4) {
                    const uint4 nv = R4[((f - c0) >> 2) + 1];
                    uint32_t en[4];
                    en[0] = mis == 0 ? bv.x : mis == 1 ? bv.y : mis == 2 ? bv.z : bv.w;
                    en[1] = mis == 0 ? bv.y : mis == 1 ? bv.z : mis == 2 ? bv.w : nv.x;
                    en[2] = mis == 0 ? bv.z : mis == 1 ? bv.w : mis == 2 ? nv.x : nv.y;
                    en[3] = mis == 0 ? bv.w : mis == 1 ? nv.x : mis == 2 ? nv.y : nv.z;
                    bv = nv;
                    const int nvalid = (int)min(4u, c1 - f);
                    float4 q[4];
#pragma unroll
                    for (int j = 0; j < 4; j++)
                        if (j < nvalid) q[j] = ldpos<TAIL>(k.src + (en[j] & ENT_IDX));
#pragma unroll
                    for (int j = 0; j < 4; j++)
                        if (j < nvalid)
                            add_term<TAIL>(inner ? pair_term<true>(p, q[j], en[j], th) : pair_term<false>(p, q[j], en[j], th),
                                           en[j], k, cx, cy, cz, act);
                }
                // chunk m completes: right child at each level whose bit of m is set
#pragma unroll
                for (int L = 0; L < 5; L++) {
                    if ((m >> L) & 1u) {
                        cx = __fadd_rn(px[L], cx);
                        cy = __fadd_rn(py[L], cy);
                        cz = __fadd_rn(pz[L], cz);
                    } else {
                        px[L] = cx;
                        py[L] = cy;
                        pz[L] = cz;
                        break;
                    }
                }
                if (m == 31u) {  // a full group: the tree's root is (cx, cy, cz)
                    Gx = __fadd_rn(Gx, cx);
                    Gy = __fadd_rn(Gy, cy);
                    Gz = __fadd_rn(Gz, cz);
                }
            }
            if (m < 32u) {  // partial group: pending left operands, lowest level first (zero padding)
                bool have = false;
                float ax = 0.0f, ay = 0.0f, az = 0.0f;
#pragma unroll
                for (int L = 0; L < 5; L++) {
                    if ((m >> L) & 1u) {
                        if (have) {
                            ax = __fadd_rn(px[L], ax);
                            ay = __fadd_rn(py[L], ay);
                            az = __fadd_rn(pz[L], az);
                        } else {
                            ax = px[L];
                            ay = py[L];
                            az = pz[L];
                            have = true;
                        }
                    }
                }
                Gx = __fadd_rn(Gx, ax);
                Gy = __fadd_rn(Gy, ay);
                Gz = __fadd_rn(Gz, az);
            }
        }
        gx = Gx;
        gy = Gy;
        gz = Gz;
        any_active = act;
    }
    int flags = 0;
    bool awake = false;
    if (valid && !a.count_only) {
        const int t = k.t;
        const int replay_from = (fz != 0u && fz != FZ_NEVER) ? (int)fz + 1 : t;  // zero-gradient
        flags = update<TAIL>(a, e, p, gx, gy, gz, t, replay_from, k.dst);             // steps missed while frozen
        if (replay_from < t) k.cn[((flags & 4) ? 5 : 6) * PGD_THREADS] += (unsigned)(t - replay_from);
        if (a.frontier) {
            awake = frontier_after(a, e, t, flags, any_active, fz);
            if (awake) k.cn[2 * PGD_THREADS]++;
            if (flags & 1) k.cn[3 * PGD_THREADS] += len;
        }
    }
    if (TAIL || k.build) {  // a mover touches its owned partners for t+1
        const unsigned mv_all = __ballot_sync(0xffffffffu, (flags & 1) != 0);
        // short rows whose entries are still staged (the batch fit one chunk): every lane
        // touches the staged entries at its positions
        const bool staged = KIND != 1 && T <= CH;
        if (staged && (mv_all & ~lmask)) {
            for (uint32_t f = lane; f < T; f += 32u) {
                const int o = ws.seg[f];
                const uint32_t jj = ws.ent[f];
                if (((mv_all >> o) & 1u) && jj < a.E) {
                    if (TAIL) tail_push(k, jj);
                    else atomicOr(&k.unext[jj >> 5], 1u << (jj & 31));  // fire-and-forget (RED)
                }
            }
        }
        // the other movers walk their own rows, all lanes in parallel (4 entries in flight)
        if ((flags & 1) && (lng || !staged)) {
            uint32_t i = 0;
            for (; i + 4 <= len; i += 4) {
                uint32_t jj[4];
#pragma unroll
                for (int q = 0; q < 4; q++) jj[q] = a.rows[k0 + i + q] & ENT_IDX;
#pragma unroll
                for (int q = 0; q < 4; q++)
                    if (jj[q] < a.E) {
                        if (TAIL) tail_push(k, jj[q]);
                        else atomicOr(&k.unext[jj[q] >> 5], 1u << (jj[q] & 31));
                    }
            }
            for (; i < len; i++) {
                const uint32_t j = a.rows[k0 + i] & ENT_IDX;
                if (j < a.E) {
                    if (TAIL) tail_push(k, j);
                    else atomicOr(&k.unext[j >> 5], 1u << (j & 31));
                }
            }
        }
    }
    return awake;
}

// statistic s of the block (warp-cooperative; all lanes get it).  LFX layout: 0, 1 counters;
// 2..7 loss limbs; 8.. schedule counters 2..
__device__ __forceinline__ unsigned long long block_stat(int s, int lane,
                                                         const unsigned long long (*lim_sh)[PGD_THREADS],
                                                         const uint32_t (*cn_sh)[PGD_THREADS]) {
    unsigned long long v = 0ull;
    if (s >= 2 && s < LFX_STATS)
        for (int i = lane; i < PGD_THREADS; i += 32) v += lim_sh[s - 2][i];
    else
        for (int i = lane; i < PGD_THREADS; i += 32) v += cn_sh[s < 2 ? s : s - 6][i];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// the end of iteration t (one thread): publish its statistics and apply the stop rule (R11) to
// the state the iteration READ; if it holds, that buffer is the result
__device__ void k3_finish(const PgdArgs& a, Ctl* ctl, int t, const unsigned long long* tot, bool build) {
    const unsigned long long tu = tot[0], tv = tot[1];
    const double td = lfx_value(tot + 2);
    ctl->active = tu;
    ctl->violated = tv;
    ctl->loss = td;
    ctl->loss_le = lfx_le(tot + 2, a.eps_loss) ? 1 : 0;
    ctl->ticket = 0;
    ctl->nsel = 0u;  // consumed (k_select of the next iteration refills it)
    ctl->nsel_l = 0u;
    if (!a.count_only && a.trace_s && t >= 1 && t <= a.t_max) {
        long long* ts = a.trace_s + 6 * (t - 1);
        ts[0] = (long long)tot[LFX_STATS + 2];
        ts[1] = (long long)tot[LFX_STATS];
        ts[2] = (long long)tot[LFX_STATS + 1];
        ts[3] = (long long)tot[LFX_STATS + 3];
        ts[4] = (long long)tot[LFX_STATS + 4];
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        ts[5] = (long long)gt;  // device time (ns) at the end of iteration t
    }
    if (a.frontier && !a.count_only) {
        ctl->sel = build ? 1 : 0;
        ctl->bld = (tot[LFX_STATS] + tot[LFX_STATS + 1] <= (unsigned long long)a.E * 4ull) ? 1 : 0;
    }
    if (a.red) {  // multi-GPU: the decision waits for the allreduce (dist.cu k_decide)
        for (int k = 0; k < LFX_STATS; k++) a.red[k] = tot[k];
    } else if (!a.count_only) {
        if (a.trace_a) {
            a.trace_a[t - 1] = (long long)tu;
            a.trace_l[t - 1] = td;
            a.trace_v[t - 1] = (long long)tv;
        }
        if (stop_rule(a.stop_mode, tu, ctl->loss_le != 0, tv)) {
            ctl->done = 1;
            ctl->t_res = t - 1;  // the state this launch read
            ctl->converged = 1;
        } else if (t >= a.t_max) {
            ctl->done = 1;
            ctl->t_res = t;      // the state this launch wrote
        }
        ctl->t = t;
    }
}

// One PGD iteration over the editables of one row class: MODE 0 the short rows (<= SHORT entries,
// editables [0, e_short)), MODE 1 the long rows ([e_short, E)); the two launches run back to back
// in each iteration and MODE 1's last block applies the stop rule to both launches' statistics.
template <int MODE>
__global__ void __launch_bounds__(PGD_THREADS, MODE == 0 ? 4 : 3) k_pgd(PgdArgs a) {
    Ctl* ctl = a.ctl;
    if (!a.count_only && *((volatile int*)&ctl->done)) return;
    const int t = a.count_only ? 0 : ctl->t + 1;
    // statistics: active pairs, violated pairs, loss limbs (exact sums, LFX layout), then the
    // schedule counts.  Per-thread counters live in shared memory (touched rarely; registers are
    // the occupancy limit of this latency-bound kernel): 0 active, 1 violated, 2 awake, 3 moved
    // entries, 4 processed, 5 full-replay steps, 6 proven-still replay steps
    __shared__ unsigned long long lim_sh[6][PGD_THREADS];
    __shared__ uint32_t cn_sh[NSTAT - 6][PGD_THREADS];
    __shared__ WarpSh wsh[PGD_THREADS / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    K3Ctx k;
    k.t = t;
    if (a.count_only) {
        k.src = (ctl->t_res & 1) ? a.pos1 : a.pos0;
        k.dst = nullptr;
    } else {
        k.src = ((t - 1) & 1) ? a.pos1 : a.pos0;
        k.dst = (t & 1) ? a.pos1 : a.pos0;
    }
    // frontier (exact active-set skipping): from iteration 2 on, only the editables awake after
    // t-1 or touched (a partner moved at t-1) are processed.  Bitmaps over the E editables:
    // awake A[t & 1] read / A[(t+1) & 1] written whole words; touched U[t % 3] read /
    // U[(t+1) % 3] set by atomics / U[(t+2) % 3] cleared for the next launch.
    // Building the bitmaps costs a random atomic per partner of every mover, so launch t builds
    // them only when the previous launch saw few awake editables and movers (ctl->bld); launch
    // t+1 selects iff launch t built (ctl->sel), else it processes every editable.
    k.front = a.frontier && !a.count_only;
    const bool select = k.front && ctl->sel;
    k.build = k.front && ctl->bld;
    const uint32_t nw32 = a.nwords;
    k.unext = a.ubits + (size_t)((t + 1) % 3) * nw32;
    k.tbn = k.tnext = k.n_next = nullptr;
    k.cn = &cn_sh[0][threadIdx.x];  // cn[s * PGD_THREADS] = counter s
    k.lim = &lim_sh[0][threadIdx.x];
    k.ws = &wsh[w];
    k.lane = lane;
    k.wk_e = k.wk_n = 0ull;
    // items: dense sweep = the class's editable range; selected = its segment of the list built
    // by k_select (short rows from slist[0], long rows from slist[e_short])
    const uint32_t base = MODE == 0 ? 0u : a.e_short;
    const uint32_t n_items = select ? (MODE == 0 ? ctl->nsel : ctl->nsel_l) : (MODE == 0 ? a.e_short : a.E - a.e_short);
    // a block without items (small frontier) only takes part in the final ticket
    const bool idle = blockIdx.x * (uint32_t)PGD_THREADS >= n_items;
    if (!idle) {
#pragma unroll
        for (int s = 0; s < 6; s++) lim_sh[s][threadIdx.x] = 0ull;
#pragma unroll
        for (int s = 0; s < NSTAT - 6; s++) cn_sh[s][threadIdx.x] = 0u;
    }
    uint32_t* __restrict__ anext = a.abits + (size_t)((t + 1) & 1) * nw32;

    // ---- work items: every editable (sweep) or the selected list built by k_select; a warp
    // takes 32 consecutive items per batch
    const uint32_t gw = blockIdx.x * (PGD_THREADS / 32) + w, nwarps = gridDim.x * (PGD_THREADS / 32);
    for (uint32_t b0 = gw * 32u; b0 < n_items; b0 += nwarps * 32u) {
        const uint32_t kk = b0 + lane;
        const bool valid = kk < n_items;
        const uint32_t e = valid ? (select ? a.slist[base + kk] : base + kk) : 0xFFFFFFFFu;
        const bool awake = process_batch<false, MODE>(a, k, valid ? e : 0u, valid);
        if (k.build) {  // awake bits for t+1, one atomic per distinct word of the batch
            const uint32_t word = e >> 5;
            const unsigned peers = __match_any_sync(0xffffffffu, word);
            const uint32_t bits = __reduce_or_sync(peers, awake ? (1u << (e & 31)) : 0u);
            if (valid && bits && lane == __ffs(peers) - 1) atomicOr(&anext[word], bits);
        }
    }

    // ---- work counters (integers: order-free), one atomic per warp
    if (!a.count_only) {
        for (int o = 16; o > 0; o >>= 1) {
            k.wk_e += __shfl_down_sync(0xffffffffu, k.wk_e, o);
            k.wk_n += __shfl_down_sync(0xffffffffu, k.wk_n, o);
        }
        if (lane == 0 && k.wk_e) {
            atomicAdd(&a.work[0], k.wk_e);
            atomicAdd(&a.work[1], k.wk_n);
        }
    }

    // ---- statistics: integer sums (LFX), so the order of warps, blocks and ranks is free
    __shared__ bool am_last;
    __syncthreads();
    for (int s = w; s < NSTAT && !idle; s += PGD_THREADS / 32) {  // warp w sums statistics w, w+8, ...
        const unsigned long long v = block_stat(s, lane, lim_sh, cn_sh);
        if (lane == 0 && v) atomicAdd(&ctl->acc[s], v);
    }
    if (MODE == 0) return;  // the long-row launch that follows finishes the iteration
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned int tk = atomicAdd(&ctl->ticket, 1u);
        am_last = (tk == gridDim.x - 1);
    }
    __syncthreads();
    if (!am_last || threadIdx.x != 0) return;
    // last block: every other block's sums are in ctl->acc
    __threadfence();
    unsigned long long tot[NSTAT];
    for (int s = 0; s < NSTAT; s++) {
        tot[s] = ((volatile unsigned long long*)ctl->acc)[s];
        ctl->acc[s] = 0ull;
    }
    k3_finish(a, ctl, t, tot, k.build);
    __threadfence();
}

// k_tail's grid barrier.  The TAIL_BLOCKS blocks are co-resident (one per SM at most, nothing
// else runs on the stream); acquire loads + fences make the other blocks' writes visible.
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void tail_grid_sync(Ctl* ctl) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = ld_acquire(&ctl->bar_gen);
        __threadfence();
        if (atomicAdd(&ctl->bar_count, 1u) == gridDim.x - 1) {
            ctl->bar_count = 0u;  // nobody arrives at the next barrier before the generation moves
            __threadfence();
            atomicAdd(&ctl->bar_gen, 1u);
        } else {
            while (ld_acquire(&ctl->bar_gen) == g) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

// K3 tail: once the frontier is small (the long convergence tail: a few hundred
// editables per iteration for ~1,200 iterations on C4), TAIL_BLOCKS co-resident blocks run the
// remaining iterations back to back in one launch, separated by grid barriers -- the same
// per-editable work as k_pgd, with lists instead of bitmaps, and the list spread over all warps
// (a short list gets one editable per warp, so rows are evaluated with all lanes).  It takes
// over after k_select of a selected iteration whose list has at most TAIL_ENTER editables, and
// runs until the stop rule or T_max ends the loop, or hands back to the grid kernels (the next
// iteration a full sweep, exact) when a list would exceed TAIL_CAP.  The list for t+1 holds the
// editables left awake at t and the partners of those that moved at t (deduplicated by a
// membership bitmap): k_select's set.  Per iteration: process, block statistics -> ctl->acc,
// barrier, block 0 applies the stop rule (k3_finish), barrier.
__global__ void __launch_bounds__(PGD_THREADS, 1) k_tail(PgdArgs a) {
    Ctl* ctl = a.ctl;
    // every block reads the same entry state: nothing changes it before the first barrier
    if (!a.frontier || a.red || a.count_only || !a.tlist) return;
    if (*((volatile int*)&ctl->done) || !ctl->sel || ctl->nsel + ctl->nsel_l > TAIL_ENTER) return;
    const uint32_t ns0 = ctl->nsel;  // k_select's list: short rows at slist[0], long at slist[e_short]
    __shared__ unsigned long long lim_sh[6][PGD_THREADS];
    __shared__ uint32_t cn_sh[NSTAT - 6][PGD_THREADS];
    __shared__ WarpSh wsh[PGD_THREADS / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    K3Ctx k;
    k.front = true;
    k.build = false;
    k.unext = nullptr;
    k.n_next = &ctl->tail_nn;
    k.cn = &cn_sh[0][threadIdx.x];
    k.lim = &lim_sh[0][threadIdx.x];
    k.ws = &wsh[w];
    k.lane = lane;
    k.wk_e = k.wk_n = 0ull;
    const uint32_t* cur = a.slist;
    uint32_t n_cur = ctl->nsel + ctl->nsel_l;
    int t = ctl->t + 1;
    const uint32_t nwarps = gridDim.x * (PGD_THREADS / 32), gw = blockIdx.x * (PGD_THREADS / 32) + w;
    const uint32_t gt = blockIdx.x * PGD_THREADS + threadIdx.x, gs = gridDim.x * PGD_THREADS;
    for (;;) {
        uint32_t* nxt = a.tlist + (size_t)(t & 1) * TAIL_CAP;
        k.t = t;
        k.src = ((t - 1) & 1) ? a.pos1 : a.pos0;
        k.dst = (t & 1) ? a.pos1 : a.pos0;
        k.tbn = a.tbits + (size_t)(t & 1) * a.nwords;
        k.tnext = nxt;
#pragma unroll
        for (int s = 0; s < 6; s++) lim_sh[s][threadIdx.x] = 0ull;
#pragma unroll
        for (int s = 0; s < NSTAT - 6; s++) cn_sh[s][threadIdx.x] = 0u;
        __syncthreads();
        // gi editables per warp batch, so that the list covers all warps once
        const uint32_t gi = min(32u, max(1u, (n_cur + nwarps - 1) / nwarps));
        const uint32_t nbatch = (n_cur + gi - 1) / gi;
        for (uint32_t bt = gw; bt < nbatch; bt += nwarps) {
            const uint32_t kk = bt * gi + lane;
            const bool valid = lane < (int)gi && kk < n_cur;
            const uint32_t e = !valid ? 0u
                               : (cur != a.slist ? __ldcg(cur + kk)
                                                 : (kk < ns0 ? __ldcg(cur + kk) : __ldcg(cur + a.e_short + (kk - ns0))));
            const bool awake = process_batch<true, 2>(a, k, e, valid);
            if (valid && awake) tail_push(k, e);
        }
        __syncthreads();
        for (int s = w; s < NSTAT; s += PGD_THREADS / 32) {
            const unsigned long long v = block_stat(s, lane, lim_sh, cn_sh);
            if (lane == 0 && v) atomicAdd(&ctl->acc[s], v);
        }
        // the current list's members leave its membership bitmap (clean for the list of t+2)
        if (cur != a.slist) {
            uint32_t* tbc = a.tbits + (size_t)((t - 1) & 1) * a.nwords;
            for (uint32_t i = gt; i < n_cur; i += gs) tbc[__ldcg(cur + i) >> 5] = 0u;
        }
        tail_grid_sync(ctl);
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            unsigned long long tot[NSTAT];
            for (int s = 0; s < NSTAT; s++) {
                tot[s] = ((volatile unsigned long long*)ctl->acc)[s];
                ctl->acc[s] = 0ull;
            }
            k3_finish(a, ctl, t, tot, false);
            const uint32_t nn = *((volatile unsigned*)&ctl->tail_nn);
            int go = !ctl->done;
            if (go && nn > TAIL_CAP) {  // hand back: the next iteration sweeps every editable
                ctl->sel = 0;
                ctl->bld = 0;
                go = 0;
            }
            ctl->tail_go = go;
            ctl->tail_ncur = nn;
            ctl->tail_nn = 0u;
            __threadfence();
        }
        tail_grid_sync(ctl);
        const int go = *((volatile int*)&ctl->tail_go);
        const uint32_t nn = *((volatile unsigned*)&ctl->tail_ncur);
        if (!go) {  // leave the membership bitmap of the list for t+1 clean
            uint32_t* tbn = k.tbn;
            if (nn > TAIL_CAP)
                for (uint32_t i = gt; i < a.nwords; i += gs) tbn[i] = 0u;
            else
                for (uint32_t i = gt; i < nn; i += gs) tbn[__ldcg(nxt + i) >> 5] = 0u;
            break;
        }
        cur = nxt;
        n_cur = nn;
        t++;
    }
    for (int o = 16; o > 0; o >>= 1) {
        k.wk_e += __shfl_down_sync(0xffffffffu, k.wk_e, o);
        k.wk_n += __shfl_down_sync(0xffffffffu, k.wk_n, o);
    }
    if (lane == 0 && k.wk_e) {
        atomicAdd(&a.work[0], k.wk_e);
        atomicAdd(&a.work[1], k.wk_n);
    }
}

// Frontier selection for iteration t (runs before k_pgd in every iteration): the editables
// awake after t-1 or touched at t-1 (A[t & 1] | U[t % 3]) as a list, sorted within each block's
// 8192-editable segment; segments are placed by one atomic per block-step.  Also clears the
// touched bitmap U[(t+2) % 3] (written next at t+1) and, when t builds, the awake bitmap
// A[(t+1) & 1] it will fill.
__global__ void __launch_bounds__(PGD_THREADS) k_select(PgdArgs a) {
    Ctl* ctl = a.ctl;
    if (!a.frontier || *((volatile int*)&ctl->done)) return;
    const int t = ctl->t + 1;
    const uint32_t nw32 = a.nwords;
    const uint32_t gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
    uint32_t* uclr = a.ubits + (size_t)((t + 2) % 3) * nw32;
    for (uint32_t i = gt; i < nw32; i += gs) uclr[i] = 0u;
    if (ctl->bld) {
        uint32_t* anext = a.abits + (size_t)((t + 1) & 1) * nw32;
        for (uint32_t i = gt; i < nw32; i += gs) anext[i] = 0u;
    }
    if (!ctl->sel) return;
    const uint32_t* __restrict__ acur = a.abits + (size_t)(t & 1) * nw32;
    const uint32_t* __restrict__ ucur = a.ubits + (size_t)(t % 3) * nw32;
    // short-row editables (index < e_short) go to slist[0 ..), long-row ones to slist[e_short ..):
    // the two k_pgd launches each read their own segment.  Per-thread counts are packed as
    // short | long << 16 (a block-step holds at most 8192 editables) and scanned together.
    __shared__ uint32_t wsum[PGD_THREADS / 32];
    __shared__ uint32_t bbase_s, bbase_l;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (uint32_t w0 = blockIdx.x * blockDim.x; w0 < nw32; w0 += gs) {  // block-uniform loop
        const uint32_t wi = w0 + threadIdx.x;
        const uint32_t mask = wi < nw32 ? (acur[wi] | ucur[wi]) : 0u;
        const uint32_t lo = wi * 32u;
        const uint32_t smask = lo + 32u <= a.e_short ? mask
                               : (lo >= a.e_short ? 0u : mask & ((1u << (a.e_short - lo)) - 1u));
        const uint32_t lmask = mask & ~smask;
        const uint32_t cnt = (uint32_t)__popc(smask) | ((uint32_t)__popc(lmask) << 16);
        uint32_t pre = cnt;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, pre, o);
            if (lane >= o) pre += v;
        }
        if (lane == 31) wsum[w] = pre;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t tot = 0;
            for (int k = 0; k < PGD_THREADS / 32; k++) {
                const uint32_t v = wsum[k];
                wsum[k] = tot;
                tot += v;
            }
            bbase_s = (tot & 0xFFFFu) ? atomicAdd(&ctl->nsel, tot & 0xFFFFu) : 0u;
            bbase_l = (tot >> 16) ? atomicAdd(&ctl->nsel_l, tot >> 16) : 0u;
        }
        __syncthreads();
        const uint32_t ex = wsum[w] + pre - cnt;
        uint32_t ps = bbase_s + (ex & 0xFFFFu), pl = a.e_short + bbase_l + (ex >> 16);
        for (uint32_t m = smask; m; m &= m - 1) a.slist[ps++] = lo + (uint32_t)(__ffs(m) - 1);
        for (uint32_t m = lmask; m; m &= m - 1) a.slist[pl++] = lo + (uint32_t)(__ffs(m) - 1);
        __syncthreads();
    }
}

__global__ void k_ctl_reset(Ctl* ctl) {
    ctl->done = 0;
    ctl->t = 0;
    ctl->t_res = 0;
    ctl->converged = 0;
    ctl->ticket = 0;
    ctl->nsel = 0u;  // consumed (k_select of the next iteration refills it)
    ctl->active = 0;
    ctl->violated = 0;
    ctl->loss = 0.0;
    for (int k = 0; k < 14; k++) ctl->acc[k] = 0ull;
    ctl->sel = 0;
    ctl->bld = 1;  // iteration 1 (a full sweep) builds the bitmaps: iteration 2 already selects
    ctl->nsel = 0u;
    ctl->nsel_l = 0u;
    ctl->tail_nn = 0u;
    ctl->tail_ncur = 0u;
    ctl->tail_go = 0;
    ctl->bar_count = 0u;
    ctl->bar_gen = 0u;
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
    const uint32_t e = eidx[s];
    float4 d = dec4[s];
    if (e != 0xFFFFFFFFu) {
        const float4 r = res[e];
        d.x = r.x;
        d.y = r.y;
        d.z = r.z;
    }
    cor4[s] = d;
}

// the decompressed inputs streamed to the outputs: 16-byte vectors when every pointer allows
// (the copy engine's D2D memcpy reached ~2 TB/s on these 1.1 GB arrays; SM copies run near HBM)
// (no __restrict__: an output may alias its own input, cc.h)
__global__ void __launch_bounds__(256) k_copy3(int64_t n, const float* a0, const float* a1, const float* a2,
                                               float* b0, float* b1, float* b2, int vec) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    if (vec) {
        const int64_t n4 = n >> 2;
        for (int64_t i = tid; i < n4; i += nt) {
            const float4 u = reinterpret_cast<const float4*>(a0)[i];
            const float4 v = reinterpret_cast<const float4*>(a1)[i];
            const float4 w = reinterpret_cast<const float4*>(a2)[i];
            reinterpret_cast<float4*>(b0)[i] = u;
            reinterpret_cast<float4*>(b1)[i] = v;
            reinterpret_cast<float4*>(b2)[i] = w;
        }
        for (int64_t i = (n4 << 2) + tid; i < n; i += nt) {
            b0[i] = a0[i];
            b1[i] = a1[i];
            b2[i] = a2[i];
        }
    } else {
        for (int64_t i = tid; i < n; i += nt) {
            b0[i] = a0[i];
            b1[i] = a1[i];
            b2[i] = a2[i];
        }
    }
}

// outputs in input order (owned particles): the decompressed inputs were copied first; the owned
// editables overwrite their entries with the PGD result (x^(0) = P_hat, only editables move)
__global__ void k_output_edits(uint32_t e_own, const uint32_t* __restrict__ slotE, const float4* __restrict__ dec4,
                               const float4* __restrict__ res, float* __restrict__ xo, float* __restrict__ yo,
                               float* __restrict__ zo) {
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= e_own) return;
    const float4 d = dec4[slotE[e]];
    const uint32_t i = __float_as_uint(d.w);  // input index
    const float4 r = res[e];
    // only the coordinates PGD changed (bitwise): the copy already wrote the others, and most
    // editables never move at small xi (each skipped store is a DRAM read-modify-write saved)
    if (__float_as_uint(r.x) != __float_as_uint(d.x)) xo[i] = r.x;
    if (__float_as_uint(r.y) != __float_as_uint(d.y)) yo[i] = r.y;
    if (__float_as_uint(r.z) != __float_as_uint(d.z)) zo[i] = r.z;
}

PgdArgs make_args(cc_ctx* c, int count_only) {
    PgdArgs a;
    std::memset(&a, 0, sizeof(a));  // padding too: the bytes are the graph signature
    a.E = (uint32_t)c->E;
    a.rowptr = reinterpret_cast<const unsigned long long*>(c->rowptr.p);
    a.rows = c->rows.p;
    a.origE = c->origE.p;
    a.e_short = (uint32_t)(c->E_cls[0] + c->E_cls[1]);  // rows <= 16 entries (one chunk)
    a.pos0 = c->posA.p;
    a.pos1 = c->posB.p;
    a.mom = c->mom.p;
    a.bc = c->bc.p;
    a.t = c->th;
    // owners at least 2 search radii inside the periodic box: every partner difference of the
    // current positions (within xi_f of the originals, partners within r_pair) is far below L/2
    if (c->p.periodic && 8.0 * c->r_pair < c->p.box) {
        a.imin = (float)(2.0 * c->r_pair);
        a.imax = (float)(c->p.box - 2.0 * c->r_pair);
    } else if (!c->p.periodic) {
        a.imin = -INFINITY;
        a.imax = INFINITY;
    } else {
        a.imin = 1.0f;  // empty interval: every row takes the minimum image
        a.imax = 0.0f;
    }
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
    a.trace_a = c->trace_a.p;
    a.trace_l = c->trace_l.p;
    a.trace_v = c->trace_v.p;
    a.trace_s = c->trace_s.p;
    a.count_only = count_only;
    a.red = c->nranks > 1 ? c->red.p : nullptr;
    a.frontier = c->p.frontier ? 1 : 0;
    a.frozen = c->frozen.p;
    a.errs = c->counters.p + 15;
    a.work = c->k3work.p;
    a.nwords = (uint32_t)((std::max<int64_t>(c->E, 1) + 31) / 32);
    a.abits = c->fbits.p;
    a.slist = c->slist.p;
    a.ubits = c->fbits.p + 2 * (size_t)a.nwords;
    a.tbits = c->fbits.p + 5 * (size_t)a.nwords;
    a.tlist = c->tlist.p;
    return a;
}

// frontier state at the start of cc_correct: everyone awake; rows with a ghost partner
// (multi-GPU) are never frozen, so moves of ghosts (refreshed each iteration) are always seen
__global__ void k_frontier_init(uint32_t E, const unsigned long long* __restrict__ rowptr,
                                const uint32_t* __restrict__ rows, uint32_t* __restrict__ frozen) {
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    bool ghost = false;
    for (unsigned long long k = rowptr[e]; k < rowptr[e + 1]; k++) ghost |= (rows[k] & ENT_IDX) >= E;
    frozen[e] = ghost ? FZ_NEVER : 0u;
}

int pgd_blocks(int64_t E) {
    int64_t b = (E + PGD_THREADS - 1) / PGD_THREADS;
    if (b > PGD_MAX_BLOCKS) b = PGD_MAX_BLOCKS;
    if (b < 1) b = 1;
    return (int)b;
}

}  // namespace

const float4* pgd_result(cc_ctx* c) { return (c->last_iters & 1) ? c->posB.p : c->posA.p; }

// (active, loss, violated) of the count-only pass just enqueued, summed over ranks
// (synchronising); *loss_le = L_tight <= eps_L decided exactly on the integer limbs
static cc_status global_check(cc_ctx* c, double* al, bool* loss_le = nullptr) {
    if (c->nranks > 1) {
        CC_TRY(dist_allreduce_u64(c, c->red.p, LFX_STATS));
        CC_CUDA(c, cudaMemcpyAsync(c->h_red, c->red.p, LFX_STATS * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                   c->stream));
        CC_CUDA(c, cudaStreamSynchronize(c->stream));
        al[0] = (double)c->h_red[0];
        al[1] = lfx_value(c->h_red + 2);
        al[2] = (double)c->h_red[1];
        if (loss_le) *loss_le = lfx_le(c->h_red + 2, c->p.eps_loss);
    } else {
        CC_CUDA(c, cudaMemcpyAsync(c->h_ctl, c->ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, c->stream));
        CC_CUDA(c, cudaStreamSynchronize(c->stream));
        al[0] = (double)c->h_ctl->active;
        al[1] = c->h_ctl->loss;
        al[2] = (double)c->h_ctl->violated;
        if (loss_le) *loss_le = c->h_ctl->loss_le != 0;
    }
    return CC_OK;
}

cc_status pgd_run(cc_ctx* c, cc_corr_info* info) {
    const int64_t E = c->E, Ea = c->E_all;
    const int tmax = c->p.t_max;
    CC_TRY(cc_ensure(c, c->mom, (size_t)std::max<int64_t>(6 * E, 1), "adam moments"));
    CC_TRY(cc_ensure(c, c->bc, (size_t)std::max(tmax, 1), "bias corrections"));
    CC_TRY(cc_ensure(c, c->ctl, 1, "ctl"));
    CC_TRY(cc_ensure(c, c->trace_a, (size_t)tmax + 1, "trace"));
    CC_TRY(cc_ensure(c, c->trace_l, (size_t)tmax + 1, "trace"));
    CC_TRY(cc_ensure(c, c->trace_v, (size_t)tmax + 1, "trace"));
    CC_TRY(cc_ensure(c, c->trace_s, 6 * ((size_t)tmax + 1), "trace"));
    if (c->nranks > 1) CC_TRY(cc_ensure(c, c->red, LFX_STATS, "allreduce buffer"));
    if (!work_counters(c)) return cc_fail(c, CC_E_OOM, "work counters");
    CC_TRY(cc_ensure(c, c->frozen, (size_t)std::max<int64_t>(E, 1), "frontier state"));
    const size_t nwords = (size_t)((std::max<int64_t>(E, 1) + 31) / 32);
    CC_TRY(cc_ensure(c, c->fbits, 7 * nwords, "frontier bitmaps"));
    CC_TRY(cc_ensure(c, c->slist, (size_t)std::max<int64_t>(E, 1), "frontier selection"));
    CC_TRY(cc_ensure(c, c->tlist, 2 * (size_t)TAIL_CAP, "frontier tail lists"));
    CC_CUDA(c, cudaMemsetAsync(c->fbits.p, 0, 7 * nwords * sizeof(uint32_t), c->stream));
    CC_TRY(cc_ensure(c, c->counters, 16, "counters"));
    CC_CUDA(c, cudaMemsetAsync(c->counters.p + 15, 0, sizeof(unsigned long long), c->stream));
    if (E > 0)
        CCL(c, k_frontier_init<<<(unsigned)((E + 255) / 256), 256, 0, c->stream>>>(
                   (uint32_t)E, reinterpret_cast<const unsigned long long*>(c->rowptr.p), c->rows.p, c->frozen.p));
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
    const int nb = pgd_blocks(E);
    const int64_t e_short = c->E_cls[0] + c->E_cls[1];
    const int nb0 = pgd_blocks(e_short), nb1 = pgd_blocks(E - e_short);  // short / long-row launches
    const int batch = c->p.graph_batch > 0 ? c->p.graph_batch : 16;
    // k_tail (single GPU; CC_NO_TAIL=1 disables it, a diagnostic)
    const bool use_tail = c->nranks == 1 && !(std::getenv("CC_NO_TAIL") && std::getenv("CC_NO_TAIL")[0] == '1');
    
    // k_tail's blocks wait on each other (grid barrier): it is a COOPERATIVE launch, so the
    // driver guarantees co-residency or rejects it; the count is clamped to what the occupancy
    // calculator says fits
    int tail_blocks = TAIL_BLOCKS;
    {
        int sms = 0, per_sm = 0;
        CC_CUDA(c, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
        CC_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tail, PGD_THREADS, 0));
        tail_blocks = std::min<int>(tail_blocks, std::max(sms, 1) * std::max(per_sm, 0));
    }
    const bool tail_on = use_tail && tail_blocks > 0;
    const int k3_per_iter = tail_on ? 4 : 3;  // k_select (+ k_tail) + k_pgd<0> + k_pgd<1>
    PgdArgs a = make_args(c, 0);
    // initial statistics of P_hat^(0) for the report: iteration 1 evaluates exactly that state
    // (a full sweep) and records them in the trace (entry 0); a separate counting pass only
    // when no iteration runs
    if (tmax <= 0) {
        PgdArgs a0 = make_args(c, 1);
        CCL(c, k_pgd<0><<<nb0, PGD_THREADS, 0, c->stream>>>(a0));
        CCL(c, k_pgd<1><<<nb1, PGD_THREADS, 0, c->stream>>>(a0));
        CC_CUDA(c, cudaGetLastError());
        double al[3];
        CC_TRY(global_check(c, al));
        info->active0 = (int64_t)al[0];
        info->loss0 = al[1];
        info->violated0 = (int64_t)al[2];
    }
    CCL(c, k_ctl_reset<<<1, 1, 0, c->stream>>>(c->ctl.p));
    // multi-GPU peer exchange: a fresh epoch range per run (identical on every rank)
    c->epoch_base += (unsigned)tmax + 2u;
    CC_CUDA(c, cudaMemcpyAsync(&c->ctl.p->ep_base, &c->epoch_base, sizeof(unsigned), cudaMemcpyHostToDevice,
                               c->stream));
    CC_CUDA(c, cudaStreamSynchronize(c->stream));  // the source is a host field

    int iters = 0;
    if (tmax > 0 && c->vgroup) {
        // virtual ranks (comm.cu): the exchange is host-matched across the group's threads, so
        // no graph -- every iteration is launched directly and the global stop is read back
        for (;;) {
            CCL(c, k_select<<<nb, PGD_THREADS, 0, c->stream>>>(a));
            CCL(c, k_pgd<0><<<nb0, PGD_THREADS, 0, c->stream>>>(a));
            CCL(c, k_pgd<1><<<nb1, PGD_THREADS, 0, c->stream>>>(a));
            CC_TRY(dist_iter_tail(c, c->posA.p, c->posB.p));
            CC_CUDA(c, cudaGetLastError());
            CC_CUDA(c, cudaMemcpyAsync(c->h_ctl, c->ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, c->stream));
            CC_CUDA(c, cudaStreamSynchronize(c->stream));
            if (c->h_ctl->done) {
                iters = c->h_ctl->t_res;
                break;
            }
        }
    } else if (tmax > 0) {
        // (re)capture a graph of `batch` iterations, each bracketed by event records
        // the graph bakes in every argument of k_pgd: re-capture when any of them changed
        // signature: every byte k_pgd and the multi-GPU tail bake in
        std::vector<unsigned char> sig;
        auto put = [&sig](const void* v, size_t sz) {
            const unsigned char* b = static_cast<const unsigned char*>(v);
            sig.insert(sig.end(), b, b + sz);
        };
        put(&a, sizeof(a));
        put(&nb, sizeof(nb));
        put(&nb0, sizeof(nb0));
        put(&nb1, sizeof(nb1));
        put(&batch, sizeof(batch));
        put(&tail_on, sizeof(tail_on));
        if (c->nranks > 1) {
            for (int d = 0; d < 2; d++) {
                const void* ptrs[4] = {c->send_e[d].p, c->recv_e[d].p, c->rsb[d].p, c->rrb[d].p};
                put(ptrs, sizeof(ptrs));
                put(&c->n_ref_send[d], sizeof(int64_t));
                put(&c->n_ref_recv[d], sizeof(int64_t));
            }
            const void* r = c->red.p;
            put(&r, sizeof(r));
            put(&c->pm_ok, sizeof(c->pm_ok));
            put(c->pm_peer, sizeof(c->pm_peer));
            put(c->pm_peer_cap, sizeof(c->pm_peer_cap));
            put(c->pm_cap, sizeof(c->pm_cap));
            const void* rs = c->red_sum.p;
            put(&rs, sizeof(rs));
        }
        const bool same = c->pgd_exec && sig == c->pgd_sig;
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
                CCL(c, k_select<<<nb, PGD_THREADS, 0, c->stream>>>(a));
                if (tail_on) {
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = dim3((unsigned)tail_blocks);
                    cfg.blockDim = dim3(PGD_THREADS);
                    cfg.stream = c->stream;
                    cudaLaunchAttribute attr[1];
                    attr[0].id = cudaLaunchAttributeCooperative;
                    attr[0].val.cooperative = 1;
                    cfg.attrs = attr;
                    cfg.numAttrs = 1;
                    const cudaError_t le = cudaLaunchKernelEx(&cfg, k_tail, a);
                    if (le != cudaSuccess) {
                        cudaGraph_t g2 = nullptr;
                        cudaStreamEndCapture(c->stream, &g2);
                        if (g2) cudaGraphDestroy(g2);
                        return cc_cuda_check(c, le, "cooperative k_tail launch");
                    }
                    c->launches++;
                }
                CCL(c, k_pgd<0><<<nb0, PGD_THREADS, 0, c->stream>>>(a));
                CCL(c, k_pgd<1><<<nb1, PGD_THREADS, 0, c->stream>>>(a));
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
            c->launches -= k3_per_iter * batch;  // captured, not launched
            cudaError_t ce = cudaStreamEndCapture(c->stream, &graph);
            CC_CUDA(c, ce);
            CC_CUDA(c, cudaGraphInstantiate(&c->pgd_exec, graph, 0));
            cudaGraphDestroy(graph);
            c->pgd_sig = sig;
        }
        int t_before = 0;
        for (;;) {
            CC_CUDA(c, cudaGraphLaunch(c->pgd_exec, c->stream));
            c->launches += batch * (k3_per_iter + c->launches_per_iter_tail);
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
    const bool stopped = tmax > 0 && c->h_ctl->converged != 0;  // the stop rule held at state iters
    c->h_ctl->t_res = iters;
    CC_CUDA(c, cudaMemcpyAsync(&c->ctl.p->t_res, &c->h_ctl->t_res, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    double al[3];
    bool le = false;
    if (tmax > 0) {  // trace entry s = the statistics of state s (read by iteration s + 1)
        long long ta[2];
        double tl[2];
        long long tv[2];
        const int last = stopped ? iters : 0;
        CC_CUDA(c, cudaMemcpyAsync(&ta[0], c->trace_a.p, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
        CC_CUDA(c, cudaMemcpyAsync(&tl[0], c->trace_l.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CC_CUDA(c, cudaMemcpyAsync(&tv[0], c->trace_v.p, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
        CC_CUDA(c, cudaMemcpyAsync(&ta[1], c->trace_a.p + last, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
        CC_CUDA(c, cudaMemcpyAsync(&tl[1], c->trace_l.p + last, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CC_CUDA(c, cudaMemcpyAsync(&tv[1], c->trace_v.p + last, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
        CC_CUDA(c, cudaStreamSynchronize(c->stream));
        info->active0 = ta[0];
        info->loss0 = tl[0];
        info->violated0 = tv[0];
        al[0] = (double)ta[1];
        al[1] = tl[1];
        al[2] = (double)tv[1];
    }
    if (!stopped) {  // T_max (or no iteration): evaluate the returned state
        PgdArgs af = make_args(c, 1);
        int tok = cc_prof_begin(c, "K3_final_check");
        CCL(c, k_pgd<0><<<nb0, PGD_THREADS, 0, c->stream>>>(af));
        CCL(c, k_pgd<1><<<nb1, PGD_THREADS, 0, c->stream>>>(af));
        cc_prof_end(c, tok);
        CC_CUDA(c, cudaGetLastError());
        CC_TRY(global_check(c, al, &le));
    }
    info->iterations = iters;
    info->active_final = (int64_t)al[0];
    info->loss_final = al[1];
    info->violated_final = (int64_t)al[2];
    info->converged = stopped ||
                      stop_rule(c->p.stop_mode, (unsigned long long)al[0], le, (unsigned long long)al[2]) ||
                      (c->p.stop_mode == CC_STOP_NONE && al[0] == 0.0);
    c->final_active = (unsigned long long)al[0];
    c->final_loss = al[1];
    c->final_violated = (unsigned long long)al[2];
    if (c->p.frontier) {
        CC_CUDA(c, cudaMemcpyAsync(c->h_counters + 15, c->counters.p + 15, sizeof(unsigned long long),
                                   cudaMemcpyDeviceToHost, c->stream));
        CC_CUDA(c, cudaStreamSynchronize(c->stream));
        if (c->h_counters[15] != 0)  // a frozen particle would have moved: the skip was not exact
            return cc_fail(c, CC_E_DATA, "frontier: " + std::to_string(c->h_counters[15]) +
                                             " unsafe freezes (rerun with params.frontier = 0)");
    }
    return CC_OK;
}

cc_status write_output(cc_ctx* c, const float4* res, float* xo, float* yo, float* zo) {
    // every owned particle's decompressed input streamed to the output (coalesced copies), then
    // one scattered write per owned editable: round 1 gathered all n outputs from a slot-order
    // buffer through slot_of (a random 32-byte sector per particle, 8.3 ms at C4)
    c->cor4_valid = false;
    int tok = cc_prof_begin(c, "K3_output");
    const int64_t n = c->n_in;
    if (n > 0 && xo) {
        if (xo != c->in_dec[0] || yo != c->in_dec[1] || zo != c->in_dec[2]) {
            auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0u; };
            const int vec = al(xo) && al(yo) && al(zo) && al(c->in_dec[0]) && al(c->in_dec[1]) && al(c->in_dec[2]);
            CCL(c, k_copy3<<<148 * 8, 256, 0, c->stream>>>(n, c->in_dec[0], c->in_dec[1], c->in_dec[2], xo, yo, zo,
                                                            vec));
        }
        if (c->E > 0)
            CCL(c, k_output_edits<<<(unsigned)((c->E + 255) / 256), 256, 0, c->stream>>>(
                       (uint32_t)c->E, c->slotE.p, c->dec4.p, res, xo, yo, zo));
    }
    cc_prof_end(c, tok);
    CC_CUDA(c, cudaGetLastError());
    return CC_OK;
}

// corrected positions in slot order (the FoF(CORR) near-shell test), from the result buffer
cc_status ensure_cor4(cc_ctx* c) {
    if (c->cor4_valid) return CC_OK;
    const int64_t n = c->n;
    CC_TRY(cc_ensure(c, c->cor4, (size_t)std::max<int64_t>(n, 1), "cor4"));
    if (n > 0)
        CCL(c, k_cor4<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(n, c->dec4.p, c->eidx.p, (uint32_t)c->E,
                                                                          pgd_result(c), c->cor4.p));
    CC_CUDA(c, cudaGetLastError());
    c->cor4_valid = true;
    return CC_OK;
}

}  // namespace cc
