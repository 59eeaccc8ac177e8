// cc_internal.cuh -- shared internals of libcc (the CUDA path).  Independent of oracle/.
//
// Data layout in HBM:
//   per local particle, cell-sorted "slot" order s:
//     orig4[s] = (x, y, z, gid bits)          float4, original P           (S1)
//     dec4[s]  = (xh, yh, zh, input index i)  float4, decompressed P_hat^(0)
//     cell_start[c]  u32 (n_cell + 1), slot_of[i] u32 (input index -> slot)
//     deg[s] u32, rowoff[s] u64 (exclusive scan of deg), eidx[s] u32 (editable rank)
//   per editable particle e (compacted in slot order, S3):
//     posA/posB[e] float4 (x, y, z, gid bits) ping-pong, origE[e] float4, slotE[e] u32,
//     rowptr[e] u64, Adam moments m,v as 6 float SoA arrays
//   rows[k] u32 (2|V| directed entries, sorted by partner gid within a row):
//     bits 0..29 partner editable index, bit 30 partner gid > own gid, bit 31 original link
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

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
};

// uniform grid on ORIGINAL positions, x fastest; ncell = nx*ny*nz.  Cell coordinate computed
// in fp64 as floor((x - x0) * inv_w) clamped to [0, n-1] (x0 = 0 for one GPU; the slab's
// lower ghost edge for multi-GPU, where x is first shifted by -L if it lies above the slab).
struct Grid {
    int nx, ny, nz;
    double inv_w;      // cells per unit length (same on all axes)
    double x0;         // lower x edge of the local grid
    double L;          // box
    int xwrap;         // 1: x axis periodic inside this grid (single GPU)
    double slab_hi;    // multi-GPU: x above slab_hi + ghost width belongs to the image -L
};

// per-iteration control block of the PGD loop (device resident)
struct Ctl {
    int done;          // 1 once the loop has ended (later launches return immediately)
    int t;             // iterations whose stop check has run
    int t_res;         // updates contained in the result buffer
    int converged;
    unsigned int ticket;
    int pad;
    unsigned long long active;   // active count of the last check
    double loss;
};

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

    // sizes
    int64_t n_in = 0;      // particles given by the caller (owned)
    int64_t n = 0;         // local particles (owned + ghost)
    int64_t E = 0;         // editable (owned rows)
    int64_t E_all = 0;     // editable incl. ghost partners (multi-GPU)
    int64_t nent = 0;      // directed row entries

    // device buffers
    cc::DBuf<float4> orig4, dec4, cor4, posA, posB, origE;
    cc::DBuf<uint32_t> key, rnk, cell_count, cell_start, slot_of, deg, eidx, rows, slotE, parent, mingid,
        gsize, scratch_u32;
    cc::DBuf<uint64_t> rowoff, rowptr, scratch_u64;
    cc::DBuf<float> mom;         // 6 * E floats: mx, my, mz, vx, vy, vz
    cc::DBuf<float2> bc;         // Adam bias corrections per iteration
    cc::DBuf<double> partial_d;  // block partials
    cc::DBuf<unsigned long long> partial_u, counters;
    cc::DBuf<cc::Ctl> ctl;
    cc::DBuf<long long> trace_a;
    cc::DBuf<double> trace_l;
    cc::DBuf<unsigned char> tmp_bytes;  // scan scratch
    cc::DBuf<float> in_f;        // cc_run host staging: 6 n floats
    cc::DBuf<uint32_t> in_gid;

    // pinned host mirrors
    cc::Ctl* h_ctl = nullptr;
    unsigned long long* h_counters = nullptr;

    // PGD graph cache
    cudaGraphExec_t pgd_exec = nullptr;
    const void* pgd_key[4] = {nullptr, nullptr, nullptr, nullptr};
    int pgd_batch = 0;
    int64_t pgd_E = -1;
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

// the cell of an ORIGINAL position (used identically by binning and by the searches)
__device__ __forceinline__ void cell_of(float x, float y, float z, const Grid& g, int& cx, int& cy, int& cz) {
    cx = cell_coord(local_u((double)x, g), 0.0, g.inv_w, g.nx);
    cy = cell_coord((double)y, 0.0, g.inv_w, g.ny);
    cz = cell_coord((double)z, 0.0, g.inv_w, g.nz);
}

__device__ __forceinline__ int wrapi(int a, int n) { return a < 0 ? a + n : (a >= n ? a - n : a); }

// Visit the candidate slot ranges of the 27-cell neighbourhood of cell (cx,cy,cz): the three
// x-adjacent cells of a (y,z) row are one contiguous slot range when they do not wrap.
// Offsets are de-duplicated when an axis has fewer than 3 cells (R1).  f(a, b) gets [a,b).
template <class F>
__device__ __forceinline__ void for_each_neighbour_range(const Grid& g, const uint32_t* __restrict__ cs,
                                                         int cx, int cy, int cz, bool periodic_yz, F&& f) {
    const int ny_off = g.ny >= 3 ? 3 : g.ny, nz_off = g.nz >= 3 ? 3 : g.nz, nx_off = g.nx >= 3 ? 3 : g.nx;
    const int offs[3] = {0, 1, -1};
    for (int kz = 0; kz < nz_off; kz++) {
        int zz = cz + offs[kz];
        if (periodic_yz) zz = wrapi(zz, g.nz);
        else if (zz < 0 || zz >= g.nz) continue;
        for (int ky = 0; ky < ny_off; ky++) {
            int yy = cy + offs[ky];
            if (periodic_yz) yy = wrapi(yy, g.ny);
            else if (yy < 0 || yy >= g.ny) continue;
            const int64_t base = ((int64_t)zz * g.ny + yy) * g.nx;
            if (cx >= 1 && cx <= g.nx - 2) {
                f(cs[base + cx - 1], cs[base + cx + 2]);
            } else {
                for (int kx = 0; kx < nx_off; kx++) {
                    int xx = cx + offs[kx];
                    if (g.xwrap) xx = wrapi(xx, g.nx);
                    else if (xx < 0 || xx >= g.nx) continue;
                    f(cs[base + xx], cs[base + xx + 1]);
                }
            }
        }
    }
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
cc_status scan_deg(cc_ctx* c, const uint32_t* deg, uint64_t* rowoff, uint32_t* eidx, int64_t n,
                   const float4* dec4, int64_t n_own, unsigned long long* totals_dev);
cc_status bin_particles(cc_ctx* c, const float* x, const float* y, const float* z, const float* xh,
                        const float* yh, const float* zh, const uint32_t* gid, int64_t n);
cc_status pairs_count(cc_ctx* c);
cc_status pairs_fill(cc_ctx* c);
cc_status rows_finish(cc_ctx* c);
cc_status pgd_run(cc_ctx* c, cc_corr_info* info);
cc_status write_output(cc_ctx* c, const float4* pos_res, float* xo, float* yo, float* zo);
cc_status fof_run(cc_ctx* c, int which, uint32_t* labels, int64_t* n_groups);
cc_status mcc_run(cc_ctx* c, int which, unsigned long long* counts_dev);
cc_status get_pairs_run(cc_ctx* c, uint32_t* gi, uint32_t* gj, uint8_t* flags, int64_t cap,
                        unsigned long long* n_dev);
cc_status halo_sizes_run(cc_ctx* c, int64_t min_size, int64_t* sizes_h, int64_t cap, int64_t* n_h);
const float4* pgd_result(cc_ctx* c);
}  // namespace cc
