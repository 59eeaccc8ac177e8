// bin.cu -- K1, cell binning (S1).  §III-C: "each thread maps one particle to its grid
// cell and atomically increments per-cell counts ...; a device-wide exclusive prefix sum then
// converts these counts into cell-start offsets, after which a scatter kernel places each
// particle into a cell-sorted array using atomic index reservations."
//
// B200 form (the x-sorted-row structure of cc_internal.cuh):
//  1. key + histogram: coalesced SoA reads, one u32 atomic per particle whose return value is
//     its provisional rank inside the cell; checks the input contract (finite, |x_hat-x|<=xi).
//  2. reduce-then-scan of the counts (scan.cu) -> cell_start.
//  3. scatter of one full 32-byte record (x,y,z,x_hat,y_hat,z_hat,gid,i) per particle: one
//     aligned full-sector write each, instead of re-gathering six arrays later.
//  4. per-cell finish: each cell (~1/K particles on average) sorts its records by x in
//     registers (crowded cells: a block bitonic) and writes the float4 records, xk and slot_of.
//     Consecutive threads own consecutive cells, so reads and writes stream.
// The slot order is fully determined by the data (x ties broken by input index).
#include <cmath>
#include <cstdlib>

#include "cc_internal.cuh"

namespace cc {
namespace {

constexpr int BIN_THREADS = 256;
constexpr int CELL_SHORT = 16;
constexpr int CELL_MID = 64;    // 17..64: one warp per cell (k_cell_finish_mid)
constexpr int CELL_LONG_MAX = 4096;
constexpr int ROW_WIDE = 512;  // 65..512: one warp per row, bitonic in the warp's shared memory

struct __align__(16) Rec {
    float x, y, z, xh;
    float yh, zh;
    uint32_t gid, i;
};

// the local particles: i < n_own from the caller's SoA arrays (input order), then the ghosts
// (multi-GPU) from a small 7-word SoA staging of stride gm (x, y, z, xh, yh, zh, gid) -- the
// owned arrays are read in place instead of being copied into a combined staging first
struct BinSrc {
    const float *x, *y, *z, *xh, *yh, *zh;
    const uint32_t* gid;  // NULL: gid = input index
    int64_t n_own;
    const uint32_t* g7;
    int64_t gm;
    __device__ __forceinline__ void load(int64_t i, float& a, float& b, float& c, float& ah, float& bh,
                                         float& ch) const {
        if (i < n_own) {
            a = x[i];
            b = y[i];
            c = z[i];
            ah = xh[i];
            bh = yh[i];
            ch = zh[i];
        } else {
            const int64_t k = i - n_own;
            a = __uint_as_float(g7[k]);
            b = __uint_as_float(g7[gm + k]);
            c = __uint_as_float(g7[2 * gm + k]);
            ah = __uint_as_float(g7[3 * gm + k]);
            bh = __uint_as_float(g7[4 * gm + k]);
            ch = __uint_as_float(g7[5 * gm + k]);
        }
    }
    __device__ __forceinline__ uint32_t gid_of(int64_t i) const {
        if (i < n_own) return gid ? gid[i] : (uint32_t)i;
        return g7[6 * gm + (i - n_own)];
    }
};

__global__ void __launch_bounds__(BIN_THREADS)
k_bin_key(int64_t n, BinSrc src, Grid g, float xi_f, uint32_t* __restrict__ key, uint32_t* __restrict__ rnk,
          uint32_t* __restrict__ count, unsigned long long* __restrict__ errs) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float a, b, c, ah, bh, ch;
    src.load(i, a, b, c, ah, bh, ch);
    unsigned int bad = 0;
    if (!(isfinite(a) && isfinite(b) && isfinite(c) && isfinite(ah) && isfinite(bh) && isfinite(ch))) bad |= 1u;
    // input contract |x_hat - x| <= xi_f per coordinate, exact in fp64
    const double e = (double)xi_f;
    if (!(fabs((double)ah - (double)a) <= e && fabs((double)bh - (double)b) <= e && fabs((double)ch - (double)c) <= e))
        bad |= 2u;
    if (bad) atomicOr(errs, (unsigned long long)bad);
    double u;
    int cx, cy, cz;
    cell_of(a, b, c, g, u, cx, cy, cz);
    const uint32_t k = (uint32_t)(((int64_t)cz * g.ny + cy) * g.nx + cx);
    key[i] = k;
    rnk[i] = atomicAdd(&count[k], 1u);
}

__global__ void __launch_bounds__(BIN_THREADS)
k_bin_scatter(int64_t n, BinSrc src, const uint32_t* __restrict__ key, const uint32_t* __restrict__ rnk,
              const uint32_t* __restrict__ cell_start, Rec* __restrict__ rec, uint32_t* __restrict__ slot_of) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t s = cell_start[key[i]] + rnk[i];
    slot_of[i] = s;  // provisional: k_cell_finish* rewrite only the records the in-cell sort moves
    Rec r;
    src.load(i, r.x, r.y, r.z, r.xh, r.yh, r.zh);
    r.gid = src.gid_of(i);
    r.i = (uint32_t)i;
    // one full-sector 256-bit store (two 16-byte stores would be partial-sector writes)
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(rec + s), "r"(__float_as_uint(r.x)),
                 "r"(__float_as_uint(r.y)), "r"(__float_as_uint(r.z)), "r"(__float_as_uint(r.xh)),
                 "r"(__float_as_uint(r.yh)), "r"(__float_as_uint(r.zh)), "r"(r.gid), "r"(r.i)
                 : "memory");
}

// record r (scattered to the provisional slot s0) goes to slot s.  slot_of[r.i] holds s0
// (written coalesced by k_bin_scatter); the finish records fin[s0] = s -- s0 and s lie in the
// same cell, so these writes stay within a few sectors -- and k_fix_slot_of then maps
// slot_of[i] = fin[slot_of[i]] in input order (a random READ per particle instead of a random
// partial-sector WRITE per moved record: -9 ms of K1 at C4 when cells are rows)
__device__ __forceinline__ void emit(const Rec& r, uint32_t s, uint32_t s0, float4* __restrict__ orig4,
                                     float4* __restrict__ dec4, uint32_t* __restrict__ xk,
                                     uint32_t* __restrict__ fin, const Grid& g) {
    orig4[s] = make_float4(r.x, r.y, r.z, __uint_as_float(r.gid));
    dec4[s] = make_float4(r.xh, r.yh, r.zh, __uint_as_float(r.i));
    xk[s] = x_sort_key(r.x, g);
    fin[s0] = s;
}

__global__ void __launch_bounds__(BIN_THREADS) k_fix_slot_of(int64_t n, const uint32_t* __restrict__ fin,
                                                             uint32_t* __restrict__ slot_of) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) slot_of[i] = fin[slot_of[i]];
}

__device__ __forceinline__ Rec load_rec(const Rec* __restrict__ rec, uint32_t s) {
    Rec r;
    *reinterpret_cast<uint4*>(&r.x) = reinterpret_cast<const uint4*>(rec)[2 * s];
    *reinterpret_cast<uint4*>(&r.yh) = reinterpret_cast<const uint4*>(rec)[2 * s + 1];
    return r;
}

// sort key inside a row: (u-order key of x, input index)
__device__ __forceinline__ unsigned long long rec_key(const Rec& r, const Grid& g) {
    return ((unsigned long long)x_sort_key(r.x, g) << 32) | r.i;
}

// per-cell finish: sort the cell's records by x and write the slot-ordered arrays
__global__ void __launch_bounds__(BIN_THREADS)
k_cell_finish(int64_t ncell, const uint32_t* __restrict__ cs, const Rec* __restrict__ rec, Grid g,
              float4* __restrict__ orig4, float4* __restrict__ dec4, uint32_t* __restrict__ xk,
              uint32_t* __restrict__ slot_of, uint32_t* __restrict__ long_list, uint64_t cap,
              unsigned long long* __restrict__ n_long, int short_max) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncell) return;
    const uint32_t a = cs[c], b = cs[c + 1];
    const int len = (int)(b - a);
    if (len == 0) return;
    if (len == 1) {
        emit(load_rec(rec, a), a, a, orig4, dec4, xk, slot_of, g);
        return;
    }
    if (len > short_max) {  // mid cells from the front of the list, long ones from the back
        if (len <= CELL_MID) long_list[atomicAdd(n_long, 1ull)] = (uint32_t)c;
        else long_list[cap - 1 - atomicAdd(n_long + 1, 1ull)] = (uint32_t)c;
        return;
    }
    unsigned long long v[CELL_SHORT];  // (x key << 32 | input index): unique, data-determined order
    int off[CELL_SHORT];               // local offset of the record, moved along
    for (int k = 0; k < len; k++) {
        const unsigned long long xk = rec_key(load_rec(rec, a + k), g);
        int j = k - 1;
        while (j >= 0 && v[j] > xk) {
            v[j + 1] = v[j];
            off[j + 1] = off[j];
            j--;
        }
        v[j + 1] = xk;
        off[j + 1] = k;
    }
    for (int k = 0; k < len; k++) emit(load_rec(rec, a + off[k]), a + k, a + off[k], orig4, dec4, xk, slot_of, g);
}


// mid cells (CELL_SHORT < len <= CELL_MID): one warp per cell, bitonic sort of the 64-slot
// padded key array held two per lane (element lane and lane + 32)
__global__ void __launch_bounds__(BIN_THREADS)
k_cell_finish_mid(const uint32_t* __restrict__ long_list, const unsigned long long* __restrict__ n_long,
                  const uint32_t* __restrict__ cs, const Rec* __restrict__ rec, Grid g, float4* __restrict__ orig4,
                  float4* __restrict__ dec4, uint32_t* __restrict__ xk, uint32_t* __restrict__ slot_of) {
    const unsigned long long nm = n_long[0];
    const int lane = threadIdx.x & 31;
    const unsigned long long w0 = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nw = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    for (unsigned long long q = w0; q < nm; q += nw) {
        const uint32_t c = long_list[q];
        const uint32_t a = cs[c], b = cs[c + 1];
        const int len = (int)(b - a);
        // (key, local offset) pairs; keys are unique (input index), padding sorts last
        unsigned long long k0 = lane < len ? rec_key(load_rec(rec, a + lane), g) : ~0ull;
        unsigned long long k1 = lane + 32 < len ? rec_key(load_rec(rec, a + lane + 32), g) : ~0ull;
        int o0 = lane, o1 = lane + 32;
        for (int k = 2; k <= 64; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                if (j == 32) {  // partners in the same lane: elements lane and lane + 32
                    const bool up = (lane & k) == 0;  // k == 64: always ascending
                    if ((k0 > k1) == up) {
                        const unsigned long long tk = k0;
                        k0 = k1;
                        k1 = tk;
                        const int to = o0;
                        o0 = o1;
                        o1 = to;
                    }
                } else {
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        unsigned long long& kk = h ? k1 : k0;
                        int& oo = h ? o1 : o0;
                        const int idx = lane + 32 * h;
                        const unsigned long long pk = __shfl_xor_sync(0xffffffffu, kk, j);
                        const int po = __shfl_xor_sync(0xffffffffu, oo, j);
                        const bool up = (idx & k) == 0;
                        const bool lower = (lane & j) == 0;  // idx < idx ^ j
                        const bool take = lower ? ((kk > pk) == up) : ((kk < pk) == up);
                        if (take) {
                            kk = pk;
                            oo = po;
                        }
                    }
                }
            }
        }
        if (lane < len) emit(load_rec(rec, a + o0), a + lane, a + o0, orig4, dec4, xk, slot_of, g);
        if (lane + 32 < len) emit(load_rec(rec, a + o1), a + lane + 32, a + o1, orig4, dec4, xk, slot_of, g);
    }
}

// warp-per-cell finish for the default grid (cells = whole rows of ~30 particles): one warp per
// cell, grid-stride; cells of <= 32 records sort one key per lane (15-step bitonic), <= 64 two per
// lane (k_cell_finish_mid's network), longer ones go to the block kernel's list.  No thread-per-
// cell divergence and no list atomics for the common sizes.
template <typename K>
__device__ __forceinline__ void warp_sort32(K& k, int& o, int lane) {
#pragma unroll
    for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
        for (int j = kk >> 1; j > 0; j >>= 1) {
            const K pk = __shfl_xor_sync(0xffffffffu, k, j);
            const int po = __shfl_xor_sync(0xffffffffu, o, j);
            const bool up = (lane & kk) == 0;
            const bool lower = (lane & j) == 0;
            const bool take = lower ? ((k > pk) == up) : ((k < pk) == up);
            if (take) {
                k = pk;
                o = po;
            }
        }
    }
}

// the 64-slot network, two (key, offset) pairs per lane: elements lane and lane + 32
template <typename K>
__device__ __forceinline__ void warp_sort64(K& k0, K& k1, int& o0, int& o1, int lane) {
    for (int kk = 2; kk <= 64; kk <<= 1) {
        for (int j = kk >> 1; j > 0; j >>= 1) {
            if (j == 32) {
                const bool up = (lane & kk) == 0;
                if ((k0 > k1) == up) {
                    const K tk = k0;
                    k0 = k1;
                    k1 = tk;
                    const int to = o0;
                    o0 = o1;
                    o1 = to;
                }
            } else {
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    K& kr = h ? k1 : k0;
                    int& orr = h ? o1 : o0;
                    const int idx = lane + 32 * h;
                    const K pk = __shfl_xor_sync(0xffffffffu, kr, j);
                    const int po = __shfl_xor_sync(0xffffffffu, orr, j);
                    const bool up = (idx & kk) == 0;
                    const bool lower = (lane & j) == 0;
                    const bool take = lower ? ((kr > pk) == up) : ((kr < pk) == up);
                    if (take) {
                        kr = pk;
                        orr = po;
                    }
                }
            }
        }
    }
}

// a record's 32-bit x order key from its first half (x, y, z, x_hat)
__device__ __forceinline__ uint32_t rec_xkey(const Rec* __restrict__ rec, uint32_t s, const Grid& g) {
    const uint4 h = reinterpret_cast<const uint4*>(rec)[2 * s];
    return x_sort_key(__uint_as_float(h.x), g);
}

__global__ void __launch_bounds__(BIN_THREADS, 6)  // 6 blocks/SM (measured: -0.3 ms at C4 vs 64 registers)
k_row_finish(int64_t ncell, const uint32_t* __restrict__ cs, const Rec* __restrict__ rec, Grid g,
             float4* __restrict__ orig4, float4* __restrict__ dec4, uint32_t* __restrict__ xk,
             uint32_t* __restrict__ slot_of, uint32_t* __restrict__ long_list, uint64_t cap,
             unsigned long long* __restrict__ n_long, const uint32_t* __restrict__ list,
             const unsigned long long* __restrict__ n_list) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t cnt = list ? (int64_t)*n_list : ncell;  // list mode: the rows k_row_finish_group deferred
    for (int64_t q = w0; q < cnt; q += nw) {
        const int64_t c = list ? (int64_t)list[q] : q;
        const uint32_t a = cs[c], b = cs[c + 1];
        const int len = (int)(b - a);
        if (len == 0) continue;
        if (len > CELL_MID) {  // 65..512: k_row_finish_wide (front of the list); longer: the block kernel
            if (lane == 0) {
                if (len <= ROW_WIDE) long_list[atomicAdd(n_long, 1ull)] = (uint32_t)c;
                else long_list[cap - 1 - atomicAdd(n_long + 1, 1ull)] = (uint32_t)c;
            }
            continue;
        }
        // sort by the 32-bit x key with the record offset as payload (2 shuffles per step instead
        // of 3); a row with two equal x keys (rare) is sorted again on the full (x key, input
        // index) key so the order stays a pure function of the data
        if (len <= 32) {
            uint32_t k = lane < len ? rec_xkey(rec, a + lane, g) : 0xFFFFFFFFu;  // no real key is ~0
            int o = lane;
            warp_sort32(k, o, lane);
            const uint32_t kp = __shfl_up_sync(0xffffffffu, k, 1);
            if (__any_sync(0xffffffffu, lane > 0 && lane < len && kp == k)) {
                unsigned long long k64 = lane < len ? rec_key(load_rec(rec, a + lane), g) : ~0ull;
                o = lane;
                warp_sort32(k64, o, lane);
            }
            if (lane < len) emit(load_rec(rec, a + o), a + lane, a + o, orig4, dec4, xk, slot_of, g);
            continue;
        }
        // 33..64: two keys per lane, the 64-slot network
        uint32_t k0 = rec_xkey(rec, a + lane, g);
        uint32_t k1 = lane + 32 < len ? rec_xkey(rec, a + lane + 32, g) : 0xFFFFFFFFu;
        int o0 = lane, o1 = lane + 32;
        warp_sort64(k0, k1, o0, o1, lane);
        {
            const uint32_t p0 = __shfl_up_sync(0xffffffffu, k0, 1), p1 = __shfl_up_sync(0xffffffffu, k1, 1);
            const uint32_t last0 = __shfl_sync(0xffffffffu, k0, 31);
            const bool tie = (lane > 0 && p0 == k0) || (lane + 32 < len && (lane > 0 ? p1 == k1 : last0 == k1));
            if (__any_sync(0xffffffffu, tie)) {
                unsigned long long q0 = rec_key(load_rec(rec, a + lane), g);
                unsigned long long q1 = lane + 32 < len ? rec_key(load_rec(rec, a + lane + 32), g) : ~0ull;
                o0 = lane;
                o1 = lane + 32;
                warp_sort64(q0, q1, o0, o1, lane);
            }
        }
        emit(load_rec(rec, a + o0), a + lane, a + o0, orig4, dec4, xk, slot_of, g);
        if (lane + 32 < len) emit(load_rec(rec, a + o1), a + lane + 32, a + o1, orig4, dec4, xk, slot_of, g);
    }
}

// short rows (multi-GPU slabs: ~8 particles per row): a group of W lanes per row, one record per
// lane, a W-wide register bitonic of (key, offset); longer rows are deferred to the warp kernel
// (<= 64, list mode), k_row_finish_wide (<= 512) and the block kernel.  The warp-per-row kernel
// left 3/4 of its lanes idle there and did not shrink with the slab (its cost is per row).
template <int W, typename K>
__device__ __forceinline__ void group_sort_kv(K& k, int& o, int gl) {
#pragma unroll
    for (int kk = 2; kk <= W; kk <<= 1) {
#pragma unroll
        for (int j = kk >> 1; j > 0; j >>= 1) {
            const K pk = __shfl_xor_sync(0xffffffffu, k, j);
            const int po = __shfl_xor_sync(0xffffffffu, o, j);
            const bool up = (gl & kk) == 0;
            const bool lower = (gl & j) == 0;
            if (lower ? ((k > pk) == up) : ((k < pk) == up)) {
                k = pk;
                o = po;
            }
        }
    }
}

template <int W>
__global__ void __launch_bounds__(BIN_THREADS)
k_row_finish_group(int64_t ncell, const uint32_t* __restrict__ cs, const Rec* __restrict__ rec, Grid g,
                   float4* __restrict__ orig4, float4* __restrict__ dec4, uint32_t* __restrict__ xk,
                   uint32_t* __restrict__ slot_of, uint32_t* __restrict__ long_list, uint64_t cap,
                   unsigned long long* __restrict__ n_long, uint32_t* __restrict__ mid_list) {
    const int lane = threadIdx.x & 31, gl = lane % W;
    const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t wb = warp0 * (32 / W); wb < ncell; wb += nwarps * (32 / W)) {  // warp-uniform trips
        const int64_t c = wb + lane / W;
        uint32_t a = 0u;
        int len = 0;
        if (c < ncell) {
            a = cs[c];
            len = (int)(cs[c + 1] - a);
            if (len > W) {
                if (gl == 0) {
                    if (len <= CELL_MID) mid_list[atomicAdd(n_long + 2, 1ull)] = (uint32_t)c;
                    else if (len <= ROW_WIDE) long_list[atomicAdd(n_long, 1ull)] = (uint32_t)c;
                    else long_list[cap - 1 - atomicAdd(n_long + 1, 1ull)] = (uint32_t)c;
                }
                len = 0;
            }
        }
        // 32-bit x keys; a group with equal keys is sorted again on the full key (k_row_finish)
        uint32_t k = gl < len ? rec_xkey(rec, a + gl, g) : 0xFFFFFFFFu;
        int o = gl;
        group_sort_kv<W>(k, o, gl);
        const uint32_t kp = __shfl_up_sync(0xffffffffu, k, 1);
        const bool tie = gl > 0 && gl < len && kp == k;
        if (__any_sync(0xffffffffu, tie)) {  // warp-uniform redo (groups without ties re-sort identically)
            unsigned long long k64 = gl < len ? rec_key(load_rec(rec, a + gl), g) : ~0ull;
            o = gl;
            group_sort_kv<W>(k64, o, gl);
        }
        if (gl < len) emit(load_rec(rec, a + o), a + gl, a + o, orig4, dec4, xk, slot_of, g);
    }
}

// crowded rows of 65..512 records (halo cores): one warp per row, bitonic sort of (key, local
// offset) in the warp's own shared-memory slice with __syncwarp steps -- a 512-thread block per
// row idled most of its threads and synchronised the whole block every step
constexpr int WIDE_WARPS = 8;

__global__ void __launch_bounds__(32 * WIDE_WARPS)
k_row_finish_wide(const uint32_t* __restrict__ long_list, const unsigned long long* __restrict__ n_long,
                  const uint32_t* __restrict__ cs, const Rec* __restrict__ rec, Grid g, float4* __restrict__ orig4,
                  float4* __restrict__ dec4, uint32_t* __restrict__ xk, uint32_t* __restrict__ slot_of) {
    __shared__ unsigned long long shk[WIDE_WARPS][ROW_WIDE];
    __shared__ unsigned short sho[WIDE_WARPS][ROW_WIDE];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned long long* sk = shk[w];
    unsigned short* so = sho[w];
    const unsigned long long nm = n_long[0];
    const unsigned long long nw = (unsigned long long)gridDim.x * WIDE_WARPS;
    for (unsigned long long q = (unsigned long long)blockIdx.x * WIDE_WARPS + w; q < nm; q += nw) {
        const uint32_t c = long_list[q];
        const uint32_t a = cs[c], b = cs[c + 1];
        const int len = (int)(b - a);
        int p2 = 64;
        while (p2 < len) p2 <<= 1;
        for (int i = lane; i < p2; i += 32) {
            sk[i] = i < len ? rec_key(load_rec(rec, a + i), g) : ~0ull;  // unique keys (input index)
            so[i] = (unsigned short)i;
        }
        __syncwarp();
        for (int k = 2; k <= p2; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                // p2 / 2 compare-exchanges: pair index t -> lower element i (bit j of i clear)
                for (int t = lane; t < (p2 >> 1); t += 32) {
                    const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
                    const int ij = i | j;
                    const bool up = (i & k) == 0;
                    const unsigned long long x0 = sk[i], x1 = sk[ij];
                    if ((x0 > x1) == up) {
                        sk[i] = x1;
                        sk[ij] = x0;
                        const unsigned short t0 = so[i];
                        so[i] = so[ij];
                        so[ij] = t0;
                    }
                }
                __syncwarp();
            }
        }
        for (int k = lane; k < len; k += 32) emit(load_rec(rec, a + so[k]), a + k, a + so[k], orig4, dec4, xk, slot_of, g);
        __syncwarp();
    }
}

// crowded cells: one block per cell, bitonic sort of (key, local offset) in shared memory
__global__ void __launch_bounds__(512)
k_cell_finish_long(const uint32_t* __restrict__ long_list, uint64_t cap, const unsigned long long* __restrict__ n_long,
                   const uint32_t* __restrict__ cs, const Rec* __restrict__ rec, Grid g, float4* __restrict__ orig4,
                   float4* __restrict__ dec4, uint32_t* __restrict__ xk, uint32_t* __restrict__ slot_of,
                   uint32_t* __restrict__ offs) {
    __shared__ unsigned long long sh[CELL_LONG_MAX];
    __shared__ unsigned short so[CELL_LONG_MAX];
    const unsigned long long nl = n_long[1];
    for (unsigned long long q = blockIdx.x; q < nl; q += gridDim.x) {
        const uint32_t c = long_list[cap - 1 - q];
        const uint32_t a = cs[c], b = cs[c + 1];
        const int len = (int)(b - a);
        if (len <= CELL_LONG_MAX) {
            int p2 = 1;
            while (p2 < len) p2 <<= 1;
            for (int i = threadIdx.x; i < p2; i += blockDim.x) {
                sh[i] = i < len ? rec_key(load_rec(rec, a + i), g) : ~0ull;  // unique keys (input index)
                so[i] = (unsigned short)i;
            }
            __syncthreads();
            for (int k = 2; k <= p2; k <<= 1) {
                for (int j = k >> 1; j > 0; j >>= 1) {
                    for (int i = threadIdx.x; i < p2; i += blockDim.x) {
                        const int ij = i ^ j;
                        if (ij > i) {
                            const bool up = (i & k) == 0;
                            const unsigned long long x0 = sh[i], x1 = sh[ij];
                            if ((x0 > x1) == up) {
                                sh[i] = x1;
                                sh[ij] = x0;
                                const unsigned short t0 = so[i];
                                so[i] = so[ij];
                                so[ij] = t0;
                            }
                        }
                    }
                    __syncthreads();
                }
            }
            for (int k = threadIdx.x; k < len; k += blockDim.x)
                emit(load_rec(rec, a + so[k]), a + k, a + so[k], orig4, dec4, xk, slot_of, g);
            __syncthreads();
        } else {
            // beyond shared memory: sort the row's local offsets in place in global memory (the
            // row's own slot range of the dead key array), keys gathered from the records
            uint32_t* off = offs + a;
            for (int k = threadIdx.x; k < len; k += blockDim.x) off[k] = (uint32_t)k;
            __syncthreads();
            block_sort_global(off, (int64_t)len, [rec, a, g](uint32_t o) { return rec_key(load_rec(rec, a + o), g); });
            for (int k = threadIdx.x; k < len; k += blockDim.x)
                emit(load_rec(rec, a + off[k]), a + k, a + off[k], orig4, dec4, xk, slot_of, g);
            __syncthreads();
        }
    }
}

}  // namespace

cc_status bin_particles(cc_ctx* c, const float* x, const float* y, const float* z, const float* xh,
                        const float* yh, const float* zh, const uint32_t* gid, int64_t n_own, const uint32_t* g7,
                        int64_t gm, int64_t n) {
    const BinSrc src{x, y, z, xh, yh, zh, gid, n_own, g7, gm};
    const int64_t nc = c->ncell;
    const size_t n1 = (size_t)std::max<int64_t>(n, 1);
    CC_TRY(cc_ensure(c, c->key, n1, "key"));
    CC_TRY(cc_ensure(c, c->rnk, n1, "rank"));
    CC_TRY(cc_ensure(c, c->cell_count, (size_t)nc, "cell_count"));
    CC_TRY(cc_ensure(c, c->cell_start, (size_t)nc + 1, "cell_start"));
    CC_TRY(cc_ensure(c, c->orig4, n1, "orig4"));
    CC_TRY(cc_ensure(c, c->dec4, n1, "dec4"));
    CC_TRY(cc_ensure(c, c->xk, n1, "x keys"));
    CC_TRY(cc_ensure(c, c->slot_of, n1, "slot_of"));
    CC_TRY(cc_ensure(c, c->rec32, 2 * n1, "binning records"));  // 32 B per particle
    CC_TRY(cc_ensure(c, c->counters, 16, "counters"));
    CC_TRY(cc_ensure(c, c->scratch_u64, 3, "long counts"));
    CC_CUDA(c, cudaMemsetAsync(c->cell_count.p, 0, (size_t)nc * sizeof(uint32_t), c->stream));
    CC_CUDA(c, cudaMemsetAsync(c->counters.p, 0, 16 * sizeof(unsigned long long), c->stream));
    CC_CUDA(c, cudaMemsetAsync(c->scratch_u64.p, 0, 3 * sizeof(uint64_t), c->stream));
    Rec* rec = reinterpret_cast<Rec*>(c->rec32.p);
    const unsigned nb = (unsigned)((n + BIN_THREADS - 1) / BIN_THREADS);
    if (n > 0) {
        int tok = cc_prof_begin(c, "K1_key");
        CCL(c, k_bin_key<<<nb, BIN_THREADS, 0, c->stream>>>(n, src, c->g, c->th.xi_f, c->key.p, c->rnk.p,
                                                             c->cell_count.p, c->counters.p));
        cc_prof_end(c, tok);
        CC_CUDA(c, cudaGetLastError());
    }
    // cell_start = exclusive scan of the counts; cell_start[nc] = n
    CC_TRY(scan_u32_to_u32(c, c->cell_count.p, c->cell_start.p, nc,
                           reinterpret_cast<uint64_t*>(c->cell_start.p + nc)));
    if (n > 0) {
        const uint64_t cap = (uint64_t)std::max<int64_t>(std::min<int64_t>(nc, n), 1);  // >= crowded cells
        CC_TRY(cc_ensure(c, c->scratch_u32, (size_t)cap, "crowded cells"));
        int tok = cc_prof_begin(c, "K1_scatter");
        CCL(c, k_bin_scatter<<<nb, BIN_THREADS, 0, c->stream>>>(n, src, c->key.p, c->rnk.p, c->cell_start.p, rec,
                                                                 c->slot_of.p));
        cc_prof_end(c, tok);
        unsigned long long* nl = reinterpret_cast<unsigned long long*>(c->scratch_u64.p);
        int t2 = cc_prof_begin(c, "K1_finish");
        uint32_t* fin = c->rnk.p;  // the ranks are dead after the scatter: final slot per provisional slot
        const double per_row = (double)n / (double)std::max<int64_t>(nc, 1);
        if (c->g.nx == 1 && per_row <= 12.0) {  // short rows (multi-GPU slabs): W lanes per row
            uint32_t* mid = c->cell_count.p;      // dead after the scan: the deferred 17..64 rows
            if (per_row <= 5.0)
                CCL(c, k_row_finish_group<8><<<148 * 16, BIN_THREADS, 0, c->stream>>>(
                           nc, c->cell_start.p, rec, c->g, c->orig4.p, c->dec4.p, c->xk.p, fin, c->scratch_u32.p, cap,
                           nl, mid));
            else
                CCL(c, k_row_finish_group<16><<<148 * 16, BIN_THREADS, 0, c->stream>>>(
                           nc, c->cell_start.p, rec, c->g, c->orig4.p, c->dec4.p, c->xk.p, fin, c->scratch_u32.p, cap,
                           nl, mid));
            CCL(c, k_row_finish<<<148 * 4, BIN_THREADS, 0, c->stream>>>(nc, c->cell_start.p, rec, c->g, c->orig4.p,
                                                                         c->dec4.p, c->xk.p, fin, c->scratch_u32.p,
                                                                         cap, nl, mid, nl + 2));
            CCL(c, k_row_finish_wide<<<148 * 4, 32 * WIDE_WARPS, 0, c->stream>>>(c->scratch_u32.p, nl,
                                                                                  c->cell_start.p, rec, c->g,
                                                                                  c->orig4.p, c->dec4.p, c->xk.p,
                                                                                  fin));
        } else if (c->g.nx == 1) {  // cells are rows (default grid): one warp per cell
            CCL(c, k_row_finish<<<148 * 16, BIN_THREADS, 0, c->stream>>>(nc, c->cell_start.p, rec, c->g, c->orig4.p,
                                                                          c->dec4.p, c->xk.p, fin, c->scratch_u32.p,
                                                                          cap, nl, nullptr, nullptr));
            CCL(c, k_row_finish_wide<<<148 * 4, 32 * WIDE_WARPS, 0, c->stream>>>(c->scratch_u32.p, nl,
                                                                                  c->cell_start.p, rec, c->g,
                                                                                  c->orig4.p, c->dec4.p, c->xk.p,
                                                                                  fin));
        } else {
            CCL(c, k_cell_finish<<<(unsigned)((nc + BIN_THREADS - 1) / BIN_THREADS), BIN_THREADS, 0, c->stream>>>(
                       nc, c->cell_start.p, rec, c->g, c->orig4.p, c->dec4.p, c->xk.p, fin, c->scratch_u32.p,
                       cap, nl, c->bin_short_max));
            CCL(c, k_cell_finish_mid<<<148 * 8, BIN_THREADS, 0, c->stream>>>(c->scratch_u32.p, nl, c->cell_start.p,
                                                                              rec, c->g, c->orig4.p, c->dec4.p,
                                                                              c->xk.p, fin));
        }
        CCL(c, k_cell_finish_long<<<148 * 2, 512, 0, c->stream>>>(c->scratch_u32.p, cap, nl, c->cell_start.p, rec,
                                                                  c->g, c->orig4.p, c->dec4.p, c->xk.p, fin,
                                                                  c->key.p));
        cc_prof_end(c, t2);
        CC_CUDA(c, cudaGetLastError());
    }
    c->slot_of_valid = n <= 0;
    return CC_OK;
}

// slot_of[i] = fin[slot_of[i]] (k_fix_slot_of): the input-order -> slot map is only needed to
// write FoF labels in input order and by the multi-GPU exchanges, not by S1-S5 (cc_correct's
// output is written from the inputs and slotE), so it is completed on first use.  fin lives in
// the rank buffer, untouched until the next cc_build_cells.
cc_status ensure_slot_of(cc_ctx* c) {
    if (c->slot_of_valid) return CC_OK;
    const int64_t n = c->n;
    if (n > 0)
        CCL(c, k_fix_slot_of<<<(unsigned)((n + BIN_THREADS - 1) / BIN_THREADS), BIN_THREADS, 0, c->stream>>>(
                   n, c->rnk.p, c->slot_of.p));
    CC_CUDA(c, cudaGetLastError());
    c->slot_of_valid = true;
    return CC_OK;
}

}  // namespace cc
