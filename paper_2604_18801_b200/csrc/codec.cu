// codec.cu -- f1 edit log on the device: compaction and m-bit
// quantisation of the edits Delta = P_hat - P_hat0 (Alg. 1 lines 11-13; §III-B
// "Compaction, quantization, and lossless compression") and the reconstruction
// x_rec = x_hat0 + scatter(dequantise(q), flags) (§III-B "Reconstruction").
// Readings R29-R32: coordinate k = 3i + a, flags LSB-first in bytes; q =
// rint(Delta / s) in fp64 with s = xi_f 2^(1-m), then stepped toward x while the decoder's
// x_rec = fl32((double)x_hat0 + (double)q s) would leave |x_rec - x| <= xi_f (R32).
//
// One thread per particle (a block walks SUB sub-tiles of CT particles), HBM-bound and fully
// coalesced on the SoA coordinates.  A warp owns
// 32 particles = 96 coordinates = 3 flag words: each lane forms its 3-bit mask, the words are
// assembled with one shuffle + ballot each.  Edits are written in ascending k through a
// reduce-then-scan over blocks (count pass, one-block scan of the block totals, fill pass that
// recomputes the masks instead of storing them).  Decoding runs the same three passes with the
// masks read from the flags.
#include <cstdlib>

#include "cc_internal.cuh"

namespace cc {
namespace {

constexpr int CT = 256;         // threads per block; one particle per thread per sub-tile
constexpr int CW = CT / 32;
constexpr int SUB = 8;          // sub-tiles per block: a block owns CT * SUB consecutive particles
constexpr int TILE = CT * SUB;  // (keeps the block-sum scan short: N / 2048 entries)
constexpr int SCAN_ITEMS = 8;   // block sums per thread per k_edit_scan iteration

struct EncMask {
    const float *xh, *yh, *zh, *xc, *yc, *zc;
    __device__ uint32_t operator()(int64_t i) const {
        return (uint32_t)(__ldg(xc + i) != __ldg(xh + i)) | (uint32_t)(__ldg(yc + i) != __ldg(yh + i)) << 1 |
               (uint32_t)(__ldg(zc + i) != __ldg(zh + i)) << 2;
    }
};

struct DecMask {
    const uint8_t* flags;
    __device__ uint32_t operator()(int64_t i) const {
        const int64_t k = 3 * i;
        const int off = (int)(k & 7);
        uint32_t v = __ldg(flags + (k >> 3));
        if (off > 5) v |= (uint32_t)__ldg(flags + (k >> 3) + 1) << 8;  // bits 3i..3i+2 span two bytes
        return (v >> off) & 7u;
    }
};

// block-exclusive prefix of a per-thread count; *total = block total
__device__ __forceinline__ uint32_t block_excl(uint32_t v, uint32_t* total) {
    __shared__ uint32_t sw[CW];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();  // sw may still be read by the previous call
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
    }
    if (lane == 31) sw[w] = inc;
    __syncthreads();
    uint32_t wex = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < CW; k++) {
        wex += (k < w) ? sw[k] : 0u;
        tot += sw[k];
    }
    *total = tot;
    return wex + inc - v;
}

// pass 1 (encode): flags words + block edit counts; bound check |Delta| <= 2 xi_f (R30)
__global__ void __launch_bounds__(CT) k_edit_flags(int64_t n, EncMask mk, uint32_t* flags_w, int64_t nbytes,
                                                   unsigned long long* bsum, double lim, unsigned int* err) {
    const int lane = threadIdx.x & 31;
    uint32_t cnt = 0;
    for (int t = 0; t < SUB; t++) {
        const int64_t i0 = (int64_t)blockIdx.x * TILE + t * CT;
        if (i0 >= n) break;  // uniform over the block
        const int64_t i = i0 + threadIdx.x;
        uint32_t m3 = 0;
        if (i < n) {
            m3 = mk(i);
            if (m3) {
                const float* h[3] = {mk.xh, mk.yh, mk.zh};
                const float* p[3] = {mk.xc, mk.yc, mk.zc};
#pragma unroll
                for (int a = 0; a < 3; a++)
                    if ((m3 >> a & 1u) && fabs((double)p[a][i] - (double)h[a][i]) > lim) atomicOr(err, 1u);
            }
        }
        cnt += __popc(m3);
        // 96 bits of the warp's 32 particles -> 3 words (bit b of word j = coordinate 32j + b)
        const int64_t wbase = (i0 + (threadIdx.x & ~31)) / 32 * 3;
#pragma unroll
        for (int j = 0; j < 3; j++) {
            const int b = 32 * j + lane;
            const uint32_t src = __shfl_sync(0xffffffffu, m3, b / 3);
            const uint32_t word = __ballot_sync(0xffffffffu, (src >> (b % 3)) & 1u);
            const int64_t wi = wbase + j;
            if (lane == j) {
                if (4 * wi + 4 <= nbytes) {
                    flags_w[wi] = word;
                } else {
                    uint8_t* fb = reinterpret_cast<uint8_t*>(flags_w);
                    for (int64_t q = 4 * wi; q < nbytes; q++) fb[q] = (uint8_t)(word >> (8 * (q - 4 * wi)));
                }
            }
        }
    }
    uint32_t tot;
    (void)block_excl(cnt, &tot);
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// pass 1 (decode): block counts of set flags
__global__ void __launch_bounds__(CT) k_edit_count(int64_t n, DecMask mk, unsigned long long* bsum) {
    uint32_t cnt = 0;
    for (int t = 0; t < SUB; t++) {
        const int64_t i = (int64_t)blockIdx.x * TILE + t * CT + threadIdx.x;
        if (i < n) cnt += __popc(mk(i));
    }
    uint32_t tot;
    (void)block_excl(cnt, &tot);
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// pass 2: exclusive scan of the block totals in place (one block, SCAN_ITEMS per thread per
// iteration); bsum[nb] = total
__global__ void __launch_bounds__(1024) k_edit_scan(int64_t nb, unsigned long long* bsum) {
    __shared__ unsigned long long sw[32];
    __shared__ unsigned long long carry_s;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    for (int64_t off = 0; off < nb; off += 1024 * SCAN_ITEMS) {
        const int64_t i0 = off + (int64_t)threadIdx.x * SCAN_ITEMS;
        unsigned long long item[SCAN_ITEMS];
        unsigned long long v = 0;
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; k++) {
            item[k] = i0 + k < nb ? bsum[i0 + k] : 0ull;
            v += item[k];
        }
        unsigned long long inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        if (lane == 31) sw[w] = inc;
        __syncthreads();
        unsigned long long wex = 0, tot = 0;
        for (int k = 0; k < 32; k++) {
            wex += (k < w) ? sw[k] : 0ull;
            tot += sw[k];
        }
        unsigned long long run = carry_s + wex + inc - v;
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; k++) {
            if (i0 + k < nb) bsum[i0 + k] = run;
            run += item[k];
        }
        __syncthreads();
        if (threadIdx.x == 0) carry_s += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) bsum[nb] = carry_s;
}

// pass 3 (encode): q = rint(Delta / s) in ascending k (R30), bound-safe against the decoder's
// fp32 rounding (R32; err bit 2 if 8 steps do not suffice)
__global__ void __launch_bounds__(CT) k_edit_fill(int64_t n, EncMask mk, const float* x, const float* y,
                                                  const float* z, const unsigned long long* bsum, double s,
                                                  double xi_f, long long* q, int64_t cap, unsigned int* err) {
    int64_t base = (int64_t)bsum[blockIdx.x];
    const float* h[3] = {mk.xh, mk.yh, mk.zh};
    const float* p[3] = {mk.xc, mk.yc, mk.zc};
    const float* org[3] = {x, y, z};
    for (int t = 0; t < SUB; t++) {
        const int64_t i0 = (int64_t)blockIdx.x * TILE + t * CT;
        if (i0 >= n) break;  // uniform over the block
        const int64_t i = i0 + threadIdx.x;
        const uint32_t m3 = i < n ? mk(i) : 0u;  // recomputed (reading pass 1's flags instead measured slower: 4.04 vs 3.44 ms on C4)
        uint32_t tot;
        int64_t o = base + block_excl(__popc(m3), &tot);
        base += tot;
        if (!m3) continue;
#pragma unroll
        for (int a = 0; a < 3; a++) {
            if (m3 >> a & 1u) {
                const double hv = (double)h[a][i];
                const double d = (double)p[a][i] - hv;  // exact
                long long qi = (long long)rint(d / s);
                const double xo = (double)__ldg(org[a] + i);
                for (int step = 0;; step++) {
                    const double dev = (double)(float)(hv + (double)qi * s) - xo;
                    if (fabs(dev) <= xi_f) break;
                    if (step == 8) {
                        atomicOr(err, 2u);
                        break;
                    }
                    qi += dev > 0 ? -1 : 1;
                }
                if (o < cap) q[o] = qi;
                o++;
            }
        }
    }
}

// ---- single-pass encode (decoupled look-back): each block takes the next tile by ticket, builds
// its flag words and edit count (the inputs are read once), publishes the count, sums its
// predecessors' published counts / inclusive prefixes, and writes its edits at that offset.
// Replaces pass 1 + scan + pass 3 when q is written (the count-only call keeps the two-pass path).

__global__ void __launch_bounds__(CT) k_edit_encode1(int64_t n, EncMask mk, const float* x, const float* y,
                                                    const float* z, uint32_t* flags_w, int64_t nbytes,
                                                    unsigned long long* __restrict__ status,
                                                    unsigned int* __restrict__ ticket, double s, double xi_f,
                                                    double lim, long long* q, int64_t cap,
                                                    unsigned long long* total, unsigned int* err) {
    __shared__ unsigned int tile_sh;
    __shared__ unsigned long long base_sh;
    if (threadIdx.x == 0) tile_sh = atomicAdd(ticket, 1u);
    __syncthreads();
    const unsigned int tile = tile_sh;
    const int lane = threadIdx.x & 31;
    const float* h[3] = {mk.xh, mk.yh, mk.zh};
    const float* p[3] = {mk.xc, mk.yc, mk.zc};
    const float* org[3] = {x, y, z};
    // pass A: masks (kept, 3 bits per sub-tile), flag words, bound check, count
    uint32_t masks = 0u, cnt = 0u;
    for (int t = 0; t < SUB; t++) {
        const int64_t i0 = (int64_t)tile * TILE + t * CT;
        if (i0 >= n) break;  // uniform over the block
        const int64_t i = i0 + threadIdx.x;
        uint32_t m3 = 0;
        if (i < n) {
            m3 = mk(i);
            if (m3) {
#pragma unroll
                for (int a = 0; a < 3; a++)
                    if ((m3 >> a & 1u) && fabs((double)p[a][i] - (double)h[a][i]) > lim) atomicOr(err, 1u);
            }
        }
        masks |= m3 << (3 * t);
        cnt += __popc(m3);
        const int64_t wbase = (i0 + (threadIdx.x & ~31)) / 32 * 3;
#pragma unroll
        for (int j = 0; j < 3; j++) {
            const int b = 32 * j + lane;
            const uint32_t src = __shfl_sync(0xffffffffu, m3, b / 3);
            const uint32_t word = __ballot_sync(0xffffffffu, (src >> (b % 3)) & 1u);
            const int64_t wi = wbase + j;
            if (lane == j) {
                if (4 * wi + 4 <= nbytes) {
                    flags_w[wi] = word;
                } else {
                    uint8_t* fb = reinterpret_cast<uint8_t*>(flags_w);
                    for (int64_t qq = 4 * wi; qq < nbytes; qq++) fb[qq] = (uint8_t)(word >> (8 * (qq - 4 * wi)));
                }
            }
        }
    }
    uint32_t tot;
    (void)block_excl(cnt, &tot);  // the tile's edit count
    // publish, look back (warp 0, 32 predecessors per step), publish the inclusive prefix
    if (threadIdx.x < 32) {
        const unsigned long long ex = lookback_warp0(status, tile, tot);
        if (lane == 0) base_sh = ex;
        if (lane == 0 && (int64_t)(tile + 1) * TILE >= n) *total = base_sh + tot;  // the last tile
    }
    __syncthreads();
    int64_t base = (int64_t)base_sh;
    // pass B: the edits in ascending k (sub-tile by sub-tile, R30, R32); values re-read only for
    // flagged coordinates (the tile was just read: L2)
    for (int t = 0; t < SUB; t++) {
        const int64_t i0 = (int64_t)tile * TILE + t * CT;
        if (i0 >= n) break;  // uniform over the block
        const int64_t i = i0 + threadIdx.x;
        const uint32_t m3 = (masks >> (3 * t)) & 7u;
        uint32_t stot;
        int64_t o = base + block_excl(__popc(m3), &stot);
        base += stot;
        if (!m3) continue;
#pragma unroll
        for (int a = 0; a < 3; a++) {
            if (m3 >> a & 1u) {
                const double hv = (double)h[a][i];
                const double d = (double)p[a][i] - hv;  // exact
                long long qi = (long long)rint(d / s);
                const double xo = (double)__ldg(org[a] + i);
                for (int step = 0;; step++) {
                    const double dev = (double)(float)(hv + (double)qi * s) - xo;
                    if (fabs(dev) <= xi_f) break;
                    if (step == 8) {
                        atomicOr(err, 2u);
                        break;
                    }
                    qi += dev > 0 ? -1 : 1;
                }
                if (o < cap) q[o] = qi;
                o++;
            }
        }
    }
}

// pass 3 (decode): x_rec = fl32((double)x_hat0 + (double)q s) where flagged, x_hat0 elsewhere (R31)
__global__ void __launch_bounds__(CT) k_edit_apply(int64_t n, DecMask mk, const unsigned long long* bsum,
                                                   double s, const long long* q, int64_t n_edits,
                                                   const float* xh, const float* yh, const float* zh, float* xr,
                                                   float* yr, float* zr) {
    int64_t base = (int64_t)bsum[blockIdx.x];
    const float* h[3] = {xh, yh, zh};
    float* r[3] = {xr, yr, zr};
    for (int t = 0; t < SUB; t++) {
        const int64_t i0 = (int64_t)blockIdx.x * TILE + t * CT;
        if (i0 >= n) break;  // uniform over the block
        const int64_t i = i0 + threadIdx.x;
        const uint32_t m3 = i < n ? mk(i) : 0u;
        uint32_t tot;
        int64_t o = base + block_excl(__popc(m3), &tot);
        base += tot;
        if (i >= n) continue;
#pragma unroll
        for (int a = 0; a < 3; a++) {
            float v = __ldg(h[a] + i);
            if (m3 >> a & 1u) {
                if (o < n_edits) v = (float)((double)v + (double)__ldg(q + o) * s);
                o++;
            }
            r[a][i] = v;
        }
    }
}

// ---- decode with 4 particles per thread (float4 loads/stores; every pointer 16-byte aligned;
// C4: 1.99 vs 3.16 ms per decode).  Same tiles and block sums as the scalar kernels (a block = 2
// sub-tiles of 4 * CT particles), same order.
constexpr int SUB4 = TILE / (4 * CT);

__device__ __forceinline__ void ld4(const float* p, int64_t i, int64_t n, float v[4]) {
    if (i + 3 < n) {
        const float4 f = __ldg(reinterpret_cast<const float4*>(p + i));
        v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
    } else {
#pragma unroll
        for (int k = 0; k < 4; k++) v[k] = i + k < n ? __ldg(p + i + k) : 0.0f;
    }
}

__global__ void __launch_bounds__(CT) k_edit_apply4(int64_t n, const uint8_t* __restrict__ flags,
                                                    const unsigned long long* bsum, double s,
                                                    const long long* q, int64_t n_edits, const float* xh,
                                                    const float* yh, const float* zh, float* xr, float* yr,
                                                    float* zr) {
    int64_t base = (int64_t)bsum[blockIdx.x];
    const float* hp[3] = {xh, yh, zh};
    float* rp[3] = {xr, yr, zr};
    for (int t = 0; t < SUB4; t++) {
        const int64_t i0 = (int64_t)blockIdx.x * TILE + (int64_t)t * 4 * CT;
        if (i0 >= n) break;  // uniform over the block
        const int64_t i = i0 + 4 * threadIdx.x;
        uint32_t m = 0;
        if (i < n) {
            // bits 3i .. 3i+11 (3i = 12 (i/4): offset 0 or 4 inside byte 3i/8)
            const int64_t bit = 3 * i, last = 3 * (i + 3 < n ? i + 3 : n - 1) + 2;
            uint32_t v = __ldg(flags + (bit >> 3));
            if ((last >> 3) > (bit >> 3)) v |= (uint32_t)__ldg(flags + (bit >> 3) + 1) << 8;
            m = (v >> (bit & 7)) & 0xFFFu;
            const int valid = (int)(n - i < 4 ? n - i : 4);
            m &= (1u << (3 * valid)) - 1u;
        }
        uint32_t tot;
        int64_t o = base + block_excl(__popc(m), &tot);
        base += tot;
        if (i >= n) continue;
#pragma unroll
        for (int a = 0; a < 3; a++) {
            float h[4];
            ld4(hp[a], i, n, h);
            float r[4];
#pragma unroll
            for (int k = 0; k < 4; k++) r[k] = h[k];
            // edits of this thread in k-major order: particle k, axis a -> rank among set bits below
#pragma unroll
            for (int k = 0; k < 4; k++)
                if (m >> (3 * k + a) & 1u) {
                    const int64_t e = o + __popc(m & ((1u << (3 * k + a)) - 1u));
                    if (e < n_edits) r[k] = (float)((double)h[k] + (double)__ldg(q + e) * s);
                }
            if (i + 3 < n) {
                *reinterpret_cast<float4*>(rp[a] + i) = make_float4(r[0], r[1], r[2], r[3]);
            } else {
                for (int k = 0; k < 4 && i + k < n; k++) rp[a][i + k] = r[k];
            }
        }
    }
}

// m-bit packing (R33): field e = bits [e w, (e+1) w) of the LSB-first word stream, w = m + 2,
// two's complement.  Pack: one thread per output WORD gathers the fields overlapping it (no
// atomics, coalesced stores); unpack: one thread per edit reads the 2-3 words of its field.
__global__ void __launch_bounds__(CT) k_edit_pack(int64_t n_edits, int w, long long lim, const long long* __restrict__ q,
                                                  uint32_t* __restrict__ words, int64_t nw, unsigned int* err) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nw) return;
    const int64_t b0 = 32 * k;
    const int64_t e0 = b0 / w, e1 = min((b0 + 31) / w, n_edits - 1);
    const unsigned long long mask = (w >= 64) ? ~0ull : ((1ull << w) - 1ull);
    uint32_t word = 0u;
    for (int64_t e = e0; e <= e1; e++) {
        const long long v = __ldg(q + e);
        if (v > lim || v < -lim) atomicOr(err, 4u);
        const unsigned long long u = (unsigned long long)v & mask;
        const int64_t sh = e * w - b0;  // field start relative to the word, > -w and < 32
        word |= sh >= 0 ? (uint32_t)(u << sh) : (uint32_t)(u >> (-sh));
    }
    words[k] = word;
}

__global__ void __launch_bounds__(CT) k_edit_unpack(int64_t n_edits, int w, const uint32_t* __restrict__ words,
                                                    int64_t nw, long long* __restrict__ q) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n_edits) return;
    const int64_t bit = e * w, k = bit >> 5;
    const int off = (int)(bit & 31);
    const unsigned long long lo = (unsigned long long)__ldg(words + k) |
                                  (k + 1 < nw ? (unsigned long long)__ldg(words + k + 1) << 32 : 0ull);
    unsigned long long u = lo >> off;
    if (off + w > 64 && k + 2 < nw) u |= (unsigned long long)__ldg(words + k + 2) << (64 - off);
    const unsigned long long mask = (1ull << w) - 1ull;
    u &= mask;
    if ((u >> (w - 1)) & 1ull) u |= ~mask;  // sign extension
    q[e] = (long long)u;
}

bool aligned4(const void* p) { return ((uintptr_t)p & 3u) == 0; }
bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

}  // namespace
}  // namespace cc

using namespace cc;

static cc_status edit_common(cc_ctx* c, int64_t n, int64_t* nb_out) {
    if (!c) return CC_E_ARG;
    if (c->dead) return cc_fail(c, CC_E_CUDA, "context unusable after a CUDA error");
    cudaSetDevice(c->device);
    if (n < 0 || 3 * n >= ((int64_t)1 << 62)) return cc_fail(c, CC_E_ARG, "n");
    if (c->p.m < 2 || c->p.m > 40 || !(c->p.xi > 0)) return cc_fail(c, CC_E_ARG, "edit log needs xi > 0, 2 <= m <= 40");
    const int64_t nb = (n + TILE - 1) / TILE;
    CC_TRY(cc_ensure(c, c->codec_bsum, (size_t)nb + 2, "edit-log block sums"));
    *nb_out = nb;
    return CC_OK;
}

cc_status cc_edit_encode(cc_ctx* c, int64_t n, const float* x, const float* y, const float* z,
                         const float* xh0, const float* yh0, const float* zh0,
                         const float* xc, const float* yc, const float* zc, uint8_t* flags, int64_t* q,
                         int64_t cap, int64_t* n_edits_h) {
    int64_t nb = 0;
    CC_TRY(edit_common(c, n, &nb));
    if (!n_edits_h || cap < 0) return cc_fail(c, CC_E_ARG, "null n_edits_h or cap < 0");
    *n_edits_h = 0;
    if (n == 0) return CC_OK;
    if (!x || !y || !z || !xh0 || !yh0 || !zh0 || !xc || !yc || !zc || !flags || (cap > 0 && !q))
        return cc_fail(c, CC_E_ARG, "null buffer");
    if (!aligned4(flags)) return cc_fail(c, CC_E_ARG, "flags must be 4-byte aligned");
    const double xi = (double)(float)c->p.xi, s = std::ldexp(xi, 1 - c->p.m);
    unsigned long long* bsum = c->codec_bsum.p;
    unsigned int* err = reinterpret_cast<unsigned int*>(bsum + nb + 1);
    CC_CUDA(c, cudaMemsetAsync(err, 0, sizeof(unsigned long long), c->stream));
    const EncMask mk{xh0, yh0, zh0, xc, yc, zc};
    const int64_t nbytes = (3 * n + 7) / 8;
    if (cap > 0 && std::getenv("CC_CODEC_TWO_PASS") == nullptr) {
        // single pass (decoupled look-back); q must have room for every edit: if the count
        // exceeds cap the call fails with CC_E_OOM after counting (q then holds the first cap)
        CC_TRY(cc_ensure(c, c->codec_status, (size_t)nb + 2, "edit-log tile status"));
        unsigned long long* st = c->codec_status.p;
        CC_CUDA(c, cudaMemsetAsync(st, 0, ((size_t)nb + 2) * sizeof(unsigned long long), c->stream));
        unsigned int* ticket = reinterpret_cast<unsigned int*>(st + nb);
        unsigned long long* total = st + nb + 1;
        int tok = cc_prof_begin(c, "F1_encode");
        CCL(c, k_edit_encode1<<<(unsigned)nb, CT, 0, c->stream>>>(n, mk, x, y, z, reinterpret_cast<uint32_t*>(flags),
                                                                  nbytes, st, ticket, s, xi, 2.0 * xi,
                                                                  reinterpret_cast<long long*>(q), cap, total, err));
        cc_prof_end(c, tok);
        CC_CUDA(c, cudaGetLastError());
        unsigned long long ht[2];
        CC_CUDA(c, cudaMemcpyAsync(&ht[0], total, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
        CC_CUDA(c, cudaMemcpyAsync(&ht[1], err, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
        CC_CUDA(c, cudaStreamSynchronize(c->stream));
        *n_edits_h = (int64_t)ht[0];
        if ((unsigned int)ht[1] & 1u) return cc_fail(c, CC_E_BOUND, "an edit exceeds 2 xi_f (corrected coordinates out of bound)");
        if ((int64_t)ht[0] > cap) return cc_fail(c, CC_E_OOM, "more edits than cap (*n_edits_h holds the count)");
        if ((unsigned int)ht[1] & 2u) return cc_fail(c, CC_E_BOUND, "no lattice index reconstructs within xi_f (R32)");
        return CC_OK;
    }
    int tok = cc_prof_begin(c, "F1_encode");
    CCL(c, k_edit_flags<<<(unsigned)nb, CT, 0, c->stream>>>(n, mk, reinterpret_cast<uint32_t*>(flags), nbytes, bsum,
                                                           2.0 * xi, err));
    CCL(c, k_edit_scan<<<1, 1024, 0, c->stream>>>(nb, bsum));
    cc_prof_end(c, tok);
    unsigned long long h[2];
    CC_CUDA(c, cudaMemcpyAsync(h, bsum + nb, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    *n_edits_h = (int64_t)h[0];
    if ((unsigned int)h[1]) return cc_fail(c, CC_E_BOUND, "an edit exceeds 2 xi_f (corrected coordinates out of bound)");
    if ((int64_t)h[0] > cap) return cc_fail(c, CC_E_OOM, "more edits than cap (*n_edits_h holds the count)");
    tok = cc_prof_begin(c, "F1_encode");
    // (a float4 variant of this pass, 4 particles per thread, measured slower on C4: 6.57 vs
    // 5.92 ms per encode; the scalar pass stays)
    CCL(c, k_edit_fill<<<(unsigned)nb, CT, 0, c->stream>>>(n, mk, x, y, z, bsum, s, xi,
                                                          reinterpret_cast<long long*>(q), cap, err));
    cc_prof_end(c, tok);
    CC_CUDA(c, cudaGetLastError());
    unsigned int e2 = 0;
    CC_CUDA(c, cudaMemcpyAsync(&e2, err, sizeof(e2), cudaMemcpyDeviceToHost, c->stream));
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    if (e2) return cc_fail(c, CC_E_BOUND, "no lattice index reconstructs within xi_f (R32)");
    return CC_OK;
}

cc_status cc_edit_decode(cc_ctx* c, int64_t n, const float* xh0, const float* yh0, const float* zh0,
                         const uint8_t* flags, const int64_t* q, int64_t n_edits, float* xr, float* yr, float* zr) {
    int64_t nb = 0;
    CC_TRY(edit_common(c, n, &nb));
    if (n_edits < 0 || n_edits > 3 * n) return cc_fail(c, CC_E_ARG, "n_edits");
    if (n == 0) return CC_OK;
    if (!xh0 || !yh0 || !zh0 || !flags || (n_edits > 0 && !q) || !xr || !yr || !zr)
        return cc_fail(c, CC_E_ARG, "null buffer");
    const double s = std::ldexp((double)(float)c->p.xi, 1 - c->p.m);
    unsigned long long* bsum = c->codec_bsum.p;
    const DecMask mk{flags};
    int tok = cc_prof_begin(c, "F1_decode");
    CCL(c, k_edit_count<<<(unsigned)nb, CT, 0, c->stream>>>(n, mk, bsum));
    CCL(c, k_edit_scan<<<1, 1024, 0, c->stream>>>(nb, bsum));
    const bool vec = aligned16(xh0) && aligned16(yh0) && aligned16(zh0) && aligned16(xr) && aligned16(yr) &&
                     aligned16(zr) && !getenv("CC_CODEC_SCALAR");
    if (vec)
        CCL(c, k_edit_apply4<<<(unsigned)nb, CT, 0, c->stream>>>(n, flags, bsum, s,
                                                                reinterpret_cast<const long long*>(q), n_edits, xh0,
                                                                yh0, zh0, xr, yr, zr));
    else
        CCL(c, k_edit_apply<<<(unsigned)nb, CT, 0, c->stream>>>(n, mk, bsum, s,
                                                               reinterpret_cast<const long long*>(q), n_edits, xh0,
                                                               yh0, zh0, xr, yr, zr));
    cc_prof_end(c, tok);
    CC_CUDA(c, cudaGetLastError());
    unsigned long long tot = 0;
    CC_CUDA(c, cudaMemcpyAsync(&tot, bsum + nb, sizeof(tot), cudaMemcpyDeviceToHost, c->stream));
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    if ((int64_t)tot != n_edits) return cc_fail(c, CC_E_DATA, "popcount(flags) != n_edits");
    return CC_OK;
}

cc_status cc_edit_pack(cc_ctx* c, const int64_t* q, int64_t n_edits, uint32_t* words, int64_t cap_words,
                       int64_t* n_words_h) {
    int64_t nb = 0;
    CC_TRY(edit_common(c, 0, &nb));
    if (n_edits < 0 || !n_words_h) return cc_fail(c, CC_E_ARG, "n_edits < 0 or null n_words_h");
    const int w = c->p.m + 2;
    const int64_t nw = (n_edits * w + 31) / 32;
    *n_words_h = nw;
    if (nw > cap_words) return cc_fail(c, CC_E_OOM, "cap_words < ceil(n_edits (m+2) / 32)");
    if (nw == 0) return CC_OK;
    if (!q || !words) return cc_fail(c, CC_E_ARG, "null buffer");
    CC_TRY(cc_ensure(c, c->codec_bsum, 2, "edit-log flags"));
    unsigned int* err = reinterpret_cast<unsigned int*>(c->codec_bsum.p);
    CC_CUDA(c, cudaMemsetAsync(err, 0, sizeof(unsigned int), c->stream));
    int tok = cc_prof_begin(c, "F1_pack");
    CCL(c, k_edit_pack<<<(unsigned)((nw + CT - 1) / CT), CT, 0, c->stream>>>(
               n_edits, w, 1ll << c->p.m, reinterpret_cast<const long long*>(q), words, nw, err));
    cc_prof_end(c, tok);
    CC_CUDA(c, cudaGetLastError());
    unsigned int e = 0;
    CC_CUDA(c, cudaMemcpyAsync(&e, err, sizeof(e), cudaMemcpyDeviceToHost, c->stream));
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    if (e) return cc_fail(c, CC_E_DATA, "an edit index exceeds |q| <= 2^m");
    return CC_OK;
}

cc_status cc_edit_unpack(cc_ctx* c, const uint32_t* words, int64_t n_edits, int64_t* q) {
    int64_t nb = 0;
    CC_TRY(edit_common(c, 0, &nb));
    if (n_edits < 0) return cc_fail(c, CC_E_ARG, "n_edits < 0");
    if (n_edits == 0) return CC_OK;
    if (!q || !words) return cc_fail(c, CC_E_ARG, "null buffer");
    const int w = c->p.m + 2;
    const int64_t nw = (n_edits * w + 31) / 32;
    int tok = cc_prof_begin(c, "F1_unpack");
    CCL(c, k_edit_unpack<<<(unsigned)((n_edits + CT - 1) / CT), CT, 0, c->stream>>>(n_edits, w, words, nw,
                                                                                   reinterpret_cast<long long*>(q)));
    cc_prof_end(c, tok);
    CC_CUDA(c, cudaGetLastError());
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    return CC_OK;
}
