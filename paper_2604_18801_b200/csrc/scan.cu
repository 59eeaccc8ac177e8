// scan.cu -- device-wide exclusive prefix sums (reduce-then-scan, 3 launches) used by S1
// (cell histogram -> cell_start, §III-C P:461 "device-wide exclusive prefix sum") and S3
// (degrees -> CSR row offsets and editable ranks, the paper's direct-address map P:463).
#include "cc_internal.cuh"

namespace cc {
namespace {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

struct VU32 {
    uint32_t a;
    __device__ static VU32 zero() { return {0u}; }
    __device__ VU32 operator+(const VU32& o) const { return {a + o.a}; }
    __device__ VU32 shfl_up(int d) const { return {__shfl_up_sync(0xffffffffu, a, d)}; }
};

// degree scan value, per row-length class k (K3 work classes, cc_internal.cuh row_class):
// a[k] = row entries, b[k] = editable rank; g = ghost editable rank
struct VDeg {
    unsigned long long a[4];
    uint32_t b[4];
    uint32_t g, pad;
    __device__ static VDeg zero() {
        VDeg v;
        for (int k = 0; k < 4; k++) {
            v.a[k] = 0ull;
            v.b[k] = 0u;
        }
        v.g = 0u;
        v.pad = 0u;
        return v;
    }
    __device__ VDeg operator+(const VDeg& o) const {
        VDeg v;
        for (int k = 0; k < 4; k++) {
            v.a[k] = a[k] + o.a[k];
            v.b[k] = b[k] + o.b[k];
        }
        v.g = g + o.g;
        v.pad = 0u;
        return v;
    }
    __device__ VDeg shfl_up(int d) const {
        VDeg v;
        for (int k = 0; k < 4; k++) {
            v.a[k] = __shfl_up_sync(0xffffffffu, a[k], d);
            v.b[k] = __shfl_up_sync(0xffffffffu, b[k], d);
        }
        v.g = __shfl_up_sync(0xffffffffu, g, d);
        v.pad = 0u;
        return v;
    }
};

struct LoadU32 {
    const uint32_t* in;
    __device__ VU32 operator()(int64_t i) const { return {in[i]}; }
};
struct StoreU32 {
    uint32_t* out;
    __device__ void operator()(int64_t i, const VU32& v, const VU32&) const { out[i] = v.a; }
};

// deg[s] > 0 -> owned editable; deg == 0 but marked (ghost partner, dec4.w index >= n_own
// and flagged with bit 31 of deg) -> ghost editable.  The scan runs over the editable list
// (k_editable_list: the slots with deg != 0, in slot order), not over all n slots.
__device__ __forceinline__ VDeg deg_value(uint32_t d) {
    const uint32_t len = d & 0x7FFFFFFFu;
    VDeg v = VDeg::zero();
    if (len > 0u) {
        const int k = row_class(len);
        v.a[k] = len;
        v.b[k] = 1u;
    } else {
        v.g = d >> 31;
    }
    return v;
}
struct LoadCand {
    const uint32_t* deg;
    const uint32_t* cand;
    __device__ VDeg operator()(int64_t i) const { return deg_value(deg[cand[i]]); }
};
// the editable index e of slot s = its class base + its rank in the class (classes 0..3 by row
// length, then the ghosts): eidx[s] = e, and the compact per-editable arrays (slot, row offset,
// original position, PGD start = decompressed position) are written at e.  The class bases come
// from the scan total (written by k_scan_blocks before this pass).
struct StoreEdit {
    const uint32_t* cand;
    const VDeg* total;
    const float4* orig4;
    const float4* dec4;
    uint32_t* eidx;
    uint32_t* slotE;
    unsigned long long* rowptr;
    float4* origE;
    float4* posA;
    __device__ void operator()(int64_t i, const VDeg& excl, const VDeg& self) const {
        const VDeg t = *total;
        const uint32_t s = cand[i];
        uint32_t e;
        unsigned long long o;
        uint32_t eb = 0u;
        unsigned long long ob = 0ull;
        e = 0u;
        o = 0ull;
        bool own = false;
#pragma unroll
        for (int q = 0; q < 4; q++) {
            if (self.b[q]) {
                e = eb + excl.b[q];
                o = ob + excl.a[q];
                own = true;
            }
            eb += t.b[q];
            ob += t.a[q];
        }
        if (!own) {  // ghost editable: after every owned one; its row is empty
            e = eb + excl.g;
            o = ob;
        }
        const float4 p = orig4[s], d = dec4[s];
        eidx[s] = e;
        slotE[e] = s;
        rowptr[e] = o;
        origE[e] = p;
        posA[e] = make_float4(d.x, d.y, d.z, p.w);
    }
};

// the editable list: cand[0..E_all) = the slots with deg != 0 in ascending order, eidx[s] =
// 0xFFFFFFFF for every slot (the editables' entries are overwritten by the list scan).  Single
// pass, decoupled look-back; a thread owns LI consecutive slots (16-byte loads and stores).
constexpr int LT = 256, LI = 16, LTILE = LT * LI;

__global__ void __launch_bounds__(LT) k_editable_list(int64_t n, const uint32_t* __restrict__ deg,
                                                     uint32_t* __restrict__ eidx, uint32_t* __restrict__ cand,
                                                     unsigned long long* __restrict__ status,
                                                     unsigned int* __restrict__ ticket,
                                                     unsigned long long* __restrict__ total) {
    __shared__ unsigned int tile_sh;
    __shared__ unsigned long long base_sh;
    __shared__ uint32_t wsum[LT / 32];
    if (threadIdx.x == 0) tile_sh = atomicAdd(ticket, 1u);
    __syncthreads();
    const unsigned int tile = tile_sh;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t i0 = (int64_t)tile * LTILE + (int64_t)threadIdx.x * LI;
    uint32_t mask = 0u;
    if (i0 + LI <= n) {
        const uint4* d4 = reinterpret_cast<const uint4*>(deg + i0);
        uint4* e4 = reinterpret_cast<uint4*>(eidx + i0);
#pragma unroll
        for (int k = 0; k < LI / 4; k++) {
            const uint4 v = d4[k];
            mask |= (v.x != 0u ? 1u : 0u) << (4 * k) | (v.y != 0u ? 2u : 0u) << (4 * k) |
                    (v.z != 0u ? 4u : 0u) << (4 * k) | (v.w != 0u ? 8u : 0u) << (4 * k);
            e4[k] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
        }
    } else {
        for (int k = 0; k < LI; k++)
            if (i0 + k < n) {
                mask |= (deg[i0 + k] != 0u ? 1u : 0u) << k;
                eidx[i0 + k] = 0xFFFFFFFFu;
            }
    }
    // block-exclusive prefix of the per-thread counts (slot order = thread order)
    const uint32_t cnt = __popc(mask);
    uint32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    uint32_t wex = 0u, tot = 0u;
#pragma unroll
    for (int k = 0; k < LT / 32; k++) {
        wex += k < w ? wsum[k] : 0u;
        tot += wsum[k];
    }
    if (threadIdx.x < 32) {
        const unsigned long long ex = lookback_warp0(status, tile, tot);
        if (lane == 0) {
            base_sh = ex;
            if ((int64_t)(tile + 1) * LTILE >= n) *total = ex + tot;  // the last tile
        }
    }
    __syncthreads();
    unsigned long long q = base_sh + wex + inc - cnt;
    while (mask) {
        const int k = __ffs(mask) - 1;
        mask &= mask - 1u;
        cand[q++] = (uint32_t)(i0 + k);
    }
}

// inclusive warp scan then block exclusive scan; returns exclusive prefix, *total = sum
template <class V>
__device__ V block_exclusive(V v, V* total) {
    __shared__ V sh[SCAN_THREADS / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    V inc = v;
    for (int o = 1; o < 32; o <<= 1) {
        V u = inc.shfl_up(o);
        if (lane >= o) inc = inc + u;
    }
    if (lane == 31) sh[w] = inc;
    __syncthreads();
    if (w == 0) {
        V s = lane < SCAN_THREADS / 32 ? sh[lane] : V::zero();
        V si = s;
        for (int o = 1; o < 32; o <<= 1) {
            V u = si.shfl_up(o);
            if (lane >= o) si = si + u;
        }
        if (lane < SCAN_THREADS / 32) sh[lane] = si;  // inclusive warp totals
    }
    __syncthreads();
    V wex = (w == 0) ? V::zero() : sh[w - 1];
    *total = sh[SCAN_THREADS / 32 - 1];
    V ex = inc.shfl_up(1);
    if (lane == 0) ex = V::zero();
    __syncthreads();
    return wex + ex;
}

template <class V, class Load>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_reduce(int64_t n, Load load, V* bsum) {
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    V s = V::zero();
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++)
        if (base + k < n) s = s + load(base + k);
    V tot;
    (void)block_exclusive(s, &tot);
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// one block scans the tile sums in place, SCAN_ITEMS consecutive sums per thread per step (C4:
// 137K tiles in 67 steps instead of 537)
template <class V>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_blocks(int64_t nb, V* bsum, V* total) {
    V carry = V::zero();
    for (int64_t off = 0; off < nb; off += SCAN_TILE) {
        const int64_t i0 = off + (int64_t)threadIdx.x * SCAN_ITEMS;
        V v = V::zero();
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; k++)
            if (i0 + k < nb) v = v + bsum[i0 + k];
        V tot;
        V run = carry + block_exclusive(v, &tot);
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; k++)
            if (i0 + k < nb) {
                const V x = bsum[i0 + k];
                bsum[i0 + k] = run;
                run = run + x;
            }
        carry = carry + tot;
        __syncthreads();
    }
    if (threadIdx.x == 0 && total) *total = carry;
}

template <class V, class Load, class Store>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_down(int64_t n, Load load, Store store, const V* bsum) {
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    // items are re-loaded for the store pass (L1 hits) rather than held: a held array of the
    // 56-byte VDeg values cost ~112 registers per thread and spilled
    V s = V::zero();
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++)
        if (base + k < n) s = s + load(base + k);
    V tot;
    V run = bsum[blockIdx.x] + block_exclusive(s, &tot);
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) {
        if (base + k < n) {
            const V it = load(base + k);
            store(base + k, run, it);
            run = run + it;
        }
    }
}

template <class V, class Load, class Store>
cc_status scan_generic(cc_ctx* c, int64_t n, Load load, Store store, V* total_dev, const char* name) {
    if (n <= 0) {
        if (total_dev) CC_CUDA(c, cudaMemsetAsync(total_dev, 0, sizeof(V), c->stream));
        return CC_OK;
    }
    const int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
    CC_TRY(cc_ensure(c, c->tmp_bytes, (size_t)nb * sizeof(V) + 256, "scan scratch"));
    V* bsum = reinterpret_cast<V*>(c->tmp_bytes.p);
    int tok = cc_prof_begin(c, name);
    CCL(c, k_scan_reduce<V, Load><<<(unsigned)nb, SCAN_THREADS, 0, c->stream>>>(n, load, bsum));
    CCL(c, k_scan_blocks<V><<<1, SCAN_THREADS, 0, c->stream>>>(nb, bsum, total_dev));
    CCL(c, k_scan_down<V, Load, Store><<<(unsigned)nb, SCAN_THREADS, 0, c->stream>>>(n, load, store, bsum));
    cc_prof_end(c, tok);
    CC_CUDA(c, cudaGetLastError());
    return CC_OK;
}

}  // namespace

cc_status scan_u32_to_u32(cc_ctx* c, const uint32_t* in, uint32_t* out, int64_t n, uint64_t* total_dev) {
    static_assert(sizeof(VU32) == 4, "");
    // total written as u32 into the low half of *total_dev (caller zeroes it)
    return scan_generic<VU32>(c, n, LoadU32{in}, StoreU32{out}, reinterpret_cast<VU32*>(total_dev), "K1_scan");
}

cc_status editable_list(cc_ctx* c, int64_t* e_all) {
    const int64_t n = c->n;
    *e_all = 0;
    if (n <= 0) return CC_OK;
    const int64_t nt = (n + LTILE - 1) / LTILE;
    CC_TRY(cc_ensure(c, c->codec_status, (size_t)nt + 2, "look-back status"));
    unsigned long long* st = c->codec_status.p;
    unsigned int* ticket = reinterpret_cast<unsigned int*>(st + nt);
    unsigned long long* tot = c->counters.p + 9;
    CC_CUDA(c, cudaMemsetAsync(st, 0, (size_t)(nt + 1) * sizeof(unsigned long long), c->stream));
    int tok = cc_prof_begin(c, "K2_scan");
    CCL(c, k_editable_list<<<(unsigned)nt, LT, 0, c->stream>>>(n, c->deg.p, c->eidx.p, c->key.p, st, ticket, tot));
    cc_prof_end(c, tok);
    CC_CUDA(c, cudaGetLastError());
    CC_CUDA(c, cudaMemcpyAsync(c->h_counters + 9, tot, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                               c->stream));
    CC_CUDA(c, cudaStreamSynchronize(c->stream));
    *e_all = (int64_t)c->h_counters[9];
    return CC_OK;
}

cc_status scan_editables(cc_ctx* c, int64_t e_all, unsigned long long* totals_dev) {
    static_assert(sizeof(VDeg) == 56, "");
    VDeg* tot = reinterpret_cast<VDeg*>(totals_dev);
    unsigned long long* rowptr = reinterpret_cast<unsigned long long*>(c->rowptr.p);
    return scan_generic<VDeg>(c, e_all, LoadCand{c->deg.p, c->key.p},
                              StoreEdit{c->key.p, tot, c->orig4.p, c->dec4.p, c->eidx.p, c->slotE.p, rowptr,
                                        c->origE.p, c->posA.p},
                              tot, "K2_scan");
}

}  // namespace cc
