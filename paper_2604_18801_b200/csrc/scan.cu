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
    __device__ VU32 shfl(int src) const { return {__shfl_sync(0xffffffffu, a, src)}; }
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
// and flagged with bit 31 of deg) -> ghost editable.
struct LoadDeg {
    const uint32_t* deg;
    __device__ VDeg operator()(int64_t i) const {
        const uint32_t d = deg[i];
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
};
// provisional (class, rank-in-class, row offset in class); rows_resolve adds the class bases
struct StoreDeg {
    unsigned long long* rowoff;
    uint32_t* eidx;
    uint32_t* cls;
    __device__ void operator()(int64_t i, const VDeg& excl, const VDeg& self) const {
        uint32_t k = 0xFFu, r = 0xFFFFFFFFu;
        unsigned long long o = 0ull;
        for (int q = 0; q < 4; q++)
            if (self.b[q]) {
                k = (uint32_t)q;
                r = excl.b[q];
                o = excl.a[q];
            }
        if (self.g) {
            k = 4u;
            r = excl.g;
        }
        cls[i] = k;
        eidx[i] = r;
        rowoff[i] = o;
    }
};

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

cc_status scan_deg(cc_ctx* c, const uint32_t* deg, uint64_t* rowoff, uint32_t* eidx, uint32_t* cls, int64_t n,
                   unsigned long long* totals_dev) {
    static_assert(sizeof(VDeg) == 56, "");
    return scan_generic<VDeg>(c, n, LoadDeg{deg},
                              StoreDeg{reinterpret_cast<unsigned long long*>(rowoff), eidx, cls},
                              reinterpret_cast<VDeg*>(totals_dev), "K2_scan");
}

}  // namespace cc
