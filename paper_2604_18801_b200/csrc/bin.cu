// bin.cu -- K1, cell binning (S1).  §III-C: "each thread maps one particle to its grid
// cell and atomically increments per-cell counts ...; a device-wide exclusive prefix sum then
// converts these counts into cell-start offsets, after which a scatter kernel places each
// particle into a cell-sorted array using atomic index reservations."
//
// B200 form: one fused key+histogram kernel (coalesced SoA reads, one u32 atomic per particle
// whose return value is the particle's rank inside its cell), the reduce-then-scan of
// scan.cu, and one scatter kernel writing float4 (x,y,z,gid) / (xh,yh,zh,i) records so every
// later kernel reads one 16-byte vector per particle.  In-cell order is the atomic order: no
// result depends on it (rows are re-sorted by gid, FoF labels are min-gid canonical).
// Algorithmic bytes: read 24 B + write 8 B (key, rank) + atomics; scatter: read 24+8+4 B,
// write 32 B + slot_of 4 B; plus the scan over the cell counts.
#include <cmath>

#include "cc_internal.cuh"

namespace cc {
namespace {

constexpr int BIN_THREADS = 256;

__global__ void __launch_bounds__(BIN_THREADS)
k_bin_key(int64_t n, const float* __restrict__ x, const float* __restrict__ y, const float* __restrict__ z,
          const float* __restrict__ xh, const float* __restrict__ yh, const float* __restrict__ zh, Grid g,
          float xi_f, uint32_t* __restrict__ key, uint32_t* __restrict__ rnk, uint32_t* __restrict__ count,
          unsigned long long* __restrict__ errs) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float a = x[i], b = y[i], c = z[i], ah = xh[i], bh = yh[i], ch = zh[i];
    unsigned int bad = 0;
    if (!(isfinite(a) && isfinite(b) && isfinite(c) && isfinite(ah) && isfinite(bh) && isfinite(ch))) bad |= 1u;
    // input contract |x_hat - x| <= xi_f per coordinate, exact in fp64
    const double e = (double)xi_f;
    if (!(fabs((double)ah - (double)a) <= e && fabs((double)bh - (double)b) <= e && fabs((double)ch - (double)c) <= e))
        bad |= 2u;
    if (bad) atomicOr(errs, (unsigned long long)bad);
    int cx, cy, cz;
    cell_of(a, b, c, g, cx, cy, cz);
    const uint32_t k = (uint32_t)(((int64_t)cz * g.ny + cy) * g.nx + cx);
    key[i] = k;
    rnk[i] = atomicAdd(&count[k], 1u);
}

__global__ void __launch_bounds__(BIN_THREADS)
k_bin_scatter(int64_t n, const float* __restrict__ x, const float* __restrict__ y, const float* __restrict__ z,
              const float* __restrict__ xh, const float* __restrict__ yh, const float* __restrict__ zh,
              const uint32_t* __restrict__ gid, const uint32_t* __restrict__ key, const uint32_t* __restrict__ rnk,
              const uint32_t* __restrict__ cell_start, float4* __restrict__ orig4, float4* __restrict__ dec4,
              uint32_t* __restrict__ slot_of) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t s = cell_start[key[i]] + rnk[i];
    const uint32_t gi = gid ? gid[i] : (uint32_t)i;
    orig4[s] = make_float4(x[i], y[i], z[i], __uint_as_float(gi));
    dec4[s] = make_float4(xh[i], yh[i], zh[i], __uint_as_float((uint32_t)i));
    slot_of[i] = s;
}

}  // namespace

cc_status bin_particles(cc_ctx* c, const float* x, const float* y, const float* z, const float* xh,
                        const float* yh, const float* zh, const uint32_t* gid, int64_t n) {
    const int64_t nc = c->ncell;
    CC_TRY(cc_ensure(c, c->key, (size_t)std::max<int64_t>(n, 1), "key"));
    CC_TRY(cc_ensure(c, c->rnk, (size_t)std::max<int64_t>(n, 1), "rank"));
    CC_TRY(cc_ensure(c, c->cell_count, (size_t)nc, "cell_count"));
    CC_TRY(cc_ensure(c, c->cell_start, (size_t)nc + 1, "cell_start"));
    CC_TRY(cc_ensure(c, c->orig4, (size_t)std::max<int64_t>(n, 1), "orig4"));
    CC_TRY(cc_ensure(c, c->dec4, (size_t)std::max<int64_t>(n, 1), "dec4"));
    CC_TRY(cc_ensure(c, c->slot_of, (size_t)std::max<int64_t>(n, 1), "slot_of"));
    CC_TRY(cc_ensure(c, c->counters, 16, "counters"));
    CC_CUDA(c, cudaMemsetAsync(c->cell_count.p, 0, (size_t)nc * sizeof(uint32_t), c->stream));
    CC_CUDA(c, cudaMemsetAsync(c->counters.p, 0, 16 * sizeof(unsigned long long), c->stream));
    if (n > 0) {
        const unsigned nb = (unsigned)((n + BIN_THREADS - 1) / BIN_THREADS);
        int tok = cc_prof_begin(c, "K1_key");
        CCL(c, k_bin_key<<<nb, BIN_THREADS, 0, c->stream>>>(n, x, y, z, xh, yh, zh, c->g, c->th.xi_f, c->key.p, c->rnk.p,
                                                     c->cell_count.p, c->counters.p));
        cc_prof_end(c, tok);
        CC_CUDA(c, cudaGetLastError());
    }
    // cell_start = exclusive scan of the counts; cell_start[nc] = n
    CC_TRY(scan_u32_to_u32(c, c->cell_count.p, c->cell_start.p, nc,
                           reinterpret_cast<uint64_t*>(c->cell_start.p + nc)));
    if (n > 0) {
        const unsigned nb = (unsigned)((n + BIN_THREADS - 1) / BIN_THREADS);
        int tok = cc_prof_begin(c, "K1_scatter");
        CCL(c, k_bin_scatter<<<nb, BIN_THREADS, 0, c->stream>>>(n, x, y, z, xh, yh, zh, gid, c->key.p, c->rnk.p,
                                                         c->cell_start.p, c->orig4.p, c->dec4.p, c->slot_of.p));
        cc_prof_end(c, tok);
        CC_CUDA(c, cudaGetLastError());
    }
    return CC_OK;
}

}  // namespace cc
