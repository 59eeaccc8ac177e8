// bin.cu -- K1, cell binning (S1).  §III-C: "each thread maps one particle to its grid
// cell and atomically increments per-cell counts ...; a device-wide exclusive prefix sum then
// converts these counts into cell-start offsets, after which a scatter kernel places each
// particle into a cell-sorted array using atomic index reservations."
//
// B200 form (the x-sorted-row structure of cc_internal.cuh): a fused key + histogram kernel
// (coalesced SoA reads; the u32 atomic's return value is the particle's provisional rank in its
// cell; it also checks the input contract), the reduce-then-scan of scan.cu, a scatter of
// 8-byte (x-key, index) records, an in-cell sort of those records by x (cells hold ~1/K
// particles on average: thread-per-cell insertion sort, block bitonic for crowded cells), and
// a coalesced gather writing the float4 (x,y,z,gid) / (xh,yh,zh,i) records every later kernel
// reads.  The slot order is therefore fully determined by the data (x ties by input index).
#include <cmath>

#include "cc_internal.cuh"

namespace cc {
namespace {

constexpr int BIN_THREADS = 256;
constexpr int CELL_SHORT = 32;
constexpr int CELL_LONG_MAX = 4096;

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
    double u;
    int cx, cy, cz;
    cell_of(a, b, c, g, u, cx, cy, cz);
    const uint32_t k = (uint32_t)(((int64_t)cz * g.ny + cy) * g.nx + cx);
    key[i] = k;
    rnk[i] = atomicAdd(&count[k], 1u);
}

__global__ void __launch_bounds__(BIN_THREADS)
k_bin_scatter(int64_t n, const float* __restrict__ x, const uint32_t* __restrict__ key, const uint32_t* __restrict__ rnk,
              const uint32_t* __restrict__ cell_start, Grid g, unsigned long long* __restrict__ rec) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t s = cell_start[key[i]] + rnk[i];
    rec[s] = ((unsigned long long)x_sort_key(x[i], g) << 32) | (unsigned long long)(uint32_t)i;
}

// sort each cell's records: short cells in registers, crowded ones queued for a block
__global__ void __launch_bounds__(BIN_THREADS)
k_cell_sort_short(int64_t ncell, const uint32_t* __restrict__ cs, unsigned long long* __restrict__ rec,
                  uint32_t* __restrict__ long_list, unsigned long long* __restrict__ n_long) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncell) return;
    const uint32_t a = cs[c], b = cs[c + 1];
    const int len = (int)(b - a);
    if (len <= 1) return;
    if (len > CELL_SHORT) {
        const unsigned long long q = atomicAdd(n_long, 1ull);
        long_list[q] = (uint32_t)c;
        return;
    }
    unsigned long long v[CELL_SHORT];
    for (int i = 0; i < len; i++) {
        const unsigned long long xk = rec[a + i];
        int j = i - 1;
        while (j >= 0 && v[j] > xk) {
            v[j + 1] = v[j];
            j--;
        }
        v[j + 1] = xk;
    }
    for (int i = 0; i < len; i++) rec[a + i] = v[i];
}

__global__ void __launch_bounds__(512)
k_cell_sort_long(const uint32_t* __restrict__ long_list, const unsigned long long* __restrict__ n_long,
                 const uint32_t* __restrict__ cs, unsigned long long* __restrict__ rec) {
    __shared__ unsigned long long sh[CELL_LONG_MAX];
    const unsigned long long nl = *n_long;
    for (unsigned long long q = blockIdx.x; q < nl; q += gridDim.x) {
        const uint32_t c = long_list[q];
        const uint32_t a = cs[c], b = cs[c + 1];
        const int len = (int)(b - a);
        if (len <= CELL_LONG_MAX) {
            int p2 = 1;
            while (p2 < len) p2 <<= 1;
            for (int i = threadIdx.x; i < p2; i += blockDim.x) sh[i] = i < len ? rec[a + i] : ~0ull;
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
                            }
                        }
                    }
                    __syncthreads();
                }
            }
            for (int i = threadIdx.x; i < len; i += blockDim.x) rec[a + i] = sh[i];
            __syncthreads();
        } else if (threadIdx.x == 0) {  // pathological crowding: serial insertion sort (correct, slow)
            for (int i = 1; i < len; i++) {
                const unsigned long long xk = rec[a + i];
                int j = i - 1;
                while (j >= 0 && rec[a + j] > xk) {
                    rec[a + j + 1] = rec[a + j];
                    j--;
                }
                rec[a + j + 1] = xk;
            }
        }
    }
}

__global__ void __launch_bounds__(BIN_THREADS)
k_bin_gather(int64_t n, const float* __restrict__ x, const float* __restrict__ y, const float* __restrict__ z,
             const float* __restrict__ xh, const float* __restrict__ yh, const float* __restrict__ zh,
             const uint32_t* __restrict__ gid, const unsigned long long* __restrict__ rec, float4* __restrict__ orig4,
             float4* __restrict__ dec4, float* __restrict__ xs, uint32_t* __restrict__ slot_of) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const uint32_t i = (uint32_t)(rec[s] & 0xFFFFFFFFull);
    const float xi_ = x[i];
    const uint32_t gi = gid ? gid[i] : i;
    orig4[s] = make_float4(xi_, y[i], z[i], __uint_as_float(gi));
    dec4[s] = make_float4(xh[i], yh[i], zh[i], __uint_as_float(i));
    xs[s] = xi_;
    slot_of[i] = (uint32_t)s;
}

}  // namespace

cc_status bin_particles(cc_ctx* c, const float* x, const float* y, const float* z, const float* xh,
                        const float* yh, const float* zh, const uint32_t* gid, int64_t n) {
    const int64_t nc = c->ncell;
    const size_t n1 = (size_t)std::max<int64_t>(n, 1);
    CC_TRY(cc_ensure(c, c->key, n1, "key"));
    CC_TRY(cc_ensure(c, c->rnk, n1, "rank"));
    CC_TRY(cc_ensure(c, c->cell_count, (size_t)nc, "cell_count"));
    CC_TRY(cc_ensure(c, c->cell_start, (size_t)nc + 1, "cell_start"));
    CC_TRY(cc_ensure(c, c->orig4, n1, "orig4"));
    CC_TRY(cc_ensure(c, c->dec4, n1, "dec4"));
    CC_TRY(cc_ensure(c, c->xs, n1, "xs"));
    CC_TRY(cc_ensure(c, c->slot_of, n1, "slot_of"));
    CC_TRY(cc_ensure(c, c->rowoff, n1 + 1, "records"));  // reused: sort records now, row offsets later
    CC_TRY(cc_ensure(c, c->counters, 16, "counters"));
    CC_TRY(cc_ensure(c, c->scratch_u64, 2, "long count"));
    CC_CUDA(c, cudaMemsetAsync(c->cell_count.p, 0, (size_t)nc * sizeof(uint32_t), c->stream));
    CC_CUDA(c, cudaMemsetAsync(c->counters.p, 0, 16 * sizeof(unsigned long long), c->stream));
    CC_CUDA(c, cudaMemsetAsync(c->scratch_u64.p, 0, sizeof(uint64_t), c->stream));
    unsigned long long* rec = reinterpret_cast<unsigned long long*>(c->rowoff.p);
    const unsigned nb = (unsigned)((n + BIN_THREADS - 1) / BIN_THREADS);
    if (n > 0) {
        int tok = cc_prof_begin(c, "K1_key");
        CCL(c, k_bin_key<<<nb, BIN_THREADS, 0, c->stream>>>(n, x, y, z, xh, yh, zh, c->g, c->th.xi_f, c->key.p,
                                                             c->rnk.p, c->cell_count.p, c->counters.p));
        cc_prof_end(c, tok);
        CC_CUDA(c, cudaGetLastError());
    }
    // cell_start = exclusive scan of the counts; cell_start[nc] = n
    CC_TRY(scan_u32_to_u32(c, c->cell_count.p, c->cell_start.p, nc,
                           reinterpret_cast<uint64_t*>(c->cell_start.p + nc)));
    if (n > 0) {
        CC_TRY(cc_ensure(c, c->scratch_u32, (size_t)std::max<int64_t>(std::min<int64_t>(nc, n), 1), "crowded cells"));
        int tok = cc_prof_begin(c, "K1_scatter_sort");
        CCL(c, k_bin_scatter<<<nb, BIN_THREADS, 0, c->stream>>>(n, x, c->key.p, c->rnk.p, c->cell_start.p, c->g, rec));
        unsigned long long* nl = reinterpret_cast<unsigned long long*>(c->scratch_u64.p);
        CCL(c, k_cell_sort_short<<<(unsigned)((nc + BIN_THREADS - 1) / BIN_THREADS), BIN_THREADS, 0, c->stream>>>(
                   nc, c->cell_start.p, rec, c->scratch_u32.p, nl));
        CCL(c, k_cell_sort_long<<<148 * 2, 512, 0, c->stream>>>(c->scratch_u32.p, nl, c->cell_start.p, rec));
        cc_prof_end(c, tok);
        int t2 = cc_prof_begin(c, "K1_gather");
        CCL(c, k_bin_gather<<<nb, BIN_THREADS, 0, c->stream>>>(n, x, y, z, xh, yh, zh, gid, rec, c->orig4.p, c->dec4.p,
                                                                c->xs.p, c->slot_of.p));
        cc_prof_end(c, t2);
        CC_CUDA(c, cudaGetLastError());
    }
    return CC_OK;
}

}  // namespace cc
