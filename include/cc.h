/*
 * cc.h -- C ABI of libcc, the B200-native (sm_100a) hot path of arXiv 2604.18801,
 * "Preserving Clusters in Error-Bounded Lossy Compression of Particle Data":
 * the post-decompression friends-of-friends (FoF) connectivity correction.
 *
 * Citations: "P:n" = PAPER.md line n (one paragraph per line) with the section / equation /
 * algorithm it falls in; "R<k>" = reading k of DESIGN.md §3 where the paper is silent.
 *
 * Conventions for every entry point
 *  - All array pointers are DEVICE pointers (CUDA global memory of the context's device)
 *    unless the parameter name ends in `_h` (host memory).  Exception: cc_run() takes host or
 *    device pointers as its `flags` say.
 *  - Particle arrays are structure-of-arrays float32 of length n, index i = input order.
 *  - All work is enqueued on the stream given to cc_create(); functions with `_h` outputs
 *    synchronise that stream before returning, and so do the steps whose status depends on
 *    device results (cc_build_cells, cc_find_vulnerable, cc_correct, as each states).
 *  - The caller owns every input/output buffer; the library owns its scratch (allocated with
 *    stream-ordered cudaMallocAsync on the context's stream, freed by cc_destroy()).  Inputs
 *    are never written; cc_build_cells() snapshots them into cell-sorted copies, and
 *    cc_correct() reads the decompressed inputs xh,yh,zh of the last cc_build_cells() once more
 *    (they are the output of every non-editable particle): keep those three arrays valid and
 *    unchanged until cc_correct() has returned (cc_run() does this itself).
 *  - Every function returns a cc_status; no exception, abort or exit crosses the ABI.  On a
 *    non-OK status cc_last_error() describes it.  Calling steps out of order returns
 *    CC_E_STATE.  A CUDA failure returns CC_E_CUDA and leaves the context unusable.
 *  - There is NO CPU fallback: without a CUDA device cc_create() returns CC_E_CUDA.
 */
#ifndef CC_H
#define CC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cc_ctx cc_ctx;

typedef enum {
    CC_OK = 0,
    CC_NOT_CONVERGED = 2,  /* T_max reached with active pairs left; outputs valid, in bound   */
    CC_E_ARG = 64,         /* invalid argument (usage)                                        */
    CC_E_DATA = 65,        /* invalid data (NaN/Inf, sizes beyond the 2^30 index space)       */
    CC_E_BOUND = 66,       /* decompressed input violates |x_hat - x| <= xi_f         */
    CC_E_OOM = 67,         /* device allocation failed                                        */
    CC_E_CUDA = 68,        /* CUDA runtime error (or no device)                               */
    CC_E_NCCL = 69,        /* NCCL error                                                      */
    CC_E_STATE = 70        /* step called out of order                                        */
} cc_status;

enum { CC_STOP_ACTIVE = 0,  /* stop when no pair is L_tight-active (R11; default)             */
       CC_STOP_EPS = 1,     /* stop when L_tight <= eps_loss (Alg. 1 line 6)           */
       CC_STOP_NONE = 2,    /* run exactly t_max updates (truncated mode)        */
       CC_STOP_RESTORED = 3 }; /* L_tight <= eps_loss AND every vulnerable pair's link status
                                  restored (MCC = 1; Alg. 1 l.6 + north_star's stop)          */
enum { CC_OPT_ADAM = 0, CC_OPT_VANILLA = 1 };
enum { CC_ORIG = 0, CC_DECOMP = 1, CC_CORR = 2 };  /* which positions cc_fof_label/cc_mcc use */

/* Alg. 1 REQUIRE line plus the periodic box. */
typedef struct {
    double box;            /* cubic box side L > 0; particles' original coords in [0, L)      */
    int periodic;          /* 1: minimum-image distances; 0: open box               */
    double b;              /* linking length; if <= 0: eta * (L^3/N)^(1/3)        */
    double eta;            /* linking parameter when b <= 0 (0.2)                      */
    double xi;             /* absolute per-coordinate bound; rounded to fp32 xi_f (R6)       */
    int m;                 /* edit bit depth, 2..52 (16)                              */
    double alpha, beta1, beta2, eps_adam; /* Adam (1e-3, .9, .999, 1e-8)         */
    int t_max;             /* iteration cap T_max >= 0                                       */
    double eps_loss;       /* epsilon_L for CC_STOP_EPS (1e-10)                        */
    int stop_mode;         /* CC_STOP_*                                                      */
    int optimizer;         /* CC_OPT_*                                                       */
    double vanilla_step;   /* step of CC_OPT_VANILLA                                         */
    int graph_batch;       /* PGD iterations per CUDA-graph launch (perf only; 0 = default)  */
    double cells_per_particle; /* grid budget K: at most K*N cells (perf only; 0 = default)  */
    int profile;           /* 1: time each kernel class with CUDA events (cc_kernel_stats)   */
    int frontier;          /* 1: skip particles whose state provably cannot change (exact;   */
                           /*    perf only, results identical; 0 = sweep every editable)    */
    /* Optional scratch allocator (e.g. torch's caching allocator): alloc_fn(bytes, user) returns
     * device memory usable on the context's stream (NULL = failure, CC_E_OOM); free_fn(ptr,
     * user) releases it, stream-ordered after the work already enqueued.  NULL = cudaMallocAsync
     * / cudaFreeAsync on the context's stream.  Called only from the thread making the cc_* call. */
    void* (*alloc_fn)(size_t bytes, void* user);
    void (*free_fn)(void* ptr, void* user);
    void* alloc_user;
} cc_params;

/* fill *p with the paper's defaults (eta 0.2, m 16, Adam 1e-3/.9/.999/1e-8, t_max 10000,
 * eps_loss 1e-10, CC_STOP_ACTIVE, periodic); box and xi must still be set. */
void cc_default_params(cc_params* p);

/* Multi-GPU (§III-D): x-slab decomposition, rank r owns original x in
 * [r L/R, (r+1) L/R).  nccl_id = 128-byte ncclUniqueId identical on all ranks (from
 * cc_nccl_unique_id() on rank 0, broadcast by the caller).  dist == NULL means one GPU.
 * vgroup != NULL (from cc_vgroup_create): the R ranks are contexts of ONE process on one GPU,
 * each driven by its own host thread; collectives become device copies and reduction kernels
 * ordered by events (comm.cu) -- a correctness mode that runs the multi-rank protocol on a
 * single GPU (results bit-identical to NCCL ranks and to one rank); nccl_id_h is then unused. */
typedef struct {
    int rank, nranks;
    const void* nccl_id_h;
    void* vgroup;
} cc_dist;

cc_status cc_nccl_unique_id(void* id_h /* 128 bytes */);

/* An in-process group of nranks (1..8) virtual ranks (see cc_dist.vgroup).  Destroy it after
 * every context of the group was destroyed.  Every rank of the group must make the same
 * sequence of calls (each collective blocks until all ranks reach it). */
cc_status cc_vgroup_create(int nranks, void** group_h);
void cc_vgroup_destroy(void* group);

/* Create a context on `device` enqueuing on `stream` (a cudaStream_t; NULL = legacy
 * default stream).  *ctx is NULL on failure. */
cc_status cc_create(cc_ctx** ctx, int device, void* stream, const cc_params* p, const cc_dist* dist);
void cc_destroy(cc_ctx* ctx);
const char* cc_last_error(const cc_ctx* ctx);

/* S1 -- cell binning (§III-C): counting sort of the n particles by the cell of their
 * ORIGINAL position (grid of side >= b + 2 sqrt3 xi), producing the cell-sorted copies
 * of original and decompressed positions.  x,y,z = original P, xh,yh,zh = decompressed
 * P_hat^(0); gid = global particle ids (NULL: gid = i).  Multi-GPU: the n owned
 * particles of this rank (original x inside its slab); ghost shells of width
 * b + 2 sqrt3 xi are exchanged here with NCCL.  Checks |x_hat - x| <= xi_f
 * (CC_E_BOUND) and finite inputs (CC_E_DATA).  Synchronises (the contract check is returned as
 * the status).  May be called again to start over. */
cc_status cc_build_cells(cc_ctx* ctx, int64_t n, const float* x, const float* y, const float* z,
                         const float* xh, const float* yh, const float* zh, const uint32_t* gid);

/* S2+S3 -- vulnerable pairs (§III-A; Alg. 1 line 3 P:421): every pair with
 * b - 2 sqrt3 xi < d <= b + 2 sqrt3 xi on the original positions (fp32 pinned expression R4,
 * half-open band R2), each with its original and decompressed link status (d <= b, R3), and
 * the editable set E = endpoints.  Synchronises (sizes the row buffers). */
typedef struct {
    int64_t n_pairs;        /* |V| (pairs owned by this rank, R17)                           */
    int64_t n_editable;     /* |E| (owned)                                                   */
    int64_t n_linked;       /* pairs linked in the original                                  */
    int64_t n_violated0;    /* pairs whose link status differs in the decompressed data      */
    int64_t n_local;        /* particles on this GPU, owned + ghost                          */
    int64_t cells_per_axis; /* grid used                                                     */
    double b;               /* linking length used                                           */
} cc_vp_info;
cc_status cc_find_vulnerable(cc_ctx* ctx, cc_vp_info* info_h);

/* The canonical pair list (gi < gj, global ids) with flags bit0 = original link,
 * bit1 = decompressed link, sorted by (gi, gj) (a counting sort on gi: scratch of 8 B per
 * gid up to the largest owner gid); at most `cap` written, *n_out_h = |V| (cap = 0: count only).
 * Multi-GPU: this rank's owned pairs (R17), sorted. */
cc_status cc_get_pairs(cc_ctx* ctx, uint32_t* gi, uint32_t* gj, uint8_t* flags, int64_t cap,
                       int64_t* n_out_h);

/* S4+S5 -- Alg. 1 lines 4-10: projected gradient descent (Adam) on L_tight
 * (Eq. 3) over the editable particles, box projection onto B(xi') around the
 * ORIGINAL positions, stop per params.stop_mode checked before every update.
 * Writes all n corrected coordinates in input order to xo,yo,zo (non-editable particles =
 * decompressed input, bit-exact, copied from the xh,yh,zh of the last cc_build_cells(), which
 * must still be valid; xo,yo,zo may alias them).  Returns CC_NOT_CONVERGED if T_max ended the loop with
 * active pairs left (outputs still valid and within xi').  Synchronises. */
typedef struct {
    int64_t iterations;     /* updates performed (R27)                                       */
    int64_t active0;        /* L_tight-active pairs at P_hat^(0)                             */
    int64_t active_final;   /* L_tight-active pairs at the returned positions                */
    double loss0, loss_final; /* L_tight (fp64 sums of fp32 terms; reporting only, R16)       */
    int converged;            /* the stop rule holds at the returned positions                */
    int pad;
    int64_t violated0;        /* pairs whose link status differs from the original (Eq. 1)    */
    int64_t violated_final;
} cc_corr_info;
cc_status cc_correct(cc_ctx* ctx, float* xo, float* yo, float* zo, cc_corr_info* info_h);

/* L_tight-active count, L_tight and violated-pair count per stop check of the last cc_correct
 * (the L_tight-vs-iteration trace of Fig. 6); up to cap entries each (violated_h may
 * be NULL), *n_h = iterations + 1 (the last entry is the returned state). */
cc_status cc_get_trace(cc_ctx* ctx, int64_t* active_h, double* loss_h, int64_t* violated_h, int64_t cap,
                       int64_t* n_h);

/* K3 schedule per iteration of the last cc_correct (diagnostics of the frontier):
 * sched_h[6 t + 0] = editables processed, [6 t + 1] = editables left awake, [6 t + 2] = row
 * entries of editables that moved, [6 t + 3] = zero-gradient steps replayed in full, [6 t + 4] =
 * zero-gradient steps replayed on the proven-still path, [6 t + 5] = device %globaltimer (ns)
 * when the iteration's statistics were final; up to cap iterations (cap rows of 6), *n_h =
 * iterations recorded. */
cc_status cc_get_schedule(cc_ctx* ctx, int64_t* sched_h, int64_t cap, int64_t* n_h);

/* S6 -- FoF labels (§II-B, Fig. 1) on ORIG, DECOMP or CORR positions: edge iff the
 * pinned fp32 d2 <= fl32(b^2); label = minimum gid of the connected component (R20).
 * labels: n entries in input order (owned particles).  *n_groups_h = number of components
 * (global).  CORR requires cc_correct() first. */
cc_status cc_fof_label(cc_ctx* ctx, int which, uint32_t* labels, int64_t* n_groups_h);

/* S7 -- MCC over the vulnerable pairs (§IV-A): TP/TN/FP/FN of original link vs link
 * in DECOMP or CORR positions; MCC with R21's degenerate-denominator convention. */
typedef struct {
    uint64_t tp, tn, fp, fn;
    double mcc;
} cc_mcc_info;
cc_status cc_mcc(cc_ctx* ctx, int which, cc_mcc_info* out_h);

/* S7 -- halo catalogue (threshold 20): sizes of the FoF groups of the last
 * cc_fof_label(which) with >= min_size members, descending; *n_halos_h = count (<= cap
 * written). */
cc_status cc_halo_sizes(cc_ctx* ctx, int which, int64_t min_size, int64_t* sizes_h, int64_t cap,
                        int64_t* n_halos_h);

/* HMF dn/dlog10M (§II-B-2): sizes (host) binned in n_bins equal log10 bins over
 * [lo, hi] (lo >= hi: the catalogue's own [min, max], R22), counts / (vol * width).
 * edges_h: n_bins+1, density_h: n_bins.  Pure host arithmetic. */
cc_status cc_hmf(const int64_t* sizes_h, int64_t n, double vol, int n_bins, double lo, double hi,
                 double* edges_h, double* density_h);

/* Per-kernel-class device time of everything enqueued since the last call (params.profile):
 * names_h receives a '\n'-separated list; ms_h[k], launches_h[k] per class (<= cap). */
cc_status cc_kernel_stats(cc_ctx* ctx, char* names_h, int64_t names_cap, double* ms_h,
                          int64_t* launches_h, int64_t cap, int64_t* n_h, int reset);

/* End-to-end convenience (the call a user makes): S1..S5 then writes corrected coordinates.
 * flags & CC_RUN_HOST: inputs/outputs are HOST buffers (pinned for full speed); the
 * host<->device copies are part of the call.  Synchronises. */
enum { CC_RUN_HOST = 1 };
typedef struct {
    cc_vp_info vp;
    cc_corr_info corr;
} cc_run_info;
cc_status cc_run(cc_ctx* ctx, int64_t n, const float* x, const float* y, const float* z,
                 const float* xh, const float* yh, const float* zh, const uint32_t* gid,
                 float* xo, float* yo, float* zo, int flags, cc_run_info* info_h);

/* f1 -- edit log.  Alg. 1 lines 11-13 and §III-B
 * "Compaction, quantization, and lossless compression": Delta = corrected -
 * decompressed; flags = bitmask of the non-zero entries of Delta, packed into bytes; edits = the
 * non-zero Delta quantised on the uniform lattice s = xi_f 2^(1-m) (xi_f = fl32(params.xi),
 * m = params.m; readings R29-R30, R32).  Independent of the context's state (uses its
 * params, stream and allocator only); one rank encodes its own particles.
 *   n:           particles, arrays in the caller's (input) order
 *   x..z:        original coordinates P (device; Alg. 1 REQUIRE): each index is stepped toward
 *                x while the decoder's fp32 x_rec would leave |x_rec - x| <= xi_f (R32)
 *   xh0..zh0:    decompressed coordinates P_hat0 (device, n floats each)
 *   xc..zc:      corrected coordinates P_hat (device, n floats each), |Delta| <= 2 xi_f
 *   flags:       device, ceil(3n/8) bytes, 4-byte aligned; coordinate k = 3i + a (a = x,y,z) is
 *                bit k%8 of byte k/8 (LSB first); bit set iff fl32 corrected != decompressed
 *   q:           device, cap int64 quantisation indices rint(Delta/s) (fp64, half to even), one
 *                per set flag bit in ascending k; |q| <= 2^(m+1)
 *   *n_edits_h:  number of set flag bits (= edits), written whatever the status
 * Errors: CC_E_ARG (null/unaligned buffer, n < 0, xi <= 0, m outside [2, 40]); CC_E_BOUND
 * (some |Delta| > 2 xi_f, or no index within 8 steps reconstructs in bound); CC_E_OOM (n_edits > cap; flags written, q not).  Synchronises. */
cc_status cc_edit_encode(cc_ctx* ctx, int64_t n, const float* x, const float* y, const float* z,
                         const float* xh0, const float* yh0, const float* zh0,
                         const float* xc, const float* yc, const float* zc, uint8_t* flags, int64_t* q,
                         int64_t cap, int64_t* n_edits_h);

/* f1 -- reconstruction (§III-B, reading R31): x_rec = fl32((double)x_hat0 + (double)q s)
 * for every flagged coordinate (edits consumed in ascending k), x_rec = x_hat0 elsewhere.
 * flags/q as written by cc_edit_encode (device); xr..zr: device outputs, n floats each.
 * Errors: CC_E_ARG; CC_E_DATA if popcount(flags) != n_edits (outputs then undefined).
 * Synchronises.  The quantisation-safety re-check is cc_build_cells +
 * cc_find_vulnerable on (P, x_rec): n_violated0 must be 0 and no CC_E_BOUND. */
cc_status cc_edit_decode(cc_ctx* ctx, int64_t n, const float* xh0, const float* yh0, const float* zh0,
                         const uint8_t* flags, const int64_t* q, int64_t n_edits, float* xr, float* yr,
                         float* zr);

/* f1 -- m-bit packing of the quantised edits (Alg. 1 line 13 P:433 "quantized to m bits"; reading
 * R33).  |q| <= 2^m, so every index is an (m+2)-bit two's-complement field; field e
 * occupies bits [e (m+2), (e+1)(m+2)) of an LSB-first stream of 32-bit words (bit b = bit b % 32 of
 * word b / 32): ceil(n_edits (m+2) / 32) words, (m+2)/8 bytes per edit.  m = params.m.
 *   cc_edit_pack:   q (device, n_edits int64) -> words (device, cap_words u32); *n_words_h = words
 *                   needed (written whatever the status).  CC_E_OOM if cap_words is too small;
 *                   CC_E_DATA if some |q| > 2^m.  Synchronises.
 *   cc_edit_unpack: words (device) -> q (device, n_edits int64), sign-extended.  Synchronises. */
cc_status cc_edit_pack(cc_ctx* ctx, const int64_t* q, int64_t n_edits, uint32_t* words, int64_t cap_words,
                       int64_t* n_words_h);
cc_status cc_edit_unpack(cc_ctx* ctx, const uint32_t* words, int64_t n_edits, int64_t* q);

/* S0 thresholds actually used (after cc_build_cells; near_pairs after the first FoF labelling
 * of ORIG or CORR, -1 before), for
 * the boundary tests: every fp32 value is the single rounding of the paper's formula (Alg. 1
 * l.1-3 P:419-421, Eq. 3; readings R2-R8 of DESIGN.md §3).  lo2s/hi2s: the
 * proven-link shells: original d2 <= lo2s => linked under any positions within
 * xi_f of the originals, d2 > hi2s => never linked (_i interior pairs, _w pairs whose minimum
 * image wraps).  r_search: ghost width / pair-search radius; r_link: FoF(ORIG) search radius. */
typedef struct {
    float xi_f, xip_f, b2, lo2, hi2, c_b, c_f, Lf, hLf;
    float lo2s_i, hi2s_i, lo2s_w, hi2s_w;
    int pad;
    double b, eps_q, mu, r_search, r_link;
    int64_t near_pairs;    /* pairs in (lo2s, lo2] U (hi2, hi2s] (the FoF near-shell list)     */
} cc_thresholds;
cc_status cc_get_thresholds(cc_ctx* ctx, cc_thresholds* out_h);

#ifdef __cplusplus
}
#endif
#endif /* CC_H */
