/*
 * fda.h — C ABI of the B200-native fast directional algorithm (FDA) for the
 * Burton–Miller collocation BEM (Cao, Wen & Xiao, arXiv 1403.4747).
 *
 * The library builds, for one closed triangle mesh, the kernel-independent
 * wideband FDA of PAPER.md §3-§4 and applies the Burton–Miller LHS operator
 *
 *     y = A x,  A = ½I + D + αH,
 *     (A x)_i = ½ x_i + Σ_j ∫_Δj [∂G/∂n_y + α ∂²G/∂n_x∂n_y](x_i, y) dS_y x_j
 *
 * (Eq. (4) left side, discretised as Eq. (5), P:189-211,
 * by collocation at centroids with piecewise-constant elements, P:896-906;
 * G = e^{ikr}/(4πr), Eq. (3)) on an NVIDIA B200 (sm_100a).
 *
 * Conventions (all calls):
 *  * complex numbers: interleaved (re, im).  Device vectors are complex64
 *    (float2); host vectors passed with FDA_HOST are complex128 (double re,im)
 *    and are converted by the library.
 *  * element order: vectors are in CALLER order (the order of `triangles`);
 *    the library permutes to its internal Morton order and back.
 *  * triangles must be counter-clockwise seen from OUTSIDE the scatterer; the
 *    library negates that normal for the kernels (kernel normal n points out
 *    of the acoustic domain, into the body — SURVEY reading C1).
 *  * ownership: the caller owns every buffer passed in; the library copies the
 *    mesh at build time and owns everything it allocates (freed by fda_free).
 *    x and y must not alias.  A context is not thread-safe: one caller thread
 *    and one stream at a time.
 *  * errors: every call returns an fda_status; fda_last_error(ctx) returns a
 *    human-readable message for the last failing call on that context.
 */
#ifndef FDA_H
#define FDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FDA_OK = 0,
  FDA_E_INVALID_ARG = 1,   /* k <= 0, eps outside (0, 0.1], nt < 1, bad index, aliasing */
  FDA_E_MESH = 2,          /* degenerate triangle, repeated vertex, open/inconsistent mesh */
  FDA_E_NOMEM = 3,         /* host or device allocation failed */
  FDA_E_CUDA = 4,          /* CUDA runtime error (message has the CUDA error string) */
  FDA_E_NCCL = 5,          /* NCCL load / communicator / collective error (sharded contexts) */
  FDA_E_NOT_CONVERGED = 6, /* bm_solve hit max_iter; u holds the best iterate */
  FDA_E_STATE = 7,         /* call not valid in this state (e.g. matvec on a host-only build) */
  FDA_E_INTERNAL = 8
} fda_status;

typedef struct fda_ctx fda_ctx;          /* opaque, library-owned */
typedef struct { double re, im; } fda_cplx;

/* flags for fda_matvec / fda_rhs_plane_wave / bm_solve */
#define FDA_HOST   0   /* x, y, b, u are host complex128 arrays (copied in/out) */
#define FDA_DEVICE 1   /* x, y, b, u are device complex64 arrays on opt.device  */
#define FDA_LOCAL  2   /* (nranks > 1) return this rank's rows only, others zero; no collective */
/* (nranks > 1, with FDA_DEVICE | FDA_LOCAL) the two halves of a sharded matvec
 * around the exchange of partial outgoing states: UP = gather, near field
 * (launched), S2M + M2M of this rank's elements, pack; DOWN = unpack, M2L,
 * L2L, L2T, scatter.  Used with fda_exchange_local as a one-GPU test
 * transport; fda_matvec without these flags does UP, NCCL, DOWN. */
#define FDA_PHASE_UP   4
#define FDA_PHASE_DOWN 8
/* with FDA_HOST: the host x and y of fda_matvec / fda_rhs_apply are complex64 (float re,im)
 * instead of complex128 — the device computes in fp32 anyway, so this halves the H2D / D2H
 * bytes of a host-buffer call (pinned buffers recommended).  Not accepted by bm_solve. */
#define FDA_HOST_C64   16

typedef struct {
  int32_t max_leaf;      /* split an octree cube while it owns more elements (64)        */
  int32_t p_eq;          /* equivalent points per cube edge (8; reading C13)  */
  int32_t p_chk_lf;      /* LF check points per edge (8)                                 */
  int32_t p_chk_hf;      /* HF directional check points per edge (12; C12)               */
  double eq_scale;       /* equivalent cube side / box width (1.05; C14)                 */
  double chk_scale_lf;   /* LF check cube side / box width (2.95; C14)                   */
  double tier1_rho;      /* ρ below which the 448-point rule is used (1.5; C6)           */
  double tier2_rho;      /* ρ below which the 6-point rule is used (3.0; C6)             */
  int32_t direct_all;    /* 1: every leaf pair is direct (exact O(N²) operator)          */
  int32_t device;        /* CUDA device ordinal; -1 = host-only build (no matvec)        */
  int32_t build_threads; /* host threads for the build (0 = all)                         */
  int32_t use_graph;     /* capture the matvec as a CUDA graph (1)                       */
  int32_t verbose;       /* print build statistics to stderr                             */
  int32_t m2l_lowrank;   /* 1: second-stage SVD K̃ ≈ ÛV̂ where r < T/2 (PAPER §4.2) */
  int32_t rhs_operator;  /* 1: also build the RHS pass B (fda_rhs_apply)        */
  int32_t rank;          /* this rank (0-based) when the operator is sharded over nranks GPUs */
  int32_t nranks;        /* ranks sharing the operator (1 = unsharded)                      */
  int32_t tensor_cores;  /* dense translations (M2M, L2L, dense M2L) on tcgen05 tensor cores,
                            3xTF32: 0 never, 1 every eligible stage (factored M2L too),
                            2 (default) stages of ≥ 0.1 GFLOP with ≥ 64 ops per matrix (CUDA
                            cores elsewhere); A/B variants on every eligible stage (dense
                            ones; the factored M2L keeps its fused kernels): 3 the
                            deep-pipeline one-CTA-per-SM kernels, 4 the warp-specialised
                            persistent kernel for ≤ 2 row tiles, 5 the BF16x3 persistent
                            kernel k_xlate_bf (matrices with ≤ 128 rows; unsharded)        */
  int32_t hf_leaves;     /* 0 (default): HF cubes are always split, all leaves are LF (reading
                            C9); 1: the count rule at every level, leaves may be HF, with
                            directional S2M / L2T per used wedge (PAPER.md P:344-346,
                            P:449-454)                                                     */
  int32_t lr_tensor_cores;  /* §4.2 factored M2L (r ≤ 32, T ≤ 160) on the fused tcgen05 kernel
                            (both products on the tensor cores, tmp kept on chip; persistent,
                            warp-specialised k_m2l_bf / k_m2l_tcw): 0 never (fused CUDA-core
                            kernel), 1 always, 2 (default) every level with m2l_bf16 = 1, with
                            3xTF32 only levels with ≥ 64 ops per factored K̃ and ≥ 3 GFLOP
                            (DESIGN.md §5); needs tensor_cores ≠ 0                          */
  int32_t build_on_device;  /* 1 (default): the fp64 operator and correction tables of
                            fda_build are computed on opt.device (build_dev.cu: kernel-matrix
                            generation, batched fp64 complex GEMMs, tier quadrature), the
                            same definitions as the host build; 0: host C++/OpenMP only.
                            Ignored (host) when opt.device = -1                             */
  int32_t m2l_bf16;      /* the tensor-core factored M2L (lr_tensor_cores) in BF16x3: operands
                            split once into bf16 hi / lo, hi·hi + hi·lo + lo·hi on tcgen05
                            kind::f16 (≈ 2⁻¹⁶ relative per product) — 1 (default);
                            0: 3xTF32 (fp32-accurate products)                             */
} fda_options;

typedef struct {
  int32_t iterations;     /* GMRES iterations performed                                  */
  int32_t converged;      /* 1 if ‖b - Au‖/‖b‖ (recursive estimate) <= tol                */
  double rel_residual;    /* recursive GMRES residual estimate |g_{j+1}|/‖b‖              */
  double true_residual;   /* ‖b - Au‖/‖b‖ recomputed with one extra matvec                */
  double t_solve_s;       /* wall time of the solve (device-synchronised)                 */
} fda_solve_info;

typedef struct {
  int64_t n_elements;
  int32_t n_levels;
  int32_t n_hf_levels;
  int64_t n_boxes;
  int64_t n_leaves;
  int64_t n_out_states;
  int64_t n_in_states;
  int64_t n_m2l_pairs;
  int64_t n_m2m_ops;
  int64_t n_l2l_ops;
  int64_t n_direct_leaf_pairs;
  int64_t n_direct_element_pairs;
  int64_t n_corrections;
  int64_t n_matrices;
  int64_t table_bytes;          /* complex64 operator tables on the device              */
  double t_build_s;             /* wall time of fda_build                               */
  int32_t rank[32];             /* retained SVD rank T per level (0 = no states)        */
  int32_t dirs[32];             /* directions per level (0 = LF)                        */
  double width[32];             /* cube width per level                                 */
} fda_build_info;

/* Defaults listed above. */
fda_status fda_options_default(fda_options* opt);

/* Build the FDA for the mesh (fda_build(mesh, k, alpha, eps) of BASELINE.json).
 * vertices: nv×3 float64, triangles: nt×3 int32 (0-based, CCW from outside),
 * k > 0 wavenumber (Eq. 1), alpha the Burton–Miller coupling
 * (Eq. 4; i/k recommended, Im α ≠ 0), eps ∈ (0, 0.1] the SVD
 * truncation threshold σ_i < ε σ_0 (Eq. (eq_epsg)/(eq_epsk), P:692-695,
 * P:803-806).  opt may be NULL (defaults).  On success *out owns the context.
 * Setup = PAPER.md Algorithm Step 1 plus the compressed tables of
 * §4 and the near-field correction table; fp64 numerics. */
fda_status fda_build(const double* vertices, int64_t nv, const int32_t* triangles, int64_t nt,
                     double k, fda_cplx alpha, double eps, const fda_options* opt,
                     fda_ctx** out);

/* y = A x (the LHS Burton–Miller operator, Eq. (5)) via the FDA: upward pass
 * (S2M, M2M), downward pass (M2L, L2L, L2T) and near field (S2T), PAPER.md
 * Algorithm Steps 2-4.  flags: FDA_HOST or FDA_DEVICE.  stream:
 * cudaStream_t the call is ordered on (NULL = the legacy default stream); with
 * FDA_DEVICE the call is asynchronous w.r.t. the host. */
fda_status fda_matvec(fda_ctx* ctx, const void* x, void* y, int32_t flags, void* stream);

/* b_i = u_inc(x_i) + α ∂u_inc/∂n(x_i) for u_inc = e^{ik d·x} (Eq. (4) right
 * side with ∂u/∂n = 0, reading C22).  dir need not be unit. */
fda_status fda_rhs_plane_wave(fda_ctx* ctx, const double dir[3], void* b, int32_t flags);

/* b_i = u_inc(x_i) + α ∂u_inc/∂n(x_i) for a unit point source
 * u_inc(x) = e^{ikR}/(4πR), R = |x - src| (Eq. (3)), outside the
 * scatterer — the incident field of PAPER.md §5.2 ("The point source is at
 * (-2, 0, 0)"; Table 3).  n_i is the kernel normal (into the
 * body, reading C1).  src: 3 doubles (host).  b: caller order, FDA_HOST
 * (complex128) or FDA_DEVICE (complex64), computed in fp64 on the device.
 * FDA_E_INVALID_ARG if src is not finite or coincides with a collocation
 * point. */
fda_status fda_rhs_point_source(fda_ctx* ctx, const double src[3], void* b, int32_t flags);

/* b = B v with B = -(α/2)I + S + αK' — the right-hand-side operator of Eq. (4)
 * (P:176-181): (B v)_i = -(α/2) v_i + Σ_j ∫_Δj [G + α ∂G/∂n_x](x_i, y) dS_y v_j,
 * applied by the second fast directional pass (G sources, the same target
 * kernel and translation tables).  For a Neumann problem with
 * ∂u/∂n = v (n into the body) the BM system is A u = B v.  Needs a context
 * built with opt.rhs_operator = 1 (FDA_E_STATE otherwise).  Same vector
 * conventions as fda_matvec. */
fda_status fda_rhs_apply(fda_ctx* ctx, const void* v, void* b, int32_t flags, void* stream);

/* Solve A u = rhs by GMRES (§5: tolerance on the relative
 * residual, no preconditioner; reading C20).  restart = 0: no restart.
 * Returns FDA_E_NOT_CONVERGED (u = last iterate, info filled) at max_iter.
 * Sharded contexts (opt.nranks > 1, collective over the ranks, after
 * fda_comm_init): every Krylov vector holds only the rank's own rows; the inner
 * products are all-reduced (ncclAllReduce of j + 1 complex values per CGS
 * pass), each matvec all-gathers its input (ncclBroadcast of every rank's
 * slice) and keeps its output local; rhs and u are full-length on every rank. */
fda_status bm_solve(fda_ctx* ctx, const void* rhs, void* u, double tol, int32_t max_iter,
                    int32_t restart, fda_solve_info* info, int32_t flags);

fda_status fda_stats(const fda_ctx* ctx, fda_build_info* info);

/* Multi-GPU.  With opt.nranks > 1 every rank builds the same
 * mesh with its own opt.rank; the leaves are split into contiguous Morton
 * ranges balanced by estimated work.  Per matvec each rank runs the upward
 * pass (S2M, M2M; Algorithm Step 2) on its own elements only,
 * producing PARTIAL outgoing states (the full state is the sum over ranks, by
 * linearity); one grouped ncclSend/ncclRecv then delivers to every rank the
 * other ranks' partials of exactly the outgoing states its M2L ops read (the
 * equivalent densities of boxes in its interaction lists, including the top
 * levels of the tree); the rank adds them and runs M2L/L2L for the incoming
 * states of boxes containing its leaves, L2T and the near field (which
 * overlaps the exchange) for its own leaves.  fda_matvec / fda_rhs_apply then
 * sum the ranks' rows with one NCCL all-reduce of y (skipped with FDA_LOCAL),
 * so every rank returns the full y and bm_solve runs unchanged on every rank.
 * Vectors x are full-length on every rank.
 * fda_nccl_unique_id: 128-byte NCCL id generated on one rank (libnccl is
 * loaded on first use); the caller broadcasts it (e.g. torch.distributed);
 * fda_comm_init: collective over the nranks ranks, before the first matvec. */
fda_status fda_nccl_unique_id(void* id128);
fda_status fda_comm_init(fda_ctx* ctx, const void* id128);

/* Test transport of the sharded exchange on ONE GPU ("fake-partition mode",
 * SURVEY §4): ctxs[0..n) are the n rank contexts of one sharded build
 * (opt.nranks = n, opt.rank = index), all on the same device, each having
 * completed fda_matvec(..., FDA_DEVICE | FDA_LOCAL | FDA_PHASE_UP); copies
 * every rank's packed partials into its peers' receive buffers (synchronous),
 * after which each rank runs FDA_PHASE_DOWN.  FDA_E_INTERNAL if the ranks'
 * send / receive plans disagree. */
fda_status fda_exchange_local(fda_ctx** ctxs, int32_t n);

/* Per-stage device times (ms, CUDA events) of the last fda_matvec timed with
 * fda_set_profiling(ctx, 1): [gather, near, s2m, m2m, m2l, l2l, l2t, scatter].
 * n = capacity of ms; returns the number of stages written in *n. */
fda_status fda_set_profiling(fda_ctx* ctx, int32_t on);
/* Device time (ms) of the near-field kernel (row a7) in the last fda_matvec /
 * fda_rhs_apply, from CUDA events recorded on its own stream inside the
 * captured graph, i.e. while it runs concurrently with the far field (no
 * profiling mode needed).  Synchronises on that event.  FDA_E_STATE before
 * the first matvec. */
fda_status fda_near_time(fda_ctx* ctx, double* ms);
fda_status fda_stage_times(fda_ctx* ctx, double* ms, int32_t* n);
/* Per-kernel-family device time (ms, CUDA events around every launch on the
 * one stream of a profiled, serialised matvec: fda_set_profiling(ctx, 1) then
 * fda_matvec(..., FDA_DEVICE, ...) on an unsharded context), summed over the
 * family's launches, in the order [k_gather, k_near, k_s2m, k_xlate,
 * k_xlate_tc, k_xlate_tcw, k_m2l_lr, k_m2l_tcw, k_l2t, k_scatter, memset, k_xlate_bf] —
 * the launch-list share of each __global__ function.  n = capacity; returns
 * the count written in *n.  FDA_E_STATE before such a matvec. */
fda_status fda_kernel_times(fda_ctx* ctx, double* ms, int32_t* n);

/* Copy a named host-side build table (for host-logic tests; see
 * paper_1403_4747_b200/fda.py for the names).  If dst is NULL only *count
 * (number of elements) and *elem_bytes are returned. */
fda_status fda_debug_table(const fda_ctx* ctx, const char* name, void* dst, int64_t* count,
                           int32_t* elem_bytes);

const char* fda_last_error(const fda_ctx* ctx);
const char* fda_status_string(fda_status s);
void fda_free(fda_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* FDA_H */
