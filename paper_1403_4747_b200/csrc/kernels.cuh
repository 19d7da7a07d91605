// Device kernels of the FDA matvec (sm_100a).  See DESIGN.md §5 for the
// roofline of each kernel and its algorithmic bytes / evaluations per unit.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace fda {

// per source element, positions local to the source leaf centre in wave
// units (k·(y_q - c_leaf)): a = (Y0.x, Y0.y, Y0.z, n.x), b = (Y1.xyz, n.y), c = (Y2.xyz, n.z)
struct __align__(16) SrcElem {
  float4 a, b, c;
};

// near-field CTA (one target leaf): elements [tb, tb+nt), source slots [s0, s1)
// of the slot table (int2: source element, index into near_off)
struct NearTask {
  int32_t tb, nt, s0, s1;
};

struct KernelParams {
  float k;          // wavenumber
  float alpha_re;   // Burton–Miller coupling α
  float alpha_im;
  float ak_re;      // k·Re α (near kernel in wave units)
  float ak_im;      // k·Im α
  float inv_k;      // 1/k
  int skip_corr;    // FDA_NEAR_NOCORR=1 (measurement only): the near kernel skips the correction SpMV
};

// one CTA of the grouped translation kernel: a tile of XR rows × ≤ XO ops of
// dst[op] += M · src[op], all ops sharing M (rows × cols, column-major).
// 128 threads as 16 (rows) × 8 (ops); each thread owns MR × MO outputs.
// Variants (MR, MO) = (2, 8) → 32 × 64, (4, 4) → 64 × 32, (8, 2) → 128 × 16,
// (1, 16) → 16 × 128 (the r-row V̂ stage of the factored M2L);
// the host picks per matrix the variant with the least padding.
constexpr int XK = 16;   // k (column) chunk
constexpr int XV = 4;    // number of variants
struct XTask {
  int64_t mat_off;
  int32_t rows, cols;
  int32_t row0;
  int32_t op_begin, op_count;
  int32_t k_begin, k_end;   // column range (split-K: partial products are accumulated atomically)
  int32_t pad;
};
inline int xvar_rows(int v) { return v == 0 ? 32 : (v == 1 ? 64 : (v == 2 ? 128 : 16)); }
inline int xvar_ops(int v) { return v == 0 ? 64 : (v == 1 ? 32 : (v == 2 ? 16 : 128)); }

// fused §4.2 M2L task: for ≤ LR_O ops sharing K̃ ≈ Û V̂ (r ≤ 64):
// tmp = V̂ · src (r × ops, shared memory), dst += Û · tmp
constexpr int LR_O = 128;   // max ops per fused M2L CTA
struct LrTask {
  int64_t v_off, u_off;     // V̂ (r × T) and Û (T × r), column-major, in the pool
  int32_t T, r;
  int32_t op_begin, op_count;
};

// tcgen05 translation task (kernels_tc.cu): all rows of one matrix (R × C complex,
// ntile = ⌈2R/128⌉ ≤ 3 tiles of the interleaved real matrix) × ≤ 128 or 256 ops sharing it.
// The A operand is pre-laid-out per (tile, TC_KC-float K chunk) as [hi | lo] 128 × TC_KC tiles.
constexpr int TC_KC = 16;   // floats of K per pipeline stage
constexpr int TC_NV = 7;    // kernel variants (N, tiles, stages, CTAs/SM), see kernels_tc.cu
struct TcTask {
  int64_t a_off;      // float offset of the matrix's pre-laid-out A in the tensor-core pool
  int32_t R, C;       // matrix shape (complex)
  int32_t nkc;        // K chunks of the whole matrix: ⌈2C / TC_KC⌉ (layout stride of the A pool)
  int32_t ntile;      // 128-row tiles of the real matrix
  int32_t op_begin, op_count;
  int32_t kc0, kc1;   // this task's K chunks (split-K: partial products accumulate atomically)
};
int tc_variant(int n, int tiles, bool multi);   // multi: the 2-stage, several-CTAs-per-SM variants

// fused §4.2 M2L on the tensor cores (kernels_tc.cu, k_m2l_tcw): ≤ 128 ops sharing K̃ ≈ Û V̂
// with r ≤ 32; B operands pre-laid-out in the tensor-core pool (engine.cu: tc_bop)
struct LrTcTask {
  int64_t b1_off;     // float offset of A_Vᵀ: n1 rows × 2T (padded to nk1·16) K, per 16-float chunk [hi | lo]
  int64_t b2_off;     // float offset of A_Uᵀ: n2 rows × n1 K
  int32_t T, r;
  int32_t n1, n2;     // 2·⌈r/8⌉·8 and 2·⌈T/8⌉·8
  int32_t nk1;        // ⌈2T / 16⌉
  int32_t op_begin, op_count;
};
constexpr int LRTC_MAX_R = 32;
constexpr int LRBF_MAX_R = 48;    // BF16x3 form (k_m2l_bf): n1 ≤ 96, phase-2 A region ≤ 48 KB
constexpr int LRTC_MAX_T = 160;   // keeps 3 ring stages + the phase-2 A region ≤ 220 KB (n1 ≤ 64, n2 ≤ 320)
// warp-specialised persistent variant (k_m2l_tcw): launch plan from the level's max n1 / n2
struct LrTcPlan {
  int stages = 3, stage_fl = 0, b2_fl = 0, n1max = 16;
  uint32_t ncols = 32;
  size_t smem = 0;
};
LrTcPlan m2l_tcw_plan(int n1max, int n2max);
cudaError_t m2l_tcw_prepare();
// BF16x3 form (k_m2l_bf): same tasks with b1_off / b2_off → kind-2 (bf16) B layouts and
// nk1 = ⌈2T / 32⌉; the source states as pre-split bf16 hi / lo planes (launch_split_bf16)
LrTcPlan m2l_bf_plan(int n1max, int n2max);
cudaError_t m2l_bf_prepare();
void launch_m2l_bf(int ntask, const LrTcTask* tasks, const int64_t* src_off, const int64_t* dst_off,
                   const float* tcpool, const __nv_bfloat16* shi, const __nv_bfloat16* slo, float2* dst,
                   const LrTcPlan& pl, int grid, cudaStream_t s);
// dense translations in BF16x3 (k_xlate_bf): ≤ 128 ops sharing one matrix M (R × C, R ≤ 128);
// B = real 2R × 2C form of M as a bf16 B operand (k_tc_layout kind 2: n rows, nk 32-element chunks)
struct XbfTask {
  int64_t b_off;      // float offset of the bf16 B operand in the tensor-core pool
  int32_t R, C;       // matrix shape (complex)
  int32_t n;          // B rows = MMA N: 2R padded to a multiple of 16 (≤ 256)
  int32_t nk;         // ⌈2C / 32⌉
  int32_t op_begin, op_count;
};
LrTcPlan xlate_bf_plan(int nmax);
cudaError_t xlate_bf_prepare();
void launch_xlate_bf(int ntask, const XbfTask* tasks, const int64_t* src_off, const int64_t* dst_off,
                     const float* tcpool, const __nv_bfloat16* shi, const __nv_bfloat16* slo, float2* dst,
                     const LrTcPlan& pl, int grid, cudaStream_t s);
void launch_split_bf16(const float* x, int64_t n, __nv_bfloat16* hi, __nv_bfloat16* lo, cudaStream_t s);
void launch_m2l_tcw(int ntask, const LrTcTask* tasks, const int64_t* src_off, const int64_t* dst_off,
                    const float* tcpool, const float2* src, float2* dst, const LrTcPlan& pl, int grid,
                    cudaStream_t s);
int tc_variant_ops(int v);

// leaf-level ops (S2M / L2T)
struct LeafTask {
  int64_t mat_off;   // -1: no matrix (L2T writes zeros)
  int64_t state_off;
  int32_t elem_begin, elem_count;
  int32_t T;
  int32_t pad;
};

void launch_pack(const float2* out, const int64_t* idx, float2* send, int64_t n, cudaStream_t s);
void launch_unpack_add(const float2* recv, const int64_t* idx, float2* out, int64_t n, cudaStream_t s);
void launch_gather_f32(const float2* x_caller, const int32_t* perm, float2* x_tree, int n, cudaStream_t s);
void launch_gather_f64(const double2* x_caller, const int32_t* perm, float2* x_tree, int n, cudaStream_t s);
void launch_scatter_f32(const float2* y_near, const float2* y_far, const int32_t* perm, float2* y_caller, int n,
                        int e0, int e1, cudaStream_t s);
void launch_scatter_f64(const float2* y_near, const float2* y_far, const int32_t* perm, double2* y_caller, int n,
                        int e0, int e1, cudaStream_t s);
void launch_near(int ntask, const NearTask* tasks, const int2* slots, const float4* near_off, const float4* tgt_pos,
                 const float4* tgt_nrm, const SrcElem* src, const float* src_w, const int32_t* corr_ptr,
                 const int32_t* corr_col, const float2* corr_val, const float2* x, float2* y, KernelParams kp,
                 bool alpha_pure_imag, int kind, bool wide, cudaStream_t s);   // wide: 256-thread CTAs
void launch_s2m(int ntask, const LeafTask* tasks, const float2* pool, const float2* x, float2* out, int max_rows,
                cudaStream_t s);
void launch_l2t(int ntask, const LeafTask* tasks, const float2* pool, const float2* in, float2* y, cudaStream_t s,
                bool accumulate = false);
void launch_xlate(int variant, bool atomic, int ntask, const XTask* tasks, const int64_t* src_off,
                  const int64_t* dst_off, const float2* pool, const float2* src, float2* dst, cudaStream_t s);
// fused §4.2 M2L for r ≤ 64; cls = m2l_lr_class(r) (phase-1 rows m2l_lr_rows(cls) = 16 / 24 / 32 / 64)
constexpr int LR_NCLS = 4;
void launch_m2l_lr(int cls, int ntask, const LrTask* tasks, const int64_t* src_off, const int64_t* dst_off,
                   const float2* pool, const float2* src, float2* dst, cudaStream_t s);
int m2l_lr_class(int r);
int m2l_lr_rows(int cls);
int m2l_lr_ops(int cls);   // ops per CTA of a class
constexpr int LR_MAX_R = 64;
cudaError_t m2l_lr_prepare();
// src / dst state offsets must be even (16-byte aligned complex64 states)
void launch_xlate_tc(int variant, int ntask, const TcTask* tasks, const int64_t* src_off, const int64_t* dst_off,
                     const float* tcpool, const float2* src, float2* dst, cudaStream_t s);
cudaError_t tc_prepare();
// device layout of the tensor-core operand pool from the complex64 matrix pool (engine.cu:
// tc_matrix / tc_bop record one job per matrix and operand form)
struct TcLayoutJob {
  int64_t dst;        // float offset in the tensor-core pool
  int64_t src;        // complex offset of the matrix (R × C, column-major) in the pool
  int32_t R, C;
  int32_t a;          // kind 0: row tiles of 128; kind 1: padded row count nrp
  int32_t nkc;        // TC_KC-float K chunks
  int32_t kind;       // 0: A tiles [tile][chunk][hi | lo] 128 × TC_KC; 1: B operand [chunk][hi | lo] nrp × TC_KC;
                      // 2: bf16 B operand [32-element chunk][hi | lo] nrp × 32 (nkc = 32-element chunks)
  int32_t pad;        // kind 2: rows per block (0 = one block of nrp rows)
};
void launch_tc_layout(int njob, const TcLayoutJob* jobs, const float2* pool, float* tcpool, cudaStream_t s);
// warp-specialised persistent translation kernel (N = 128 ops per task, tiles ≤ 2)
cudaError_t xlate_tcw_prepare();
void launch_xlate_tcw(int tiles, int ntask, const TcTask* tasks, const int64_t* src_off, const int64_t* dst_off,
                      const float* tcpool, const float2* src, float2* dst, int grid, cudaStream_t s);
// GMRES / BLAS-1 helpers (fp64 accumulation)
void launch_dots(const float2* V, int64_t ldv, int nv, const float2* w, int64_t n, double2* partial, int nchunks,
                 cudaStream_t s);
void launch_update(float2* w, const float2* V, int64_t ldv, int nv, const double2* h, int64_t n, double sign,
                   cudaStream_t s);
void launch_norm2(const float2* w, int64_t n, double* partial, int nchunks, cudaStream_t s);
// out[i] = Σ_c partial[c*nv + i]  (device-side reduction, no host round trip)
void launch_reduce_partials(const double2* partial, int nv, int nchunks, double2* out, cudaStream_t s);
void launch_reduce_norm(const double* partial, int nchunks, double* out, cudaStream_t s);   // out = sqrt(Σ)
void launch_scale_by_inv(float2* dst, const float2* src, const double* nrm, int64_t n, cudaStream_t s);
void launch_reduce_sum(const double* partial, int nchunks, double* out, cudaStream_t s);   // out = Σ (no root)
void launch_sqrt1(double* x, cudaStream_t s);
void launch_add_slice(const float2* a, const float2* b, int64_t off, int64_t n, float2* y, cudaStream_t s);
void launch_scale(float2* dst, const float2* src, double sre, double sim, int64_t n, cudaStream_t s);
void launch_axpby(float2* y, const float2* x, double a, double b, int64_t n, cudaStream_t s);  // y = a*x + b*y (real)
void launch_plane_wave(const double* cen, const double* nrm, const int32_t* perm, int n, double k, double are,
                       double aim, double dx, double dy, double dz, float2* b32, double2* b64, cudaStream_t s);
void launch_point_source(const double* cen, const double* nrm, const int32_t* perm, int n, double k, double are,
                         double aim, double sx, double sy, double sz, float2* b32, double2* b64, cudaStream_t s);
void launch_f64_to_f32(const double2* a, float2* b, int64_t n, cudaStream_t s);
void launch_f32_to_f64(const float2* a, double2* b, int64_t n, cudaStream_t s);

}  // namespace fda
