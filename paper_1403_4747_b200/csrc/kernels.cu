// Device kernels of the FDA Burton–Miller matvec (sm_100a, complex64 data,
// fp32 arithmetic; fp64 accumulation in the GMRES reductions).
#include <cuda_runtime.h>
#include <math_constants.h>

#include "kernels.cuh"

namespace fda {

// ------------------------------------------------------------------ permutes
// a1 gather: x_tree[i] = x_caller[perm[i]]  (HBM-bound, 16 B/element)
__global__ void k_gather_f32(const float2* __restrict__ xc, const int32_t* __restrict__ perm,
                             float2* __restrict__ xt, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) xt[i] = xc[perm[i]];
}
__global__ void k_gather_f64(const double2* __restrict__ xc, const int32_t* __restrict__ perm,
                             float2* __restrict__ xt, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    double2 v = xc[perm[i]];
    xt[i] = make_float2((float)v.x, (float)v.y);
  }
}
// a8 scatter: y_caller[perm[i]] = y_near[i] + y_far[i] for owned rows i ∈ [e0, e1), 0 otherwise
__global__ void k_scatter_f32(const float2* __restrict__ yn, const float2* __restrict__ yf,
                              const int32_t* __restrict__ perm, float2* __restrict__ yc, int n, int e0, int e1) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    float2 v = make_float2(0.f, 0.f);
    if (i >= e0 && i < e1) {
      float2 a = yn[i], b = yf[i];
      v = make_float2(a.x + b.x, a.y + b.y);
    }
    yc[perm[i]] = v;
  }
}
__global__ void k_scatter_f64(const float2* __restrict__ yn, const float2* __restrict__ yf,
                              const int32_t* __restrict__ perm, double2* __restrict__ yc, int n, int e0, int e1) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    double2 v = make_double2(0.0, 0.0);
    if (i >= e0 && i < e1) {
      float2 a = yn[i], b = yf[i];
      v = make_double2((double)a.x + (double)b.x, (double)a.y + (double)b.y);
    }
    yc[perm[i]] = v;
  }
}

void launch_gather_f32(const float2* x, const int32_t* perm, float2* xt, int n, cudaStream_t s) {
  k_gather_f32<<<(n + 255) / 256, 256, 0, s>>>(x, perm, xt, n);
}
void launch_gather_f64(const double2* x, const int32_t* perm, float2* xt, int n, cudaStream_t s) {
  k_gather_f64<<<(n + 255) / 256, 256, 0, s>>>(x, perm, xt, n);
}
void launch_scatter_f32(const float2* yn, const float2* yf, const int32_t* perm, float2* yc, int n, int e0, int e1,
                        cudaStream_t s) {
  k_scatter_f32<<<(n + 255) / 256, 256, 0, s>>>(yn, yf, perm, yc, n, e0, e1);
}
void launch_scatter_f64(const float2* yn, const float2* yf, const int32_t* perm, double2* yc, int n, int e0, int e1,
                        cudaStream_t s) {
  k_scatter_f64<<<(n + 255) / 256, 256, 0, s>>>(yn, yf, perm, yc, n, e0, e1);
}

// ------------------------------------------------------------------ near field (a7)
// y_i = Σ_{j ∈ direct(i)} A^{Q3}_ij x_j + Σ_{j: ρ_ij<3} C_ij x_j
// A^{Q3}_ij = (A_j/3) Σ_q [∂G/∂n_y + α ∂²G/∂n_x∂n_y](x_i, y_jq)   (Eq. 5)
// One CTA per target leaf; the source elements of all direct leaves are staged
// through shared memory in chunks; P = ⌊NT/n_B⌋ threads share one target and
// split the sources; partial sums are reduced in shared memory.
constexpr int NEAR_NT = 128;
constexpr int NEAR_MAXS = 256;
constexpr int NEAR_MAXL = 256;

// MUFU.RSQ without the denormal guard of rsqrtf (r² ≥ 1e-12 here, never denormal)
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// One Q3 point of the LHS kernel, accumulated into acc:
//   acc += [∂G/∂n_y + α ∂²G/∂n_x∂n_y](x, y) · w      (w = x_j A_j/(12π))
// With q = kr, a = ∂r/∂n_x, b = ∂r/∂n_y, c = n_x·n_y:
//   4π r² e^{-iq} ∂G/∂n_y          = (iq - 1) b
//   4π r² e^{-iq} ∂²G/∂n_x∂n_y     = (1/r) [ (3 - q²) ab + c - iq (3ab + c) ]
// PURE_IMAG specialises α = i·alpha_im (α = i/k).
template <bool PURE_IMAG>
__device__ __forceinline__ void lhs_eval(float3 x, float3 nx, float3 y, float3 ny, float cn, float2 w,
                                         const KernelParams& kp, float2& acc) {
  const float dx = x.x - y.x, dy = x.y - y.y, dz = x.z - y.z;
  const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
  const float ir = rsqrt_ftz(r2);
  const float q = kp.k * (r2 * ir);
  const float a = fmaf(dx, nx.x, fmaf(dy, nx.y, dz * nx.z)) * ir;   // ∂r/∂n_x
  const float b = -fmaf(dx, ny.x, fmaf(dy, ny.y, dz * ny.z)) * ir;  // ∂r/∂n_y
  const float ab = a * b;
  float sn, cs;
  __sincosf(q, &sn, &cs);  // SFU sin/cos; |q| ≤ k·(near range), argument error ≤ ulp(q/2π)
  const float g = fmaf(3.0f, ab, cn);           // 3ab + c
  const float u1 = fmaf(fmaf(-q, q, 3.0f), ab, cn);  // (3 - q²) ab + c
  float P, Q;
  if (PURE_IMAG) {
    // -b - α_i ir u2 with u2 = -q g and ir·q = k  →  -b + (α_i k) g
    P = fmaf(kp.alpha_im * kp.k, g, -b);
    Q = fmaf(kp.alpha_im * ir, u1, q * b);   //  q b + α_i ir u1
  } else {
    const float u2 = -q * g;
    P = fmaf(ir, kp.alpha_re * u1 - kp.alpha_im * u2, -b);
    Q = fmaf(ir, kp.alpha_re * u2 + kp.alpha_im * u1, q * b);
  }
  const float ir2 = ir * ir;
  const float Er = ir2 * cs, Ei = ir2 * sn;
  const float Kr = Er * P - Ei * Q;
  const float Ki = Er * Q + Ei * P;
  acc.x = fmaf(Kr, w.x, fmaf(-Ki, w.y, acc.x));
  acc.y = fmaf(Kr, w.y, fmaf(Ki, w.x, acc.y));
}

// One Q3 point of the RHS kernel (Eq. 4 right side):
//   acc += [G + α ∂G/∂n_x](x, y) · w,   4π r² e^{-iq} (G + α ∂G/∂n_x) = r + α (iq - 1) a
__device__ __forceinline__ void rhs_eval(float3 x, float3 nx, float3 y, float2 w, const KernelParams& kp,
                                         float2& acc) {
  const float dx = x.x - y.x, dy = x.y - y.y, dz = x.z - y.z;
  const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
  const float ir = rsqrt_ftz(r2);
  const float r = r2 * ir;
  const float q = kp.k * r;
  const float a = fmaf(dx, nx.x, fmaf(dy, nx.y, dz * nx.z)) * ir;
  float sn, cs;
  __sincosf(q, &sn, &cs);
  const float P = fmaf(-a, fmaf(kp.alpha_im, q, kp.alpha_re), r);   // r - a (α_r + α_i q)
  const float Q = a * fmaf(kp.alpha_re, q, -kp.alpha_im);           // a (α_r q - α_i)
  const float ir2 = ir * ir;
  const float Er = ir2 * cs, Ei = ir2 * sn;
  const float Kr = Er * P - Ei * Q;
  const float Ki = Er * Q + Ei * P;
  acc.x = fmaf(Kr, w.x, fmaf(-Ki, w.y, acc.x));
  acc.y = fmaf(Kr, w.y, fmaf(Ki, w.x, acc.y));
}

// y_i = Σ_{j ∈ direct(i)} A^{Q3}_ij x_j + Σ_{j: ρ_ij<3} C_ij x_j   (a7)
// A^{Q3}_ij = (A_j/3) Σ_q [∂G/∂n_y + α ∂²G/∂n_x∂n_y](x_i, y_jq)   (Eq. 5)
// One CTA per target leaf (leaves launched in descending-work order); the
// source elements of all direct leaves are staged through shared memory in
// chunks; P = ⌊NT/n_B⌋ threads share one target and split the sources;
// partial sums are reduced in shared memory.
// KIND 0: LHS operator A (Eq. 5); KIND 1: RHS operator B (G sources).
template <int KIND, bool PURE_IMAG>
__global__ void __launch_bounds__(NEAR_NT) k_near(
    const int32_t* __restrict__ order, const int32_t* __restrict__ leaf_begin, const int32_t* __restrict__ leaf_end,
    const int32_t* __restrict__ near_ptr, const int32_t* __restrict__ near_idx,
    const float4* __restrict__ near_off, const float4* __restrict__ tgt_pos, const float4* __restrict__ tgt_nrm,
    const SrcElem* __restrict__ src, const float* __restrict__ src_w, const int32_t* __restrict__ corr_ptr,
    const int32_t* __restrict__ corr_col, const float2* __restrict__ corr_val, const float2* __restrict__ x,
    float2* __restrict__ y, KernelParams kp) {
  __shared__ float4 sa[NEAR_MAXS], sb[NEAR_MAXS], sc[NEAR_MAXS];
  __shared__ float2 sx[NEAR_MAXS];
  __shared__ int spre[NEAR_MAXL + 1];
  __shared__ float2 sred[NEAR_NT];
  const int leaf = order[blockIdx.x];
  const int tb = leaf_begin[leaf];
  const int nt = leaf_end[leaf] - tb;
  const int P = max(1, NEAR_NT / nt);
  const int tid = threadIdx.x;
  const int ti = tid % nt, part = tid / nt;
  const bool active = part < P && ti < nt;
  float3 xt = make_float3(0.f, 0.f, 0.f), nx = xt;
  if (active) {
    float4 p = tgt_pos[tb + ti], q = tgt_nrm[tb + ti];
    xt = make_float3(p.x, p.y, p.z);
    nx = make_float3(q.x, q.y, q.z);
  }
  float2 acc = make_float2(0.f, 0.f);
  const int lb = near_ptr[leaf], le = near_ptr[leaf + 1];
  for (int e0 = lb; e0 < le; e0 += NEAR_MAXL) {
    const int ne = min(NEAR_MAXL, le - e0);
    __syncthreads();
    if (tid < 32) {  // warp-parallel exclusive scan of the source-leaf sizes
      int carry = 0;
      for (int j0 = 0; j0 < ne; j0 += 32) {
        const int j = j0 + tid;
        int v = 0;
        if (j < ne) {
          const int c = near_idx[e0 + j];
          v = leaf_end[c] - leaf_begin[c];
        }
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          int t = __shfl_up_sync(0xffffffffu, incl, o);
          if (tid >= o) incl += t;
        }
        if (j < ne) spre[j] = carry + incl - v;
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (tid == 0) spre[ne] = carry;
    }
    __syncthreads();
    const int total = spre[ne];
    for (int base = 0; base < total; base += NEAR_MAXS) {
      const int ns = min(NEAR_MAXS, total - base);
      for (int slot = tid; slot < ns; slot += NEAR_NT) {
        const int g = base + slot;
        int lo = 0, hi = ne - 1;  // last j with spre[j] <= g
        while (lo < hi) {
          int mid = (lo + hi + 1) >> 1;
          if (spre[mid] <= g) lo = mid; else hi = mid - 1;
        }
        const int c = near_idx[e0 + lo];
        const int el = leaf_begin[c] + (g - spre[lo]);
        const float4 off = near_off[e0 + lo];  // c_B - c_C
        SrcElem se = src[el];
        se.a.x -= off.x; se.a.y -= off.y; se.a.z -= off.z;
        se.b.x -= off.x; se.b.y -= off.y; se.b.z -= off.z;
        se.c.x -= off.x; se.c.y -= off.y; se.c.z -= off.z;
        sa[slot] = se.a; sb[slot] = se.b; sc[slot] = se.c;
        const float2 xv = x[el];
        const float wv = src_w[el];
        sx[slot] = make_float2(xv.x * wv, xv.y * wv);
      }
      __syncthreads();
      if (active) {
#pragma unroll 2
        for (int s = part; s < ns; s += P) {
          const float4 A = sa[s], B = sb[s], C = sc[s];
          const float2 w = sx[s];
          if (KIND == 0) {
            const float3 ny = make_float3(A.w, B.w, C.w);
            const float cn = fmaf(nx.x, ny.x, fmaf(nx.y, ny.y, nx.z * ny.z));
            lhs_eval<PURE_IMAG>(xt, nx, make_float3(A.x, A.y, A.z), ny, cn, w, kp, acc);
            lhs_eval<PURE_IMAG>(xt, nx, make_float3(B.x, B.y, B.z), ny, cn, w, kp, acc);
            lhs_eval<PURE_IMAG>(xt, nx, make_float3(C.x, C.y, C.z), ny, cn, w, kp, acc);
          } else {
            rhs_eval(xt, nx, make_float3(A.x, A.y, A.z), w, kp, acc);
            rhs_eval(xt, nx, make_float3(B.x, B.y, B.z), w, kp, acc);
            rhs_eval(xt, nx, make_float3(C.x, C.y, C.z), w, kp, acc);
          }
        }
      }
      __syncthreads();
    }
  }
  // correction SpMV, rows split over the P parts
  if (active) {
    const int i = tb + ti;
    const int cb = corr_ptr[i], ce = corr_ptr[i + 1];
    for (int e = cb + part; e < ce; e += P) {
      const float2 v = corr_val[e];
      const float2 xv = x[corr_col[e]];
      acc.x = fmaf(v.x, xv.x, fmaf(-v.y, xv.y, acc.x));
      acc.y = fmaf(v.x, xv.y, fmaf(v.y, xv.x, acc.y));
    }
  }
  sred[tid] = active ? acc : make_float2(0.f, 0.f);
  __syncthreads();
  if (tid < nt) {
    float2 s = make_float2(0.f, 0.f);
    for (int p = 0; p < P; ++p) {
      float2 v = sred[p * nt + tid];
      s.x += v.x; s.y += v.y;
    }
    y[tb + tid] = s;
  }
}

void launch_near(int nleaf, const int32_t* order, const int32_t* leaf_begin, const int32_t* leaf_end,
                 const int32_t* near_ptr, const int32_t* near_idx, const float4* near_off, const float4* tgt_pos,
                 const float4* tgt_nrm, const SrcElem* src, const float* src_w, const int32_t* corr_ptr,
                 const int32_t* corr_col, const float2* corr_val, const float2* x, float2* y, KernelParams kp,
                 bool alpha_pure_imag, int kind, cudaStream_t s) {
  if (nleaf <= 0) return;
#define NEAR(K, PI)                                                                                          \
  k_near<K, PI><<<nleaf, NEAR_NT, 0, s>>>(order, leaf_begin, leaf_end, near_ptr, near_idx, near_off, tgt_pos, \
                                          tgt_nrm, src, src_w, corr_ptr, corr_col, corr_val, x, y, kp)
  if (kind == 1) NEAR(1, false);
  else if (alpha_pure_imag) NEAR(0, true);
  else NEAR(0, false);
#undef NEAR
}

// ------------------------------------------------------------------ S2M (a2) / L2T (a6)
// S2M: m̃_B = S̃_B x_B (T × n_B, column-major); one CTA per leaf, thread = row.
__global__ void k_s2m(const LeafTask* __restrict__ tasks, const float2* __restrict__ pool,
                      const float2* __restrict__ x, float2* __restrict__ out) {
  __shared__ float2 sx[128];
  const LeafTask t = tasks[blockIdx.x];
  for (int j = threadIdx.x; j < t.elem_count; j += blockDim.x) sx[j] = x[t.elem_begin + j];
  __syncthreads();
  const float2* M = pool + t.mat_off;
  for (int r = threadIdx.x; r < t.T; r += blockDim.x) {
    float2 acc = make_float2(0.f, 0.f);
    for (int j = 0; j < t.elem_count; ++j) {
      const float2 m = M[(int64_t)j * t.T + r];
      const float2 v = sx[j];
      acc.x = fmaf(m.x, v.x, fmaf(-m.y, v.y, acc.x));
      acc.y = fmaf(m.x, v.y, fmaf(m.y, v.x, acc.y));
    }
    out[t.state_off + r] = acc;
  }
}

// L2T: y_B = T̃_B ℓ̃_B (n_B × T column-major); thread = target element.
__global__ void k_l2t(const LeafTask* __restrict__ tasks, const float2* __restrict__ pool,
                      const float2* __restrict__ in, float2* __restrict__ y) {
  __shared__ float2 sl[320];
  const LeafTask t = tasks[blockIdx.x];
  if (t.mat_off < 0) {
    for (int i = threadIdx.x; i < t.elem_count; i += blockDim.x) y[t.elem_begin + i] = make_float2(0.f, 0.f);
    return;
  }
  for (int c = threadIdx.x; c < t.T; c += blockDim.x) sl[c] = in[t.state_off + c];
  __syncthreads();
  const float2* M = pool + t.mat_off;
  for (int i = threadIdx.x; i < t.elem_count; i += blockDim.x) {
    float2 acc = make_float2(0.f, 0.f);
    for (int c = 0; c < t.T; ++c) {
      const float2 m = M[(int64_t)c * t.elem_count + i];
      const float2 v = sl[c];
      acc.x = fmaf(m.x, v.x, fmaf(-m.y, v.y, acc.x));
      acc.y = fmaf(m.x, v.y, fmaf(m.y, v.x, acc.y));
    }
    y[t.elem_begin + i] = acc;
  }
}

void launch_s2m(int ntask, const LeafTask* tasks, const float2* pool, const float2* x, float2* out, int max_rows,
                cudaStream_t s) {
  if (ntask <= 0) return;
  int bd = ((max_rows + 31) / 32) * 32;
  bd = bd < 32 ? 32 : (bd > 256 ? 256 : bd);
  k_s2m<<<ntask, bd, 0, s>>>(tasks, pool, x, out);
}
void launch_l2t(int ntask, const LeafTask* tasks, const float2* pool, const float2* in, float2* y, cudaStream_t s) {
  if (ntask <= 0) return;
  k_l2t<<<ntask, 64, 0, s>>>(tasks, pool, in, y);
}

// ------------------------------------------------------------------ translations (a3 M2M, a4 M2L, a5 L2L)
// Grouped complex GEMM with gathered inputs and scattered accumulation:
// for the ops of one task (all sharing M), D[:, p] = M[row0:row0+XR, :] S[:, p]
// with S[:, p] = src[src_off[p] : +cols]; then dst[dst_off[p] + row] += D.
// K is streamed in chunks of XK through a two-stage cp.async shared-memory
// pipeline (the copy of chunk k+1 overlaps the FMAs of chunk k); each thread keeps an
// MR × MO complex register tile, so one k step costs MR + MO shared loads for
// 4·MR·MO FFMA.  Several tasks may target one state: fp32 vector atomics.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 8 : 0;   // src-size 0 → zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_async_wait_0() { asm volatile("cp.async.wait_group 0;\n" ::); }

template <int MR, int MO, bool ATOMIC>
__global__ void __launch_bounds__(128) k_xlate(const XTask* __restrict__ tasks, const int64_t* __restrict__ src_off,
                                               const int64_t* __restrict__ dst_off, const float2* __restrict__ pool,
                                               const float2* __restrict__ src, float2* __restrict__ dst) {
  constexpr int R = 16 * MR, O = 8 * MO;
  constexpr int ML = XK * R / 128, SL = XK * O / 128;  // cp.async per thread per chunk
  __shared__ __align__(16) float2 sM[2][XK][R];
  __shared__ __align__(16) float2 sS[2][XK][O + 1];
  __shared__ int64_t soff[O];
  const XTask t = tasks[blockIdx.x];
  const int tid = threadIdx.x, tr = tid & 15, to = tid >> 4;
  for (int p = tid; p < O; p += 128) soff[p] = p < t.op_count ? src_off[t.op_begin + p] : -1;
  __syncthreads();
  const float2* __restrict__ M = pool + t.mat_off;
  auto issue = [&](int buf, int k0) {
#pragma unroll
    for (int e = 0; e < ML; ++e) {
      const int idx = tid + 128 * e;
      const int kk = idx / R, r = idx % R;
      const int row = t.row0 + r, col = k0 + kk;
      const bool ok = row < t.rows && col < t.k_end;
      cp_async8(&sM[buf][kk][r], ok ? (const void*)(M + (int64_t)col * t.rows + row) : (const void*)M, ok);
    }
#pragma unroll
    for (int e = 0; e < SL; ++e) {
      const int idx = tid + 128 * e;
      const int p = idx / XK, kk = idx % XK;
      const int col = k0 + kk;
      const int64_t so = soff[p];
      const bool ok = so >= 0 && col < t.k_end;
      cp_async8(&sS[buf][kk][p], ok ? (const void*)(src + so + col) : (const void*)src, ok);
    }
    cp_async_commit();
  };
  float2 acc[MR][MO];
#pragma unroll
  for (int i = 0; i < MR; ++i)
#pragma unroll
    for (int j = 0; j < MO; ++j) acc[i][j] = make_float2(0.f, 0.f);
  issue(0, t.k_begin);
  int buf = 0;
  for (int k0 = t.k_begin; k0 < t.k_end; k0 += XK) {
    if (k0 + XK < t.k_end) {
      issue(buf ^ 1, k0 + XK);
      cp_async_wait_1();
    } else {
      cp_async_wait_0();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < XK; ++kk) {
      float2 m[MR], sv[MO];
#pragma unroll
      for (int i = 0; i < MR; ++i) m[i] = sM[buf][kk][tr + 16 * i];
#pragma unroll
      for (int j = 0; j < MO; ++j) sv[j] = sS[buf][kk][to + 8 * j];
#pragma unroll
      for (int i = 0; i < MR; ++i)
#pragma unroll
        for (int j = 0; j < MO; ++j) {
          acc[i][j].x = fmaf(m[i].x, sv[j].x, fmaf(-m[i].y, sv[j].y, acc[i][j].x));
          acc[i][j].y = fmaf(m[i].x, sv[j].y, fmaf(m[i].y, sv[j].x, acc[i][j].y));
        }
    }
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int j = 0; j < MO; ++j) {
    const int op = to + 8 * j;
    if (op >= t.op_count) continue;
    float2* d = dst + dst_off[t.op_begin + op];
#pragma unroll
    for (int i = 0; i < MR; ++i) {
      const int row = t.row0 + tr + 16 * i;
      if (row < t.rows) {
        if (ATOMIC) atomicAdd(d + row, acc[i][j]);
        else d[row] = acc[i][j];
      }
    }
  }
}

void launch_xlate(int variant, bool atomic, int ntask, const XTask* tasks, const int64_t* src_off,
                  const int64_t* dst_off, const float2* pool, const float2* src, float2* dst, cudaStream_t s) {
  if (ntask <= 0) return;
#define XL(MR, MO)                                                                                        \
  (atomic ? k_xlate<MR, MO, true><<<ntask, 128, 0, s>>>(tasks, src_off, dst_off, pool, src, dst)          \
          : k_xlate<MR, MO, false><<<ntask, 128, 0, s>>>(tasks, src_off, dst_off, pool, src, dst))
  switch (variant) {
    case 0: XL(2, 8); break;
    case 1: XL(4, 4); break;
    case 2: XL(8, 2); break;
    default: XL(1, 16); break;
  }
#undef XL
}

// ------------------------------------------------------------------ fused §4.2 M2L (a4)
// PAPER.md §4.2: K̃ ≈ Û V̂.  One CTA handles ≤ 64 ops of one K̃:
// phase 1 tmp = V̂ S (r ≤ 32 rows, K = T streamed through a cp.async double
// buffer, 2×8 complex register tile per thread), tmp kept in shared memory;
// phase 2 for each 32-row tile of Û: out = Û_tile tmp (K = r from shared
// memory), accumulated into the destination states with vector atomics.
constexpr int LR_SH1 = 2 * XK * 32 + 2 * XK * (LR_O + 1);   // phase 1: sM[2][XK][32] + sS[2][XK][O+1]
constexpr int LR_SH2 = 32 * (LR_O + 1) + 32 * 33;            // phase 2: tmp[32][O+1] + sU[32][33]
constexpr int LR_SH = LR_SH1 > LR_SH2 ? LR_SH1 : LR_SH2;

template <int MR1>  // phase-1 rows = 16·MR1 ≥ r
__device__ __forceinline__ void m2l_lr_body(const LrTask& t, float2* sh, int64_t* soff,
                                            const int64_t* __restrict__ dst_off, const float2* __restrict__ pool,
                                            const float2* __restrict__ src, float2* __restrict__ dst) {
  constexpr int R = 32, O = LR_O, R1 = 16 * MR1;
  float2(*sM)[XK][R] = reinterpret_cast<float2(*)[XK][R]>(sh);
  float2(*sS)[XK][O + 1] = reinterpret_cast<float2(*)[XK][O + 1]>(sh + 2 * XK * R);
  float2(*tmp)[O + 1] = reinterpret_cast<float2(*)[O + 1]>(sh);
  float2(*sU)[R + 1] = reinterpret_cast<float2(*)[R + 1]>(sh + R * (O + 1));
  const int tid = threadIdx.x, tr = tid & 15, to = tid >> 4;
  const float2* __restrict__ V = pool + t.v_off;
  const float2* __restrict__ U = pool + t.u_off;
  auto issue = [&](int buf, int k0) {
#pragma unroll
    for (int e = 0; e < XK * R1 / 128; ++e) {
      const int idx = tid + 128 * e;
      const int kk = idx / R1, row = idx % R1, col = k0 + kk;
      const bool ok = row < t.r && col < t.T;
      cp_async8(&sM[buf][kk][row], ok ? (const void*)(V + (int64_t)col * t.r + row) : (const void*)V, ok);
    }
#pragma unroll
    for (int e = 0; e < XK * O / 128; ++e) {
      const int idx = tid + 128 * e;
      const int p = idx / XK, kk = idx % XK, col = k0 + kk;
      const int64_t so = soff[p];
      const bool ok = so >= 0 && col < t.T;
      cp_async8(&sS[buf][kk][p], ok ? (const void*)(src + so + col) : (const void*)src, ok);
    }
    cp_async_commit();
  };
  float2 acc[2][8];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = make_float2(0.f, 0.f);
  issue(0, 0);
  static_assert(MR1 == 1 || MR1 == 2, "phase-1 rows");
  int buf = 0;
  for (int k0 = 0; k0 < t.T; k0 += XK) {
    if (k0 + XK < t.T) {
      issue(buf ^ 1, k0 + XK);
      cp_async_wait_1();
    } else {
      cp_async_wait_0();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < XK; ++kk) {
      float2 m[MR1], sv[8];
#pragma unroll
      for (int i = 0; i < MR1; ++i) m[i] = sM[buf][kk][tr + 16 * i];
#pragma unroll
      for (int j = 0; j < 8; ++j) sv[j] = sS[buf][kk][to + 8 * j];
#pragma unroll
      for (int i = 0; i < MR1; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          acc[i][j].x = fmaf(m[i].x, sv[j].x, fmaf(-m[i].y, sv[j].y, acc[i][j].x));
          acc[i][j].y = fmaf(m[i].x, sv[j].y, fmaf(m[i].y, sv[j].x, acc[i][j].y));
        }
    }
    __syncthreads();
    buf ^= 1;
  }
  // tmp[row][op] (rows ≥ r are zero because V̂ rows ≥ r were zero-filled)
#pragma unroll
  for (int i = 0; i < MR1; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) tmp[tr + 16 * i][to + 8 * j] = acc[i][j];
  __syncthreads();
  for (int r0 = 0; r0 < t.T; r0 += R) {
    for (int idx = tid; idx < R * R; idx += 128) {   // sU[row][c] = Û[r0 + row, c]
      const int c = idx / R, row = idx % R;
      sU[row][c] = (r0 + row < t.T && c < t.r) ? __ldg(U + (int64_t)c * t.T + r0 + row) : make_float2(0.f, 0.f);
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = make_float2(0.f, 0.f);
#pragma unroll 4
    for (int c = 0; c < t.r; ++c) {
      float2 m[2], sv[8];
#pragma unroll
      for (int i = 0; i < 2; ++i) m[i] = sU[tr + 16 * i][c];
#pragma unroll
      for (int j = 0; j < 8; ++j) sv[j] = tmp[c][to + 8 * j];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          acc[i][j].x = fmaf(m[i].x, sv[j].x, fmaf(-m[i].y, sv[j].y, acc[i][j].x));
          acc[i][j].y = fmaf(m[i].x, sv[j].y, fmaf(m[i].y, sv[j].x, acc[i][j].y));
        }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int op = to + 8 * j;
      if (op >= t.op_count) continue;
      float2* d = dst + dst_off[t.op_begin + op] + r0;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int row = tr + 16 * i;
        if (r0 + row < t.T) atomicAdd(d + row, acc[i][j]);
      }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(128) k_m2l_lr(const LrTask* __restrict__ tasks, const int64_t* __restrict__ src_off,
                                                const int64_t* __restrict__ dst_off, const float2* __restrict__ pool,
                                                const float2* __restrict__ src, float2* __restrict__ dst) {
  __shared__ __align__(16) float2 sh[LR_SH];
  __shared__ int64_t soff[LR_O];
  const LrTask t = tasks[blockIdx.x];
  for (int p = threadIdx.x; p < LR_O; p += 128) soff[p] = p < t.op_count ? src_off[t.op_begin + p] : -1;
  __syncthreads();
  if (t.r <= 16) m2l_lr_body<1>(t, sh, soff, dst_off, pool, src, dst);
  else m2l_lr_body<2>(t, sh, soff, dst_off, pool, src, dst);
}

void launch_m2l_lr(int ntask, const LrTask* tasks, const int64_t* src_off, const int64_t* dst_off,
                   const float2* pool, const float2* src, float2* dst, cudaStream_t s) {
  if (ntask <= 0) return;
  k_m2l_lr<<<ntask, 128, 0, s>>>(tasks, src_off, dst_off, pool, src, dst);
}

// ------------------------------------------------------------------ GMRES helpers (a9)
// partial[c * nv + i] = Σ_{n ∈ chunk c} conj(V_i[n]) w[n]   (fp64 accumulation)
__global__ void k_dots(const float2* __restrict__ V, int64_t ldv, int nv, const float2* __restrict__ w, int64_t n,
                       double2* __restrict__ partial, int64_t chunk) {
  __shared__ double2 red[256];
  const int i = blockIdx.y, c = blockIdx.x;
  const int64_t b = (int64_t)c * chunk, e = min(n, b + chunk);
  const float2* v = V + (int64_t)i * ldv;
  double sr = 0, si = 0;
  for (int64_t j = b + threadIdx.x; j < e; j += blockDim.x) {
    float2 a = v[j], x = w[j];
    sr += (double)a.x * x.x + (double)a.y * x.y;
    si += (double)a.x * x.y - (double)a.y * x.x;
  }
  red[threadIdx.x] = make_double2(sr, si);
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      red[threadIdx.x].x += red[threadIdx.x + s].x;
      red[threadIdx.x].y += red[threadIdx.x + s].y;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[(int64_t)c * nv + i] = red[0];
}

void launch_dots(const float2* V, int64_t ldv, int nv, const float2* w, int64_t n, double2* partial, int nchunks,
                 cudaStream_t s) {
  int64_t chunk = (n + nchunks - 1) / nchunks;
  dim3 grid(nchunks, nv);
  k_dots<<<grid, 256, 0, s>>>(V, ldv, nv, w, n, partial, chunk);
}

// w[n] += sign * Σ_i V_i[n] h_i
__global__ void k_update(float2* __restrict__ w, const float2* __restrict__ V, int64_t ldv, int nv,
                         const double2* __restrict__ h, int64_t n, double sign) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double ar = 0, ai = 0;
  for (int i = 0; i < nv; ++i) {
    float2 v = V[(int64_t)i * ldv + j];
    double2 c = h[i];
    ar += (double)v.x * c.x - (double)v.y * c.y;
    ai += (double)v.x * c.y + (double)v.y * c.x;
  }
  float2 x = w[j];
  w[j] = make_float2((float)(x.x + sign * ar), (float)(x.y + sign * ai));
}
void launch_update(float2* w, const float2* V, int64_t ldv, int nv, const double2* h, int64_t n, double sign,
                   cudaStream_t s) {
  k_update<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(w, V, ldv, nv, h, n, sign);
}

__global__ void k_norm2(const float2* __restrict__ w, int64_t n, double* __restrict__ partial, int64_t chunk) {
  __shared__ double red[256];
  const int c = blockIdx.x;
  const int64_t b = (int64_t)c * chunk, e = min(n, b + chunk);
  double s = 0;
  for (int64_t j = b + threadIdx.x; j < e; j += blockDim.x) {
    float2 x = w[j];
    s += (double)x.x * x.x + (double)x.y * x.y;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int k = blockDim.x / 2; k > 0; k >>= 1) {
    if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[c] = red[0];
}
void launch_norm2(const float2* w, int64_t n, double* partial, int nchunks, cudaStream_t s) {
  int64_t chunk = (n + nchunks - 1) / nchunks;
  k_norm2<<<nchunks, 256, 0, s>>>(w, n, partial, chunk);
}

__global__ void k_reduce_partials(const double2* __restrict__ partial, int nv, int nchunks, double2* __restrict__ out) {
  const int i = blockIdx.x;
  __shared__ double2 red[128];
  double sr = 0, si = 0;
  for (int c = threadIdx.x; c < nchunks; c += blockDim.x) {
    double2 v = partial[(int64_t)c * nv + i];
    sr += v.x;
    si += v.y;
  }
  red[threadIdx.x] = make_double2(sr, si);
  __syncthreads();
  for (int k = blockDim.x / 2; k > 0; k >>= 1) {
    if (threadIdx.x < k) {
      red[threadIdx.x].x += red[threadIdx.x + k].x;
      red[threadIdx.x].y += red[threadIdx.x + k].y;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[i] = red[0];
}
void launch_reduce_partials(const double2* partial, int nv, int nchunks, double2* out, cudaStream_t s) {
  k_reduce_partials<<<nv, 128, 0, s>>>(partial, nv, nchunks, out);
}

__global__ void k_reduce_norm(const double* __restrict__ partial, int nchunks, double* __restrict__ out) {
  __shared__ double red[128];
  double a = 0;
  for (int c = threadIdx.x; c < nchunks; c += blockDim.x) a += partial[c];
  red[threadIdx.x] = a;
  __syncthreads();
  for (int k = blockDim.x / 2; k > 0; k >>= 1) {
    if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = sqrt(red[0]);
}
void launch_reduce_norm(const double* partial, int nchunks, double* out, cudaStream_t s) {
  k_reduce_norm<<<1, 128, 0, s>>>(partial, nchunks, out);
}

__global__ void k_scale_by_inv(float2* dst, const float2* src, const double* __restrict__ nrm, int64_t n) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double v = nrm[0];
  const double inv = v > 0 ? 1.0 / v : 0.0;
  float2 x = src[j];
  dst[j] = make_float2((float)(x.x * inv), (float)(x.y * inv));
}
void launch_scale_by_inv(float2* dst, const float2* src, const double* nrm, int64_t n, cudaStream_t s) {
  k_scale_by_inv<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(dst, src, nrm, n);
}

__global__ void k_scale(float2* dst, const float2* src, double sre, double sim, int64_t n) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  float2 x = src[j];
  dst[j] = make_float2((float)(x.x * sre - x.y * sim), (float)(x.x * sim + x.y * sre));
}
void launch_scale(float2* dst, const float2* src, double sre, double sim, int64_t n, cudaStream_t s) {
  k_scale<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(dst, src, sre, sim, n);
}

__global__ void k_axpby(float2* y, const float2* x, double a, double b, int64_t n) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  float2 u = x[j], v = y[j];
  y[j] = make_float2((float)(a * u.x + b * v.x), (float)(a * u.y + b * v.y));
}
void launch_axpby(float2* y, const float2* x, double a, double b, int64_t n, cudaStream_t s) {
  k_axpby<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(y, x, a, b, n);
}

// b_i = e^{ik d·x_i} (1 + iαk d·n_i)   (Eq. 4 right side, ∂u/∂n = 0, reading C22)
__global__ void k_plane_wave(const double* __restrict__ cen, const double* __restrict__ nrm,
                             const int32_t* __restrict__ perm, int n, double k, double are, double aim, double dx,
                             double dy, double dz, float2* b32, double2* b64) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double ph = k * (dx * cen[3 * i] + dy * cen[3 * i + 1] + dz * cen[3 * i + 2]);
  double dn = dx * nrm[3 * i] + dy * nrm[3 * i + 1] + dz * nrm[3 * i + 2];
  double s, c;
  sincos(ph, &s, &c);
  // 1 + i α k dn  with α = are + i aim
  double fr = 1.0 - aim * k * dn, fi = are * k * dn;
  double br = c * fr - s * fi, bi = c * fi + s * fr;
  int j = perm[i];
  if (b32) b32[j] = make_float2((float)br, (float)bi);
  if (b64) b64[j] = make_double2(br, bi);
}
void launch_plane_wave(const double* cen, const double* nrm, const int32_t* perm, int n, double k, double are,
                       double aim, double dx, double dy, double dz, float2* b32, double2* b64, cudaStream_t s) {
  k_plane_wave<<<(n + 255) / 256, 256, 0, s>>>(cen, nrm, perm, n, k, are, aim, dx, dy, dz, b32, b64);
}

__global__ void k_f64_to_f32(const double2* a, float2* b, int64_t n) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) b[j] = make_float2((float)a[j].x, (float)a[j].y);
}
__global__ void k_f32_to_f64(const float2* a, double2* b, int64_t n) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) b[j] = make_double2(a[j].x, a[j].y);
}
void launch_f64_to_f32(const double2* a, float2* b, int64_t n, cudaStream_t s) {
  k_f64_to_f32<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, b, n);
}
void launch_f32_to_f64(const float2* a, double2* b, int64_t n, cudaStream_t s) {
  k_f32_to_f64<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, b, n);
}

}  // namespace fda
