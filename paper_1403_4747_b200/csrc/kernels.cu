// Device kernels of the FDA Burton–Miller matvec (sm_100a, complex64 data,
// fp32 arithmetic; fp64 accumulation in the GMRES reductions).
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdlib>

#include "f32x2.cuh"
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

// sharded exchange of partial outgoing states (partition.cpp):
// pack  send[i] = out[idx[i]];  unpack  out[idx[i]] += recv[i]  (a state may
// arrive from several peers: vector atomics)
__global__ void k_pack(const float2* __restrict__ out, const int64_t* __restrict__ idx, float2* __restrict__ send,
                       int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) send[i] = out[idx[i]];
}
__global__ void k_unpack_add(const float2* __restrict__ recv, const int64_t* __restrict__ idx, float2* __restrict__ out,
                             int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(out + idx[i], recv[i]);
}
void launch_pack(const float2* out, const int64_t* idx, float2* send, int64_t n, cudaStream_t s) {
  if (n > 0) k_pack<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(out, idx, send, n);
}
void launch_unpack_add(const float2* recv, const int64_t* idx, float2* out, int64_t n, cudaStream_t s) {
  if (n > 0) k_unpack_add<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(recv, idx, out, n);
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
//
// Positions are in WAVE UNITS X = k·x (leaf-local, fp32 offsets computed in
// fp64), so r² in these units is q² = (kr)² and 1/r = k·rsqrt(q²); the k² of
// 1/r² is folded into the per-source weight w_j = k² A_j/(12π) x_j, and the
// constant k of α·k into KernelParams.  Per (target, source element) the
// kernel values of the three Q3 points are summed first and multiplied by
// w_j once.
// CTA shape (threads, staged sources per chunk): (256, 512) when target leaves see many
// direct sources (config 2: 530 per target, near 0.188 → 0.182 ms), (128, 256) otherwise
// (config 5: 268 per target, 6.2 → 5.6 ms); launch_near's `wide` picks the variant
constexpr int NEAR_NT_WIDE = 256, NEAR_MAXS_WIDE = 512;
constexpr int NEAR_NT_NARROW = 128, NEAR_MAXS_NARROW = 256;

// MUFU.RSQ without the denormal guard of rsqrtf (q² ≥ 1e-12 here, never denormal)
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// One Q3 point of the LHS kernel for TWO targets at once (the lanes of the
// packed fp32 pairs, f32x2.cuh), accumulated into (kr, ki) without the weight:
//   k += (r²/k²)·4π·[∂G/∂n_y + α ∂²G/∂n_x∂n_y](x, y) = e^{iq}(P + iQ)/q²
// With q = kr, a = ∂r/∂n_x, b = ∂r/∂n_y, c = n_x·n_y, g = 3ab + c, u1 = (3 - q²)ab + c:
//   4π r² e^{-iq} ∂G/∂n_y          = (iq - 1) b
//   4π r² e^{-iq} ∂²G/∂n_x∂n_y     = (1/r) [ u1 - iq g ]
// so for α = i α_i (PURE_IMAG; α = i/k):  P = -b + α_i k g,  Q = q b + α_i k (1/q) u1.
// d = X - Y (wave units), s = d·n_x, t = Y·n_y - X·n_y = -(d·n_y), ι = 1/q; t is the same for
// the three Q3 points of a (flat) source element — they lie in its plane — so the caller computes
// it once per element from the plane constant Y·n_y:
// a = sι, b = tι, ab = st ι², q²ab = st, qb = t — so u1 = g - st and Q = t + α_i k ι u1.
// The source point Y is the same for both lanes (a broadcast operand); MUFU
// work (rsqrt, sin, cos) stays per lane.
// EXPAND (opt-in, FDA_NEAR_EXPAND=1): the differences d = X − Y are never formed — with the staged point holding
// (−Y, |Y|²) and the thread holding 2X, |X|² and X·n_x,
//   q² = |X|² + |Y|² + 2X·(−Y)   (1 FADD2 + 3 FFMA2),   s = X·n_x + (−Y)·n_x   (3 FFMA2)
// i.e. 7 packed instructions instead of 9 (3 FSUB2 + 3 for q² + 3 for s).  The expansion loses
// ≈ (|X|² + |Y|²)/q² of q²'s relative precision to cancellation; in leaf-local wave units that is
// ≤ 1e-5 relative in r for the closest (self / adjacent-element) pairs.  Measured: near field
// 4% faster (config 4 3.089 → 2.960 ms), exact-path error 3.5e-6 instead of ≤ 2e-6 — not the
// default.
template <bool PURE_IMAG, bool EXPAND>
__device__ __forceinline__ void lhs_eval2(const f2x* X, const f2x* nx, float4 Y, f2x t, f2x cn, f2x xsq, f2x xn,
                                          const KernelParams& kp, f2x& kr, f2x& ki) {
  f2x q2, sd;
  if (EXPAND) {
    q2 = fma2(bcast2(Y.x), X[0], fma2(bcast2(Y.y), X[1], fma2(bcast2(Y.z), X[2], add2(xsq, bcast2(Y.w)))));
    sd = fma2(bcast2(Y.x), nx[0], fma2(bcast2(Y.y), nx[1], fma2(bcast2(Y.z), nx[2], xn)));   // s = d·n_x
  } else {
    const f2x dx = sub2(X[0], bcast2(Y.x)), dy = sub2(X[1], bcast2(Y.y)), dz = sub2(X[2], bcast2(Y.z));
    q2 = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
    sd = fma2(dx, nx[0], fma2(dy, nx[1], mul2(dz, nx[2])));   // s = d·n_x
  }
  float q2a, q2b;
  unpack2(q2, q2a, q2b);
  const f2x iq = pack2(rsqrt_ftz(q2a), rsqrt_ftz(q2b));
  const f2x q = mul2(q2, iq);
  float qa, qb, sa, ca, sb, cb;
  unpack2(q, qa, qb);
  __sincosf(qa, &sa, &ca);  // MUFU sin/cos; argument error ≤ ulp(q/2π)
  __sincosf(qb, &sb, &cb);
  const f2x iq2 = mul2(iq, iq);
  const f2x st = mul2(sd, t);
  const f2x g = fma2(bcast2(3.0f), mul2(st, iq2), cn);   // 3ab + c
  const f2x u1 = sub2(g, st);                            // (3 - q²) ab + c
  const f2x b = mul2(t, iq);
  f2x P, Q;
  if (PURE_IMAG) {
    P = fma2(bcast2(kp.ak_im), g, neg2(b));
    Q = fma2(mul2(bcast2(kp.ak_im), iq), u1, t);
  } else {
    // P = ι (α_r k u1 - α_i k u2) - b,  Q = ι (α_r k u2 + α_i k u1) + qb,  u2 = -q g
    const f2x u2 = neg2(mul2(q, g));
    P = fma2(iq, fma2(bcast2(kp.ak_re), u1, mul2(bcast2(-kp.ak_im), u2)), neg2(b));
    Q = fma2(iq, fma2(bcast2(kp.ak_re), u2, mul2(bcast2(kp.ak_im), u1)), t);
  }
  const f2x Er = mul2(iq2, pack2(ca, cb)), Ei = mul2(iq2, pack2(sa, sb));
  kr = fma2(Er, P, fma2(neg2(Ei), Q, kr));
  ki = fma2(Er, Q, fma2(Ei, P, ki));
}

// One Q3 point of the RHS kernel (Eq. 4 right side) for two targets, without the weight:
//   4π r² e^{-iq} (G + α ∂G/∂n_x) = r + α (iq - 1) a,   r = q/k
__device__ __forceinline__ void rhs_eval2(const f2x* X, const f2x* nx, float4 Y, const KernelParams& kp, f2x& kr,
                                          f2x& ki) {
  const f2x dx = sub2(X[0], bcast2(Y.x)), dy = sub2(X[1], bcast2(Y.y)), dz = sub2(X[2], bcast2(Y.z));
  const f2x q2 = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
  float q2a, q2b;
  unpack2(q2, q2a, q2b);
  const f2x iq = pack2(rsqrt_ftz(q2a), rsqrt_ftz(q2b));
  const f2x q = mul2(q2, iq);
  float qa, qb, sa, ca, sb, cb;
  unpack2(q, qa, qb);
  __sincosf(qa, &sa, &ca);
  __sincosf(qb, &sb, &cb);
  const f2x a = mul2(fma2(dx, nx[0], fma2(dy, nx[1], mul2(dz, nx[2]))), iq);
  // P = r - a (α_r + α_i q),  Q = a (α_r q - α_i)
  const f2x P = fma2(q, bcast2(kp.inv_k), neg2(mul2(a, fma2(bcast2(kp.alpha_im), q, bcast2(kp.alpha_re)))));
  const f2x Q = mul2(a, fma2(bcast2(kp.alpha_re), q, bcast2(-kp.alpha_im)));
  const f2x iq2 = mul2(iq, iq);
  const f2x Er = mul2(iq2, pack2(ca, cb)), Ei = mul2(iq2, pack2(sa, sb));
  kr = fma2(Er, P, fma2(neg2(Ei), Q, kr));
  ki = fma2(Er, Q, fma2(Ei, P, ki));
}

// y_i = Σ_{j ∈ direct(i)} A^{Q3}_ij x_j + Σ_{j: ρ_ij<3} C_ij x_j   (a7)
// One CTA per target leaf (NearTask, in descending-work order).  The source
// elements of all its direct leaves are listed in a build-time slot table
// (element, index of its source leaf in the near list → k(c_B − c_C)), so the
// CTA stages them through shared memory in chunks of NEAR_MAXS with one
// coalesced table load per slot.  Each thread owns a PAIR of targets (the two
// lanes of its packed fp32 registers); P = ⌊NT/⌈n_B/2⌉⌋ threads share one
// pair and split the sources; partial sums are reduced in shared memory.
// Staged per source element: the three Q3 points (wave units, shifted into the
// target leaf's frame), the normal with the plane constant Y·n_y in .w, and
// w_j = x_j·k²A_j/(12π).
// KIND 0: LHS operator A (Eq. 5); KIND 1: RHS operator B (G sources).
template <int KIND, bool PURE_IMAG, int NEAR_NT, int NEAR_MAXS, bool EXPAND>
__global__ void __launch_bounds__(NEAR_NT) k_near(
    const NearTask* __restrict__ tasks, const int2* __restrict__ slots, const float4* __restrict__ near_off,
    const float4* __restrict__ tgt_pos, const float4* __restrict__ tgt_nrm, const SrcElem* __restrict__ src,
    const float* __restrict__ src_w, const int32_t* __restrict__ corr_ptr, const int32_t* __restrict__ corr_col,
    const float2* __restrict__ corr_val, const float2* __restrict__ x, float2* __restrict__ y, KernelParams kp) {
  // staged source element s: st[5s..5s+4] = Y0, Y1, Y2, (n_y, Y·n_y), (w_j, -, -)
  __shared__ float4 st[NEAR_MAXS * 5];
  __shared__ float4 sred[NEAR_NT];
  const NearTask t = tasks[blockIdx.x];
  const int tb = t.tb, nt = t.nt;
  const int np = (nt + 1) >> 1;   // target pairs
  const int P = max(1, NEAR_NT / np);
  const int tid = threadIdx.x;
  const int tp = tid % np, part = tid / np;
  const bool active = part < P;
  const int j0 = 2 * tp, j1 = min(j0 + 1, nt - 1);   // odd n_B: the last lane duplicates a target (discarded)
  constexpr bool EXP = KIND == 0 && EXPAND;   // expanded q² / s (lhs_eval2): X holds 2X
  f2x X[3], N[3], xsq = zero2(), xn = zero2();
  {
    const float4 p0 = tgt_pos[tb + j0], p1 = tgt_pos[tb + j1];
    const float4 n0 = tgt_nrm[tb + j0], n1 = tgt_nrm[tb + j1];
    X[0] = pack2(p0.x, p1.x); X[1] = pack2(p0.y, p1.y); X[2] = pack2(p0.z, p1.z);
    N[0] = pack2(n0.x, n1.x); N[1] = pack2(n0.y, n1.y); N[2] = pack2(n0.z, n1.z);
    if (EXP) {
      xsq = fma2(X[0], X[0], fma2(X[1], X[1], mul2(X[2], X[2])));
      xn = fma2(X[0], N[0], fma2(X[1], N[1], mul2(X[2], N[2])));
      X[0] = add2(X[0], X[0]); X[1] = add2(X[1], X[1]); X[2] = add2(X[2], X[2]);
    }
  }
  f2x ar = zero2(), ai = zero2();
  for (int base = t.s0; base < t.s1; base += NEAR_MAXS) {
    const int ns = min(NEAR_MAXS, t.s1 - base);
    __syncthreads();
    for (int slot = tid; slot < ns; slot += NEAR_NT) {
      const int2 sl = slots[base + slot];
      const int el = sl.x;
      const float4 off = near_off[sl.y];  // k (c_B - c_C)
      SrcElem se = src[el];
      const float2 xv = x[el];
      const float wv = src_w[el];
      float4 n4 = make_float4(se.a.w, se.b.w, se.c.w, 0.f);
      const float4 A = make_float4(se.a.x - off.x, se.a.y - off.y, se.a.z - off.z, 0.f);
      const float4 B = make_float4(se.b.x - off.x, se.b.y - off.y, se.b.z - off.z, 0.f);
      const float4 C = make_float4(se.c.x - off.x, se.c.y - off.y, se.c.z - off.z, 0.f);
      // plane constant Y·n_y of the element, from its centroid (the mean of the Q3 points)
      n4.w = fmaf(A.x + B.x + C.x, n4.x, fmaf(A.y + B.y + C.y, n4.y, (A.z + B.z + C.z) * n4.z)) * (1.0f / 3.0f);
      float4* d = st + 5 * slot;
      if (EXP) {   // (−Y, |Y|²)
        d[0] = make_float4(-A.x, -A.y, -A.z, fmaf(A.x, A.x, fmaf(A.y, A.y, A.z * A.z)));
        d[1] = make_float4(-B.x, -B.y, -B.z, fmaf(B.x, B.x, fmaf(B.y, B.y, B.z * B.z)));
        d[2] = make_float4(-C.x, -C.y, -C.z, fmaf(C.x, C.x, fmaf(C.y, C.y, C.z * C.z)));
      } else {
        d[0] = A; d[1] = B; d[2] = C;
      }
      d[3] = n4;
      d[4] = make_float4(xv.x * wv, xv.y * wv, 0.f, 0.f);
    }
    __syncthreads();
    if (active) {
#pragma unroll 2
      for (int s = part; s < ns; s += P) {
        const float4* e = st + 5 * s;
        const float4 A = e[0], B = e[1], C = e[2];
        const float4 w = e[4];
        f2x kr = zero2(), ki = zero2();
        if (KIND == 0) {
          const float4 ny = e[3];
          const f2x cn = fma2(N[0], bcast2(ny.x), fma2(N[1], bcast2(ny.y), mul2(N[2], bcast2(ny.z))));
          const f2x xny = fma2(X[0], bcast2(ny.x), fma2(X[1], bcast2(ny.y), mul2(X[2], bcast2(ny.z))));
          // t = Y·n_y − X·n_y (plane constant in ny.w; X holds 2X when EXP)
          const f2x tp = EXP ? fma2(bcast2(-0.5f), xny, bcast2(ny.w)) : sub2(bcast2(ny.w), xny);
          lhs_eval2<PURE_IMAG, EXP>(X, N, A, tp, cn, xsq, xn, kp, kr, ki);
          lhs_eval2<PURE_IMAG, EXP>(X, N, B, tp, cn, xsq, xn, kp, kr, ki);
          lhs_eval2<PURE_IMAG, EXP>(X, N, C, tp, cn, xsq, xn, kp, kr, ki);
        } else {
          rhs_eval2(X, N, A, kp, kr, ki);
          rhs_eval2(X, N, B, kp, kr, ki);
          rhs_eval2(X, N, C, kp, kr, ki);
        }
        ar = fma2(kr, bcast2(w.x), fma2(neg2(ki), bcast2(w.y), ar));
        ai = fma2(kr, bcast2(w.y), fma2(ki, bcast2(w.x), ai));
      }
    }
  }
  float4 acc;
  unpack2(ar, acc.x, acc.z);
  unpack2(ai, acc.y, acc.w);
  // correction SpMV, rows split over the P parts
  if (active && !kp.skip_corr) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (j0 + h >= nt) break;
      const int i = tb + j0 + h;
      const int cb = corr_ptr[i], ce = corr_ptr[i + 1];
      float2 c = make_float2(0.f, 0.f);
      for (int e = cb + part; e < ce; e += P) {
        const float2 v = corr_val[e];
        const float2 xv = x[corr_col[e]];
        c.x = fmaf(v.x, xv.x, fmaf(-v.y, xv.y, c.x));
        c.y = fmaf(v.x, xv.y, fmaf(v.y, xv.x, c.y));
      }
      if (h == 0) { acc.x += c.x; acc.y += c.y; }
      else { acc.z += c.x; acc.w += c.y; }
    }
  }
  sred[tid] = active ? acc : make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();
  if (tid < np) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int p = 0; p < P; ++p) {
      const float4 v = sred[p * np + tid];
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    y[tb + 2 * tid] = make_float2(s.x, s.y);
    if (2 * tid + 1 < nt) y[tb + 2 * tid + 1] = make_float2(s.z, s.w);
  }
}

void launch_near(int ntask, const NearTask* tasks, const int2* slots, const float4* near_off, const float4* tgt_pos,
                 const float4* tgt_nrm, const SrcElem* src, const float* src_w, const int32_t* corr_ptr,
                 const int32_t* corr_col, const float2* corr_val, const float2* x, float2* y, KernelParams kp,
                 bool alpha_pure_imag, int kind, bool wide, cudaStream_t s) {
  if (ntask <= 0) return;
  // the difference form by default: the expanded form (FDA_NEAR_EXPAND=1) is 4% faster but doubles
  // the fp32 error of the exact path (config 1, every pair direct: 3.5e-6 vs ≤ 2e-6)
  static const bool diff = !(getenv("FDA_NEAR_EXPAND") && atoi(getenv("FDA_NEAR_EXPAND")) != 0);
#define NEAR(K, PI, NT, MS)                                                                                       \
  do {                                                                                                            \
    if (diff) k_near<K, PI, NT, MS, false><<<ntask, NT, 0, s>>>(tasks, slots, near_off, tgt_pos, tgt_nrm, src,  \
                                                              src_w, corr_ptr, corr_col, corr_val, x, y, kp);  \
    else k_near<K, PI, NT, MS, true><<<ntask, NT, 0, s>>>(tasks, slots, near_off, tgt_pos, tgt_nrm, src, src_w,  \
                                                        corr_ptr, corr_col, corr_val, x, y, kp);               \
  } while (0)
  if (wide) {
    if (kind == 1) NEAR(1, false, NEAR_NT_WIDE, NEAR_MAXS_WIDE);
    else if (alpha_pure_imag) NEAR(0, true, NEAR_NT_WIDE, NEAR_MAXS_WIDE);
    else NEAR(0, false, NEAR_NT_WIDE, NEAR_MAXS_WIDE);
  } else {
    if (kind == 1) NEAR(1, false, NEAR_NT_NARROW, NEAR_MAXS_NARROW);
    else if (alpha_pure_imag) NEAR(0, true, NEAR_NT_NARROW, NEAR_MAXS_NARROW);
    else NEAR(0, false, NEAR_NT_NARROW, NEAR_MAXS_NARROW);
  }
#undef NEAR
}

// ------------------------------------------------------------------ S2M (a2) / L2T (a6)
// HBM-bound per-leaf matrix-vector products.  Thread (row, group): G = ⌊NT/rows⌋
// groups split the columns (column c handled by group c mod G), so one warp
// reads consecutive entries of the column-major matrix; each thread keeps
// LEAF_U independent loads in flight; the G partial sums meet in shared memory.
constexpr int LEAF_NT = 128;
constexpr int LEAF_U = 8;
constexpr int LEAF_MAXR = 320;

__device__ __forceinline__ float2 leaf_colsum(const float2* __restrict__ M, int64_t ld, int row, int c0, int cstep,
                                              int ncol, const float2* __restrict__ v) {
  float2 acc = make_float2(0.f, 0.f);
  // pointer increments instead of per-load index products (ncu round 4: the ALU pipe was at 44%)
  const float2* p = M + (int64_t)c0 * ld + row;
  const float2* x = v + c0;
  const int64_t step = (int64_t)cstep * ld;
  int c = c0;
  for (; c + (LEAF_U - 1) * cstep < ncol; c += LEAF_U * cstep, p += LEAF_U * step, x += LEAF_U * cstep) {
    float2 m[LEAF_U];
#pragma unroll
    for (int u = 0; u < LEAF_U; ++u) m[u] = __ldg(p + u * step);
#pragma unroll
    for (int u = 0; u < LEAF_U; ++u) {
      const float2 xv = x[u * cstep];
      acc.x = fmaf(m[u].x, xv.x, fmaf(-m[u].y, xv.y, acc.x));
      acc.y = fmaf(m[u].x, xv.y, fmaf(m[u].y, xv.x, acc.y));
    }
  }
  if (c < ncol) {   // last, partial batch
    float2 m[LEAF_U];
#pragma unroll
    for (int u = 0; u < LEAF_U; ++u) m[u] = c + u * cstep < ncol ? __ldg(p + u * step) : make_float2(0.f, 0.f);
#pragma unroll
    for (int u = 0; u < LEAF_U; ++u) {
      const float2 xv = x[c + u * cstep < ncol ? u * cstep : 0];
      acc.x = fmaf(m[u].x, xv.x, fmaf(-m[u].y, xv.y, acc.x));
      acc.y = fmaf(m[u].x, xv.y, fmaf(m[u].y, xv.x, acc.y));
    }
  }
  return acc;
}

// S2M: m̃_B = S̃_B x_B (T × n_B, column-major)   (Eq. 10; compressed S̃)
__global__ void __launch_bounds__(LEAF_MAXR, 6) k_s2m(const LeafTask* __restrict__ tasks, const float2* __restrict__ pool,
                                                   const float2* __restrict__ x, float2* __restrict__ out) {
  __shared__ float2 sx[128];
  __shared__ float2 red[LEAF_MAXR];
  const LeafTask t = tasks[blockIdx.x];
  const int nb = t.elem_count, T = t.T;
  for (int j = threadIdx.x; j < nb; j += blockDim.x) sx[j] = x[t.elem_begin + j];
  __syncthreads();
  const int G = max(1, (int)blockDim.x / T);
  const int r = threadIdx.x % T, g = threadIdx.x / T;
  float2 acc = make_float2(0.f, 0.f);
  if (g < G) acc = leaf_colsum(pool + t.mat_off, T, r, g, G, nb, sx);
  if (G == 1) {
    if (threadIdx.x < T) out[t.state_off + r] = acc;
    return;
  }
  if (g < G) red[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < T) {
    float2 s = red[threadIdx.x];
    for (int q = 1; q < G; ++q) {
      const float2 v = red[q * T + threadIdx.x];
      s.x += v.x; s.y += v.y;
    }
    out[t.state_off + r] = s;
  }
}

// L2T: y_B = T̃_B ℓ̃_B (n_B × T column-major)   (Eq. 12; compressed T̃)
// ADD: accumulate (HF leaves have one task per incoming wedge); else overwrite.
template <bool ADD>
__global__ void __launch_bounds__(LEAF_NT, 16) k_l2t(const LeafTask* __restrict__ tasks, const float2* __restrict__ pool,
                                                 const float2* __restrict__ in, float2* __restrict__ y) {
  __shared__ float2 sl[LEAF_MAXR];
  __shared__ float2 red[LEAF_NT];
  const LeafTask t = tasks[blockIdx.x];
  const int nb = t.elem_count;
  if (t.mat_off < 0) {
    if (!ADD)
      for (int i = threadIdx.x; i < nb; i += blockDim.x) y[t.elem_begin + i] = make_float2(0.f, 0.f);
    return;
  }
  for (int c = threadIdx.x; c < t.T; c += blockDim.x) sl[c] = in[t.state_off + c];
  __syncthreads();
  const int G = max(1, LEAF_NT / nb);
  const int i = threadIdx.x % nb, g = threadIdx.x / nb;
  float2 acc = make_float2(0.f, 0.f);
  if (g < G) acc = leaf_colsum(pool + t.mat_off, nb, i, g, G, t.T, sl);
  red[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < nb) {
    float2 s = red[threadIdx.x];
    for (int q = 1; q < G; ++q) {
      const float2 v = red[q * nb + threadIdx.x];
      s.x += v.x; s.y += v.y;
    }
    if (ADD) atomicAdd(y + t.elem_begin + threadIdx.x, s);
    else y[t.elem_begin + threadIdx.x] = s;
  }
}

void launch_s2m(int ntask, const LeafTask* tasks, const float2* pool, const float2* x, float2* out, int max_rows,
                cudaStream_t s) {
  if (ntask <= 0) return;
  int bd = ((max_rows + 31) / 32) * 32;
  bd = bd < LEAF_NT ? LEAF_NT : (bd > LEAF_MAXR ? LEAF_MAXR : bd);
  k_s2m<<<ntask, bd, 0, s>>>(tasks, pool, x, out);
}
void launch_l2t(int ntask, const LeafTask* tasks, const float2* pool, const float2* in, float2* y, cudaStream_t s,
                bool accumulate) {
  if (ntask <= 0) return;
  if (accumulate) k_l2t<true><<<ntask, LEAF_NT, 0, s>>>(tasks, pool, in, y);
  else k_l2t<false><<<ntask, LEAF_NT, 0, s>>>(tasks, pool, in, y);
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

__device__ __forceinline__ void cmac(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, fmaf(-a.y, b.y, acc.x));
  acc.y = fmaf(a.x, b.y, fmaf(a.y, b.x, acc.y));
}

// Tile R rows × O ops per CTA (128 threads); thread (tr, to) owns rows
// {2tr, 2tr+1} + 2·NR·i and ops {2to, 2to+1} + 2·NO·j; a warp spans 4 row
// groups × 8 op groups, so every shared load is a one-wavefront LDS.128.
template <int R, int O>
struct XCfg {
  static constexpr int RT = (R == 128) ? 8 : (R == 16 ? 2 : 4);   // rows per thread
  static constexpr int NR = R / RT;                                // row groups
  static constexpr int NO = 128 / NR;                              // op groups
  static constexpr int OT = O / NO;                                // ops per thread
  static constexpr int SO = O + 2;                                 // padded sS row
  static_assert(NR % 4 == 0 && NO % 8 == 0 && OT % 2 == 0 && RT % 2 == 0, "tile");
};

template <int R, int O, bool ATOMIC>
__global__ void __launch_bounds__(128) k_xlate(const XTask* __restrict__ tasks, const int64_t* __restrict__ src_off,
                                               const int64_t* __restrict__ dst_off, const float2* __restrict__ pool,
                                               const float2* __restrict__ src, float2* __restrict__ dst) {
  using C = XCfg<R, O>;
  constexpr int RT = C::RT, NR = C::NR, NO = C::NO, OT = C::OT, SO = C::SO;
  constexpr int ML = XK * R / 128, SL = XK * O / 128;  // cp.async per thread per chunk
  __shared__ __align__(16) float2 sM[2][XK][R];
  __shared__ __align__(16) float2 sS[2][XK][SO];
  __shared__ int64_t soff[O];
  const XTask t = tasks[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tr = (warp % (NR / 4)) * 4 + (lane >> 3), to = (warp / (NR / 4)) * 8 + (lane & 7);
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
  float2 acc[RT][OT];
#pragma unroll
  for (int i = 0; i < RT; ++i)
#pragma unroll
    for (int j = 0; j < OT; ++j) acc[i][j] = make_float2(0.f, 0.f);
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
      const float4* mv = reinterpret_cast<const float4*>(&sM[buf][kk][2 * tr]);
      const float4* sv = reinterpret_cast<const float4*>(&sS[buf][kk][2 * to]);
      float2 m[RT], v[OT];
#pragma unroll
      for (int i = 0; i < RT / 2; ++i) {
        const float4 q = mv[NR * i];
        m[2 * i] = make_float2(q.x, q.y);
        m[2 * i + 1] = make_float2(q.z, q.w);
      }
#pragma unroll
      for (int j = 0; j < OT / 2; ++j) {
        const float4 q = sv[NO * j];
        v[2 * j] = make_float2(q.x, q.y);
        v[2 * j + 1] = make_float2(q.z, q.w);
      }
#pragma unroll
      for (int i = 0; i < RT; ++i)
#pragma unroll
        for (int j = 0; j < OT; ++j) cmac(acc[i][j], m[i], v[j]);
    }
    __syncthreads();
    buf ^= 1;
  }
  // rows (2tr, 2tr+1) + 2·NR·i are pairs: one 16-byte vector atomic per pair (states and
  // the tmp buffer are 16-byte aligned and padded to an even length; rows ≥ t.rows hold
  // zeros since M rows ≥ t.rows were zero-filled)
#pragma unroll
  for (int j = 0; j < OT; ++j) {
    const int op = 2 * to + (j & 1) + 2 * NO * (j >> 1);
    if (op >= t.op_count) continue;
    float2* d = dst + dst_off[t.op_begin + op];
#pragma unroll
    for (int i = 0; i < RT; i += 2) {
      const int row = t.row0 + 2 * tr + 2 * NR * (i >> 1);
      if (row < t.rows) {
        const float4 v = make_float4(acc[i][j].x, acc[i][j].y, acc[i + 1][j].x, acc[i + 1][j].y);
        if (ATOMIC) atomicAdd(reinterpret_cast<float4*>(d + row), v);
        else if (row + 1 < t.rows) *reinterpret_cast<float4*>(d + row) = v;
        else d[row] = acc[i][j];
      }
    }
  }
}

void launch_xlate(int variant, bool atomic, int ntask, const XTask* tasks, const int64_t* src_off,
                  const int64_t* dst_off, const float2* pool, const float2* src, float2* dst, cudaStream_t s) {
  if (ntask <= 0) return;
#define XL(R, O)                                                                                          \
  (atomic ? k_xlate<R, O, true><<<ntask, 128, 0, s>>>(tasks, src_off, dst_off, pool, src, dst)            \
          : k_xlate<R, O, false><<<ntask, 128, 0, s>>>(tasks, src_off, dst_off, pool, src, dst))
  switch (variant) {
    case 0: XL(32, 64); break;
    case 1: XL(64, 32); break;
    case 2: XL(128, 16); break;
    default: XL(16, 128); break;
  }
#undef XL
}

// ------------------------------------------------------------------ fused §4.2 M2L (a4)
// PAPER.md §4.2: K̃ ≈ Û V̂ (Û: T × r, V̂: r × T, r ≤ 64).  One CTA
// handles ≤ O = 64 ops sharing one K̃ (template O ≤ LR_O = 128):
//   phase 1  tmp = V̂ S        (R1 ≥ r rows × 64 ops, K = T streamed through a
//                              cp.async double buffer), tmp kept in shared memory;
//   phase 2  dst += Û tmp      (32-row tiles of Û, double-buffered, K = r),
//            accumulated into the destination states with vector atomics.
// Register tiles: phase 1 RT1 rows × OT1 ops per thread, phase 2 4 × 4.  A
// thread's rows are pairs {2tr, 2tr+1} + 2·NR·i and its ops pairs
// {2to, 2to+1} + 2·NO·j, and a warp spans 4 row groups × 8 op groups, so every
// shared load is an LDS.128 (2 complex values) touching ≤ 128 bytes: one
// wavefront per load, ≤ RT1/2 + OT1/2 wavefronts per 4·RT1·OT1 FFMA.
template <int R1, int O>
struct LrCfg {
  static constexpr int RT1 = R1 == 64 ? 8 : (R1 == 24 ? 6 : 4);
  static constexpr int NR1 = R1 / RT1;        // 4, 4, 8, 8 for R1 = 16, 24, 32, 64
  static constexpr int NO1 = 128 / NR1;       // 32, 16, 16
  static constexpr int OT1 = O / NO1;
  static constexpr int SO = O + 2;            // padded sS row (conflict-free cp.async writes, 16-B aligned rows)
  static constexpr int PH1 = 2 * XK * R1 + 2 * XK * SO;     // sV[2][XK][R1] + sS[2][XK][SO] (float2)
  static constexpr int PH2 = R1 * O + 2 * R1 * 32;           // tmp[R1][O] + sU[2][R1][32]
  static constexpr int SMEM = (PH1 > PH2 ? PH1 : PH2) * 8;
};


template <int R1, int O>
__global__ void __launch_bounds__(128) k_m2l_lr(const LrTask* __restrict__ tasks, const int64_t* __restrict__ src_off,
                                                const int64_t* __restrict__ dst_off, const float2* __restrict__ pool,
                                                const float2* __restrict__ src, float2* __restrict__ dst) {
  using C = LrCfg<R1, O>;
  constexpr int RT1 = C::RT1, NO1 = C::NO1, OT1 = C::OT1;
  extern __shared__ float4 smem4[];
  float2* sh = reinterpret_cast<float2*>(smem4);
  __shared__ int64_t soff[O];
  __shared__ int64_t doff[O];
  const LrTask t = tasks[blockIdx.x];
  const int tid = threadIdx.x;
  for (int p = tid; p < O; p += 128) {
    soff[p] = p < t.op_count ? src_off[t.op_begin + p] : -1;
    doff[p] = p < t.op_count ? dst_off[t.op_begin + p] : -1;
  }
  __syncthreads();
  const float2* __restrict__ V = pool + t.v_off;
  const float2* __restrict__ U = pool + t.u_off;

  // ---- phase 1: tmp[R1][64] = V̂ · S
  float2* sV = sh;                      // [2][XK][R1]
  constexpr int SO = C::SO;
  float2* sS = sh + 2 * XK * R1;        // [2][XK][SO]
  auto issue1 = [&](int buf, int k0) {
#pragma unroll
    for (int e = 0; e < XK * R1 / 128; ++e) {
      const int idx = tid + 128 * e;
      const int kk = idx / R1, row = idx % R1, col = k0 + kk;
      const bool ok = row < t.r && col < t.T;
      cp_async8(sV + (buf * XK + kk) * R1 + row, ok ? (const void*)(V + (int64_t)col * t.r + row) : (const void*)V,
                ok);
    }
#pragma unroll
    for (int e = 0; e < XK * O / 128; ++e) {
      const int idx = tid + 128 * e;
      const int p = idx / XK, kk = idx % XK, col = k0 + kk;
      const int64_t so = soff[p];
      const bool ok = so >= 0 && col < t.T;
      cp_async8(sS + (buf * XK + kk) * SO + p, ok ? (const void*)(src + so + col) : (const void*)src, ok);
    }
    cp_async_commit();
  };
  constexpr int NR1 = C::NR1;
  const int lane = tid & 31, warp = tid >> 5;
  const int tr1 = (warp % (NR1 / 4)) * 4 + (lane >> 3), to1 = (warp / (NR1 / 4)) * 8 + (lane & 7);
  float2 acc[RT1][OT1];
#pragma unroll
  for (int i = 0; i < RT1; ++i)
#pragma unroll
    for (int j = 0; j < OT1; ++j) acc[i][j] = make_float2(0.f, 0.f);
  issue1(0, 0);
  int buf = 0;
  for (int k0 = 0; k0 < t.T; k0 += XK) {
    if (k0 + XK < t.T) {
      issue1(buf ^ 1, k0 + XK);
      cp_async_wait_1();
    } else {
      cp_async_wait_0();
    }
    __syncthreads();
    const float4* mv = reinterpret_cast<const float4*>(sV + buf * XK * R1 + 2 * tr1);
    const float4* sv = reinterpret_cast<const float4*>(sS + buf * XK * SO + 2 * to1);
#pragma unroll
    for (int kk = 0; kk < XK; ++kk) {
      float2 m[RT1], v[OT1];
#pragma unroll
      for (int i = 0; i < RT1 / 2; ++i) {
        const float4 q = mv[kk * (R1 / 2) + NR1 * i];
        m[2 * i] = make_float2(q.x, q.y);
        m[2 * i + 1] = make_float2(q.z, q.w);
      }
#pragma unroll
      for (int j = 0; j < OT1 / 2; ++j) {
        const float4 q = sv[kk * (SO / 2) + NO1 * j];
        v[2 * j] = make_float2(q.x, q.y);
        v[2 * j + 1] = make_float2(q.z, q.w);
      }
#pragma unroll
      for (int i = 0; i < RT1; ++i)
#pragma unroll
        for (int j = 0; j < OT1; ++j) cmac(acc[i][j], m[i], v[j]);
    }
    __syncthreads();
    buf ^= 1;
  }
  // tmp[row][op] (rows ≥ r are zero: V̂ rows ≥ r were zero-filled)
  float2* tmp = sh;                    // [R1][O]
  float2* sU = sh + R1 * O;            // [2][R1][32]
#pragma unroll
  for (int i = 0; i < RT1; ++i)
#pragma unroll
    for (int j = 0; j < OT1 / 2; ++j) {
      float4 q = make_float4(acc[i][2 * j].x, acc[i][2 * j].y, acc[i][2 * j + 1].x, acc[i][2 * j + 1].y);
      const int row = 2 * tr1 + (i & 1) + 2 * NR1 * (i >> 1);
      *reinterpret_cast<float4*>(tmp + row * O + 2 * to1 + 2 * NO1 * j) = q;
    }

  // ---- phase 2: dst[:, op] += Û[r0:r0+32, :] · tmp[:, op]
  auto issue2 = [&](int b, int r0) {
    for (int idx = tid; idx < R1 * 32; idx += 128) {
      const int c = idx / 32, row = idx % 32;
      const bool ok = c < t.r && r0 + row < t.T;
      cp_async8(sU + (b * R1 + c) * 32 + row, ok ? (const void*)(U + (int64_t)c * t.T + r0 + row) : (const void*)U,
                ok);
    }
    cp_async_commit();
  };
  // rows {2·tr2, 2·tr2+1} + 16i, ops {2·to2, 2·to2+1} + 32j; warps 2 × 2 of 4 × 8 lanes
  const int tr2 = (warp & 1) * 4 + (lane >> 3), to2 = (warp >> 1) * 8 + (lane & 7);
  int b2 = 0;
  for (int oh = 0; oh < O && oh < t.op_count; oh += 64) {      // op halves of 64 (O = 128)
  issue2(b2, 0);
  for (int r0 = 0; r0 < t.T; r0 += 32) {
    if (r0 + 32 < t.T) {
      issue2(b2 ^ 1, r0 + 32);
      cp_async_wait_1();
    } else {
      cp_async_wait_0();
    }
    __syncthreads();
    float2 a2[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) a2[i][j] = make_float2(0.f, 0.f);
    const float4* uv = reinterpret_cast<const float4*>(sU + b2 * R1 * 32 + 2 * tr2);
    const float4* tv = reinterpret_cast<const float4*>(tmp + oh + 2 * to2);
#pragma unroll 4
    for (int c = 0; c < t.r; ++c) {
      float2 m[4], v[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const float4 q = uv[c * 16 + 8 * i];
        m[2 * i] = make_float2(q.x, q.y);
        m[2 * i + 1] = make_float2(q.z, q.w);
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const float4 q = tv[c * (O / 2) + 16 * j];
        v[2 * j] = make_float2(q.x, q.y);
        v[2 * j + 1] = make_float2(q.z, q.w);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) cmac(a2[i][j], m[i], v[j]);
    }
    // rows (2·tr2, 2·tr2+1) are a pair: one 16-byte vector atomic per pair (states are
    // 16-byte aligned and padded to an even length; rows ≥ T hold zeros since Û rows ≥ T
    // were zero-filled, so the pair (T-1, T) adds a zero into the padding slot)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int op = oh + 2 * to2 + (j & 1) + 32 * (j >> 1);
      if (op >= t.op_count) continue;
      float2* d = dst + doff[op] + r0;
#pragma unroll
      for (int i = 0; i < 4; i += 2) {
        const int row = 2 * tr2 + 16 * (i >> 1);
        if (r0 + row < t.T)
          atomicAdd(reinterpret_cast<float4*>(d + row),
                    make_float4(a2[i][j].x, a2[i][j].y, a2[i + 1][j].x, a2[i + 1][j].y));
      }
    }
    __syncthreads();
    b2 ^= 1;
  }
  }
}

// one launch per phase-1 row class (r ≤ 16, ≤ 32, ≤ 64); tasks[cls] sorted longest first
void launch_m2l_lr(int cls, int ntask, const LrTask* tasks, const int64_t* src_off, const int64_t* dst_off,
                   const float2* pool, const float2* src, float2* dst, cudaStream_t s) {
  if (ntask <= 0) return;
  switch (cls) {
    case 0: k_m2l_lr<16, 64><<<ntask, 128, LrCfg<16, 64>::SMEM, s>>>(tasks, src_off, dst_off, pool, src, dst); break;
    case 1: k_m2l_lr<24, 64><<<ntask, 128, LrCfg<24, 64>::SMEM, s>>>(tasks, src_off, dst_off, pool, src, dst); break;
    case 2: k_m2l_lr<32, 64><<<ntask, 128, LrCfg<32, 64>::SMEM, s>>>(tasks, src_off, dst_off, pool, src, dst); break;
    default: k_m2l_lr<64, 64><<<ntask, 128, LrCfg<64, 64>::SMEM, s>>>(tasks, src_off, dst_off, pool, src, dst); break;
  }
}
int m2l_lr_class(int r) { return r <= 16 ? 0 : (r <= 24 ? 1 : (r <= 32 ? 2 : 3)); }
int m2l_lr_rows(int cls) { return cls == 0 ? 16 : (cls == 1 ? 24 : (cls == 2 ? 32 : 64)); }
int m2l_lr_ops(int) { return 64; }
cudaError_t m2l_lr_prepare() {
  return cudaFuncSetAttribute(k_m2l_lr<64, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, LrCfg<64, 64>::SMEM);
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
// sharded GMRES helpers: Σ partial (no square root; summed over ranks before the root)
__global__ void k_reduce_sum(const double* __restrict__ partial, int nchunks, double* __restrict__ out) {
  __shared__ double red[128];
  double a = 0;
  for (int c = threadIdx.x; c < nchunks; c += blockDim.x) a += partial[c];
  red[threadIdx.x] = a;
  __syncthreads();
  for (int k = blockDim.x / 2; k > 0; k >>= 1) {
    if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}
void launch_reduce_sum(const double* partial, int nchunks, double* out, cudaStream_t s) {
  k_reduce_sum<<<1, 128, 0, s>>>(partial, nchunks, out);
}
__global__ void k_sqrt1(double* x) { x[0] = sqrt(x[0]); }
void launch_sqrt1(double* x, cudaStream_t s) { k_sqrt1<<<1, 1, 0, s>>>(x); }
// y[i] = a[off + i] + b[off + i]
__global__ void k_add_slice(const float2* __restrict__ a, const float2* __restrict__ b, int64_t off, int64_t n,
                            float2* __restrict__ y) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float2 u = a[off + i], v = b[off + i];
  y[i] = make_float2(u.x + v.x, u.y + v.y);
}
void launch_add_slice(const float2* a, const float2* b, int64_t off, int64_t n, float2* y, cudaStream_t s) {
  if (n > 0) k_add_slice<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, b, off, n, y);
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

// b_i = u_inc(x_i) + α ∂u_inc/∂n(x_i) for a unit point source u_inc = e^{ikR}/(4πR),
// R = |x_i - x_s| (§5.2; Eq. 3), n_i = kernel normal:
//   b_i = G [1 + α (ik - 1/R) (x_i - x_s)·n_i / R]      (fp64, caller order)
__global__ void k_point_source(const double* __restrict__ cen, const double* __restrict__ nrm,
                               const int32_t* __restrict__ perm, int n, double k, double are, double aim, double sx,
                               double sy, double sz, float2* b32, double2* b64) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double dx = cen[3 * i] - sx, dy = cen[3 * i + 1] - sy, dz = cen[3 * i + 2] - sz;
  const double R = sqrt(dx * dx + dy * dy + dz * dz);
  const double dRdn = (dx * nrm[3 * i] + dy * nrm[3 * i + 1] + dz * nrm[3 * i + 2]) / R;
  double s, c;
  sincos(k * R, &s, &c);
  const double g = 1.0 / (4.0 * CUDART_PI * R);
  const double gr = g * c, gi = g * s;
  // f = 1 + α (ik - 1/R) dRdn,  α (ik - 1/R) = (are + i aim)(-1/R + i k)
  const double tr = -are / R - aim * k, ti = are * k - aim / R;
  const double fr = 1.0 + tr * dRdn, fi = ti * dRdn;
  const double br = gr * fr - gi * fi, bi = gr * fi + gi * fr;
  const int j = perm[i];
  if (b32) b32[j] = make_float2((float)br, (float)bi);
  if (b64) b64[j] = make_double2(br, bi);
}
void launch_point_source(const double* cen, const double* nrm, const int32_t* perm, int n, double k, double are,
                         double aim, double sx, double sy, double sz, float2* b32, double2* b64, cudaStream_t s) {
  k_point_source<<<(n + 255) / 256, 256, 0, s>>>(cen, nrm, perm, n, k, are, aim, sx, sy, sz, b32, b64);
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
