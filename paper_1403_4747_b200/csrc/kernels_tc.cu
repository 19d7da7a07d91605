// Tensor-core (tcgen05, sm_100a) grouped complex GEMM for the dense FDA
// translations (M2M, L2L, dense M2L):
//   dst[:, op] += M · src[:, op]   for the ops of one task, all sharing M (R × C complex).
//
// Complex arithmetic as one real GEMM with interleaved K and M: the complex
// states are float2 arrays, i.e. a state is the real vector
// (re₀, im₀, re₁, im₁, …); with the real 2R × 2C matrix
//   A[2i][2j] = Re M_ij,  A[2i][2j+1] = −Im M_ij,  A[2i+1][2j] = Im M_ij,  A[2i+1][2j+1] = Re M_ij
// the product A · state is the interleaved complex result, so the B operand
// is the raw state memory (no pre-split planes) and the accumulator row 2i /
// 2i+1 is Re / Im of output i.
//
// fp32 accuracy from TF32 tensor cores by the 3-term split (3xTF32):
//   A·B ≈ A_hi·B_hi + A_hi·B_lo + A_lo·B_hi,  X_hi = tf32(X), X_lo = tf32(X − X_hi);
// A is split and pre-laid-out on the host (engine.cu: tc_matrix) in the
// canonical K-major no-swizzle UMMA layout — core matrices of 8 rows × 16 B —
// per 128-row tile and KC-float K chunk, [hi | lo] contiguous, and streamed
// with one bulk async copy (cp.async.bulk, TMA engine, mbarrier tx-count) per
// tile and chunk; B (the gathered source states, 16-B cp.async per op and
// k-group, zero-filled past the state end) is split into hi / lo in shared
// memory.  S-stage ring: the copies of chunks c+1 … c+S-1 are in flight while
// one thread issues the MMAs of chunk c (tcgen05.mma.cta_group::1.kind::tf32,
// M = 128, N ∈ {128, 256}, K = 8) into TMEM accumulators (one 128 × N block
// per row tile); tcgen05.commit on an mbarrier releases the stage.  Epilogue:
// tcgen05.ld of each accumulator block into shared memory (op-major), then
// coalesced 16-byte vector atomics into the destination states (several tasks
// may share a destination).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"

namespace fda {

namespace {
constexpr int KC = TC_KC;        // floats of K per stage (= 8 complex columns)
constexpr int A_TILE = 128 * KC;  // floats per (row tile, chunk, hi|lo)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// canonical K-major, no-swizzle UMMA shared-memory descriptor
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
  return d;
}

// instruction descriptor: kind::tf32, D = F32, A/B = TF32, both K-major, M = 128, N
template <int N>
__device__ __forceinline__ constexpr uint32_t make_idesc() {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

// bulk async copy global → shared (TMA engine), completion counted on mbar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// 16-byte cp.async with src-size (bytes beyond it are zero-filled)
__device__ __forceinline__ void cp16z(void* s, const void* g, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(s)), "l"(g), "r"(bytes));
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}

__host__ __device__ constexpr uint32_t tmem_cols(int n) { return n <= 32 ? 32 : (n <= 64 ? 64 : (n <= 128 ? 128 : (n <= 256 ? 256 : 512))); }
}  // namespace

template <int N, int TILES, int STAGES>
struct TcCfg {
  static constexpr int A_FL = TILES * 2 * A_TILE;   // A floats per stage
  static constexpr int B_FL = 2 * N * KC;          // B floats per stage (hi, lo)
  static constexpr int STAGE_FL = A_FL + B_FL;
  static constexpr int SM_FL = STAGES * STAGE_FL > N * 128 ? STAGES * STAGE_FL : N * 128;   // + epilogue
  static constexpr size_t SMEM = (size_t)SM_FL * 4 + 1024;
  static_assert(TILES * N <= 512, "TMEM columns");
};

template <int N, int TILES, int STAGES, int MINB>
__global__ void __launch_bounds__(128, MINB) k_xlate_tc(const TcTask* __restrict__ tasks,
                                                     const int64_t* __restrict__ src_off,
                                                     const int64_t* __restrict__ dst_off,
                                                     const float* __restrict__ tcpool, const float2* __restrict__ src,
                                                     float2* __restrict__ dst) {
  using Cfg = TcCfg<N, TILES, STAGES>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  float* sbase = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t mbar_a[STAGES], mbar_m[STAGES];
  __shared__ uint32_t tmem_base_sh;
  __shared__ int64_t soff[N];   // float offset of the source state (-1: padding op)
  __shared__ int64_t doff[N];   // complex offset of the destination state
  const TcTask t = tasks[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K2 = 2 * t.C;       // real K

  for (int p = tid; p < N; p += 128) {
    const bool ok = p < t.op_count;
    soff[p] = ok ? 2 * src_off[t.op_begin + p] : -1;
    doff[p] = ok ? dst_off[t.op_begin + p] : -1;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(tmem_cols(TILES * N)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&mbar_a[s], 1);
      mbar_init(&mbar_m[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = tmem_base_sh;
  const int nkc = t.nkc, kc0 = t.kc0, nk = t.kc1 - t.kc0;   // this task: chunks kc0 … kc1-1
  const float* gA = tcpool + t.a_off;

  // stage layout: [A: tile][hi|lo][128 × KC] | [B hi: N × KC][B lo: N × KC]
  auto issue = [&](int c) {   // c: local chunk index (global chunk kc0 + c)
    const int st = c % STAGES;
    const int cg = kc0 + c;
    float* sA = sbase + st * Cfg::STAGE_FL;
    float* sB = sA + Cfg::A_FL;
    if (tid == 0) {
      mbar_expect_tx(&mbar_a[st], (uint32_t)(TILES * 2 * A_TILE * 4));
#pragma unroll
      for (int ti = 0; ti < TILES; ++ti)
        bulk_g2s(sA + ti * 2 * A_TILE, gA + ((int64_t)ti * nkc + cg) * 2 * A_TILE, 2 * A_TILE * 4, &mbar_a[st]);
    }
    // B: op n, k-group kg (4 floats) → ((kg · N/8 + n/8) · 8 + n%8) · 4
    for (int idx = tid; idx < N * (KC / 4); idx += 128) {
      const int n = idx >> 2, kg = idx & 3;
      const int k = cg * KC + 4 * kg;
      const int64_t so = soff[n];
      int bytes = so >= 0 ? 4 * min(4, max(0, K2 - k)) : 0;
      const float* g = bytes ? reinterpret_cast<const float*>(src) + so + k : reinterpret_cast<const float*>(src);
      cp16z(sB + ((kg * (N / 8) + (n >> 3)) * 8 + (n & 7)) * 4, g, bytes);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };

  for (int c = 0; c < STAGES - 1; ++c) {
    if (c < nk) issue(c);
    else asm volatile("cp.async.commit_group;\n" ::);
  }
  for (int c = 0; c < nk; ++c) {
    const int st = c % STAGES;
    const int cn = c + STAGES - 1;
    if (cn < nk) {
      if (c >= 1) mbar_wait(&mbar_m[(c - 1) % STAGES], ((c - 1) / STAGES) & 1);   // MMAs of chunk c-1 done
      issue(cn);
    } else {
      asm volatile("cp.async.commit_group;\n" ::);
    }
    asm volatile("cp.async.wait_group %0;\n" ::"n"(STAGES - 1) : "memory");
    mbar_wait(&mbar_a[st], (c / STAGES) & 1);
    __syncthreads();
    float* sA = sbase + st * Cfg::STAGE_FL;
    float* sB = sA + Cfg::A_FL;
    // split B into tf32 hi (low 13 mantissa bits cleared, in place) and lo
    {
      float4* bh = reinterpret_cast<float4*>(sB);
      float4* bl = reinterpret_cast<float4*>(sB + N * KC);
      for (int i = tid; i < N * KC / 4; i += 128) {
        const float4 v = bh[i];
        const float4 h = make_float4(__uint_as_float(__float_as_uint(v.x) & 0xffffe000u),
                                     __uint_as_float(__float_as_uint(v.y) & 0xffffe000u),
                                     __uint_as_float(__float_as_uint(v.z) & 0xffffe000u),
                                     __uint_as_float(__float_as_uint(v.w) & 0xffffe000u));
        bh[i] = h;
        bl[i] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      constexpr uint32_t idesc = make_idesc<N>();
      const uint32_t b_hi = smem_u32(sB), b_lo = smem_u32(sB + N * KC);
#pragma unroll
      for (int s = 0; s < KC / 8; ++s) {
        const uint32_t bo = (uint32_t)(2 * s * (N / 8) * 128);
        const uint64_t Bh = make_desc(b_hi + bo, (N / 8) * 128, 128);
        const uint64_t Bl = make_desc(b_lo + bo, (N / 8) * 128, 128);
#pragma unroll
        for (int ti = 0; ti < TILES; ++ti) {
          const uint32_t a_hi = smem_u32(sA + ti * 2 * A_TILE), a_lo = a_hi + A_TILE * 4;
          const uint32_t ao = (uint32_t)(2 * s * 16 * 128);
          const uint64_t Ah = make_desc(a_hi + ao, 16 * 128, 128), Al = make_desc(a_lo + ao, 16 * 128, 128);
          const uint32_t d = tmem + ti * N;
          mma_tf32(d, Ah, Bh, idesc, (c > 0 || s > 0) ? 1u : 0u);
          mma_tf32(d, Ah, Bl, idesc, 1u);
          mma_tf32(d, Al, Bh, idesc, 1u);
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                       smem_u32(&mbar_m[st]))
                   : "memory");
    }
  }
  mbar_wait(&mbar_m[(nk - 1) % STAGES], ((nk - 1) / STAGES) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);

  // epilogue, per row tile: TMEM → shared memory column-major (column = op; rows 2i, 2i+1 =
  // Re, Im of output i, so an op's outputs are contiguous float2), then each warp adds whole
  // columns to the destination states with coalesced 16-byte vector atomics (2 outputs per
  // lane; states are 16-byte aligned and padded to an even length, so the pair (i, i+1 = R)
  // adds a zero into the padding slot).  The pipeline buffers are free here.
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  float* sE = sbase;                         // [N][128] floats
#pragma unroll 1
  for (int ti = 0; ti < TILES; ++ti) {
#pragma unroll 1
    for (int c0 = 0; c0 < N; c0 += 16) {
      float v[16];
      tmem_ld16(tmem + lane_base + ti * N + c0, v);
#pragma unroll
      for (int j = 0; j < 16; ++j) sE[(c0 + j) * 128 + 32 * warp + lane] = v[j];
    }
    __syncthreads();
    const int i = 64 * ti + 2 * lane;        // this lane's first output of the tile
#pragma unroll 4
    for (int op = warp; op < N; op += 4) {
      if (op < t.op_count && i < t.R) {
        const float4 q = reinterpret_cast<const float4*>(sE + op * 128)[lane];
        atomicAdd(reinterpret_cast<float4*>(dst + doff[op] + i), q);
      }
    }
    __syncthreads();
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(tmem_cols(TILES * N)));
}

// ---------------------------------------------------------------------------
// Fused §4.2 M2L on the tensor cores (§4.2):
//   dst[:, op] += Û (V̂ src[:, op])   for ≤ 128 ops sharing one factored K̃ ≈ Û V̂.
// The ops are the M = 128 rows (TMEM lanes) of both products, in the interleaved
// real form of the kernel above transposed (row op = the op's state as a real
// vector of length 2T):
//   phase 1  D1 (128 × 2R1p) = S (128 × 2T) · A_Vᵀ,   A_V = real 2r × 2T form of V̂;
//   phase 2  D2 (128 × 2Tp)  = D1 (128 × 2R1p) · A_Uᵀ, A_U = real 2T × 2r form of Û,
// so the B operands (A_Vᵀ, A_Uᵀ) are pre-laid-out constants (host, engine.cu:
// tc_bop) streamed by the TMA engine, the A operand of phase 1 is the gathered
// source states (each thread loads its op's K chunk, splits it into tf32
// hi / lo in registers and stores both into the canonical K-major layout),
// and the A operand of phase 2 is phase 1's accumulator read back from TMEM
// (tcgen05.ld) and split the same way — the r-vector tmp never leaves the SM.
// 3xTF32 throughout (hi·hi + hi·lo + lo·hi).  Epilogue: each thread holds its
// op's whole output state (tcgen05.ld of its TMEM lane) and adds it to the
// destination state with 16-byte vector atomics.
namespace {
__device__ __forceinline__ uint32_t idesc_n(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ float4 tf32_hi4(float4 v) {
  return make_float4(__uint_as_float(__float_as_uint(v.x) & 0xffffe000u), __uint_as_float(__float_as_uint(v.y) & 0xffffe000u),
                     __uint_as_float(__float_as_uint(v.z) & 0xffffe000u), __uint_as_float(__float_as_uint(v.w) & 0xffffe000u));
}
// A operand row `row` (0…127), k-group kg (4 floats) of a [hi | lo] 128 × 16-float chunk
__device__ __forceinline__ void put_a(float* chunk, int row, int kg, float4 v) {
  const float4 h = tf32_hi4(v);
  const int idx = ((kg * 16 + (row >> 3)) * 8 + (row & 7)) * 4;
  *reinterpret_cast<float4*>(chunk + idx) = h;
  *reinterpret_cast<float4*>(chunk + 128 * TC_KC + idx) = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
}
}  // namespace

// ---------------------------------------------------------------------------
// Warp-specialised persistent form (k_m2l_tcw, the default tensor-core M2L):
//   warps 0-3 (the "row" warps, thread t = op t = TMEM lane t): gather the
//     states of phase-1 ring jobs (16-B cp.async, issued S1 − 2 jobs ahead),
//     split them hi / lo in place, arrive on a_full; at each task boundary
//     drain the previous task's D2 (TMEM → 16-B vector atomics) and turn D1
//     into the phase-2 A operand;
//   warp 4 (one lane): issues every MMA and commits (frees ring stages,
//     signals D1 / D2 complete);
//   warp 5 (one lane): streams the B1 and B2 operands with the TMA engine.
// TMEM: D1 in columns [0, n1max), D2 in [n1max, n1max + n2max), so the MMAs of
// task i+1's phase 1 run while the row warps drain D2 of task i.  Barriers
// (phase parity = use count & 1): a_full[s] (128 arrivals) + b_full[s] (TMA)
// → MMA; empty[s] (MMA commit) → refill; b2_full / b2_empty (2-stage B2 ring);
// d1_full, a2_full (128), d2_full, y_free (128) once per task.
constexpr int TCW_RW = 8;                   // row warps (two threads per op row)
constexpr int TCW_NT = 32 * (TCW_RW + 2);   // + MMA warp + TMA warp
template <int S1>
__global__ void __launch_bounds__(TCW_NT, 1) k_m2l_tcw(const LrTcTask* __restrict__ tasks, int ntask,
                                                    const int64_t* __restrict__ src_off,
                                                    const int64_t* __restrict__ dst_off,
                                                    const float* __restrict__ tcpool, const float2* __restrict__ src,
                                                    float2* __restrict__ dst, int stage_fl, int b2_fl, int n1max,
                                                    uint32_t ncols) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  float* sbase = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t a_full[S1], b_full[S1], empty[S1], b2_full[2], b2_empty[2];
  __shared__ uint64_t d1_full, a2_full, d2_full, y_free;
  __shared__ uint32_t tmem_base_sh;
  constexpr int LA = S1 >= 8 ? S1 - 4 : (S1 > 4 ? S1 - 3 : S1 - 2);   // gather lookahead; the rest is MMA-completion slack
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x;
  float* sB2 = sbase + S1 * stage_fl;              // [2][b2_fl]
  float* sA2 = sB2 + 2 * b2_fl;                    // phase-2 A operand: (n1/16) × [hi | lo] 128 × 16
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  if (tid == 0) {
    for (int q = 0; q < S1; ++q) {
      mbar_init(&a_full[q], 32 * TCW_RW);
      mbar_init(&b_full[q], 1);
      mbar_init(&empty[q], 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&b2_full[q], 1);
      mbar_init(&b2_empty[q], 1);
    }
    mbar_init(&d1_full, 1);
    mbar_init(&a2_full, 32 * TCW_RW);
    mbar_init(&d2_full, 1);
    mbar_init(&y_free, 32 * TCW_RW);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = tmem_base_sh;
  const uint32_t tY = tmem + (uint32_t)n1max;      // D2 region

  if (warp == TCW_RW + 1) {
    // ---------------- TMA producer
    if (lane == 0) {
      int j = 0, b2j = 0;
      for (int ct = blockIdx.x; ct < ntask; ct += G) {
        const LrTcTask t = tasks[ct];
        for (int c = 0; c < t.nk1; ++c, ++j) {
          const int st = j % S1;
          if (j >= S1) mbar_wait(&empty[st], ((j / S1) - 1) & 1);
          const uint32_t bytes = (uint32_t)t.n1 * TC_KC * 2 * 4;
          mbar_expect_tx(&b_full[st], bytes);
          bulk_g2s(sbase + st * stage_fl + 2 * 128 * TC_KC, tcpool + t.b1_off + (int64_t)c * t.n1 * TC_KC * 2, bytes,
                   &b_full[st]);
        }
        const int nk2 = t.n1 / TC_KC;
        for (int c2 = 0; c2 < nk2; ++c2, ++b2j) {
          const int st = b2j & 1;
          if (b2j >= 2) mbar_wait(&b2_empty[st], ((b2j >> 1) - 1) & 1);
          const uint32_t bytes = (uint32_t)t.n2 * TC_KC * 2 * 4;
          mbar_expect_tx(&b2_full[st], bytes);
          bulk_g2s(sB2 + st * b2_fl, tcpool + t.b2_off + (int64_t)c2 * t.n2 * TC_KC * 2, bytes, &b2_full[st]);
        }
      }
    }
  } else if (warp == TCW_RW) {
    // ---------------- MMA issuer
    if (lane == 0) {
      int j = 0, b2j = 0, i = 0;
      for (int ct = blockIdx.x; ct < ntask; ct += G, ++i) {
        const LrTcTask t = tasks[ct];
        const int N1 = t.n1, N2 = t.n2, nk2 = N1 / TC_KC;
        const uint32_t idesc1 = idesc_n(N1);
        for (int c = 0; c < t.nk1; ++c, ++j) {
          const int st = j % S1;
          mbar_wait(&a_full[st], (j / S1) & 1);
          mbar_wait(&b_full[st], (j / S1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
          float* sA = sbase + st * stage_fl;
          const uint32_t a_hi = smem_u32(sA), a_lo = a_hi + 128 * TC_KC * 4;
          const uint32_t b_hi = smem_u32(sA + 2 * 128 * TC_KC), b_lo = b_hi + N1 * TC_KC * 4;
#pragma unroll
          for (int s = 0; s < TC_KC / 8; ++s) {
            const uint32_t ao = (uint32_t)(s * 2 * 16 * 128), bo = (uint32_t)(s * 2 * (N1 / 8) * 128);
            const uint64_t Ah = make_desc(a_hi + ao, 16 * 128, 128), Al = make_desc(a_lo + ao, 16 * 128, 128);
            const uint64_t Bh = make_desc(b_hi + bo, (N1 / 8) * 128, 128), Bl = make_desc(b_lo + bo, (N1 / 8) * 128, 128);
            mma_tf32(tmem, Ah, Bh, idesc1, (c > 0 || s > 0) ? 1u : 0u);
            mma_tf32(tmem, Ah, Bl, idesc1, 1u);
            mma_tf32(tmem, Al, Bh, idesc1, 1u);
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                           smem_u32(&empty[st]))
                       : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         smem_u32(&d1_full))
                     : "memory");
        mbar_wait(&a2_full, i & 1);                   // tmp is in shared memory (and D1 was read)
        if (i >= 1) mbar_wait(&y_free, (i - 1) & 1);  // D2 of the previous task was drained
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        for (int c2 = 0; c2 < nk2; ++c2, ++b2j) {
          const int st = b2j & 1;
          mbar_wait(&b2_full[st], (b2j >> 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
          const uint32_t b_hi = smem_u32(sB2 + st * b2_fl), b_lo = b_hi + N2 * TC_KC * 4;
          const uint32_t a_hi = smem_u32(sA2 + c2 * 2 * 128 * TC_KC), a_lo = a_hi + 128 * TC_KC * 4;
#pragma unroll
          for (int s = 0; s < TC_KC / 8; ++s) {
            const uint32_t ao = (uint32_t)(s * 2 * 16 * 128), bo = (uint32_t)(s * 2 * (N2 / 8) * 128);
            const uint64_t Ah = make_desc(a_hi + ao, 16 * 128, 128), Al = make_desc(a_lo + ao, 16 * 128, 128);
            for (int n0 = 0; n0 < N2; n0 += 256) {
              const int nn = min(256, N2 - n0);
              const uint32_t idesc = idesc_n(nn);
              const uint32_t no = (uint32_t)((n0 / 8) * 128);
              const uint64_t Bh = make_desc(b_hi + bo + no, (N2 / 8) * 128, 128);
              const uint64_t Bl = make_desc(b_lo + bo + no, (N2 / 8) * 128, 128);
              mma_tf32(tY + n0, Ah, Bh, idesc, (c2 > 0 || s > 0) ? 1u : 0u);
              mma_tf32(tY + n0, Ah, Bl, idesc, 1u);
              mma_tf32(tY + n0, Al, Bh, idesc, 1u);
            }
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                           smem_u32(&b2_empty[st]))
                       : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         smem_u32(&d2_full))
                     : "memory");
      }
    }
  } else {
    // ---------------- row warps: thread (row = tid & 127, half h = tid >> 7); warp w reads TMEM
    // lanes 32·(w & 3) …; half h copies and splits k-groups {2h, 2h+1} of each chunk and
    // converts / drains the 16-column blocks b ≡ h (mod 2)
    const int row = tid & 127, h = tid >> 7;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    int it = blockIdx.x, ic = 0, js = 0;          // issue cursor over phase-1 jobs
    LrTcTask ti = tasks[it];
    const float* isp = row < ti.op_count ? reinterpret_cast<const float*>(src) + 2 * src_off[ti.op_begin + row] : nullptr;
    auto issue_next = [&]() {
      if (it < ntask) {
        const int st = js % S1;
        if (js >= S1) mbar_wait(&empty[st], ((js / S1) - 1) & 1);
        float* sA = sbase + st * stage_fl;
        const int K2 = 2 * ti.T;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int kg = 2 * h + q;
          const int k = ic * TC_KC + 4 * kg;
          const int nb = isp ? 4 * min(4, max(0, K2 - k)) : 0;
          cp16z(sA + ((kg * 16 + (row >> 3)) * 8 + (row & 7)) * 4, nb ? (const void*)(isp + k) : (const void*)src, nb);
        }
        ++js;
        if (++ic == ti.nk1) {
          ic = 0;
          it += G;
          if (it < ntask) {
            ti = tasks[it];
            isp = row < ti.op_count ? reinterpret_cast<const float*>(src) + 2 * src_off[ti.op_begin + row] : nullptr;
          }
        }
      }
      asm volatile("cp.async.commit_group;\n" ::);
    };
    for (int q = 0; q < LA; ++q) issue_next();
    int jc = 0, i = 0;
    LrTcTask tp{};                                 // previous task (its D2 is drained at the next boundary)
    auto drain = [&](const LrTcTask& t) {
      float2* d = row < t.op_count ? dst + dst_off[t.op_begin + row] : nullptr;
      for (int c0 = 16 * h; c0 < t.n2; c0 += 32) {
        float w[16];
        tmem_ld16(tY + lane_base + c0, w);
        if (d) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int r = c0 / 2 + 2 * q;   // complex rows (r, r+1); r+1 = T is the padding slot
            if (r < t.T)
              atomicAdd(reinterpret_cast<float4*>(d + r), make_float4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]));
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
      mbar_arrive(&y_free);
    };
    for (int ct = blockIdx.x; ct < ntask; ct += G, ++i) {
      const LrTcTask t = tasks[ct];
      for (int c = 0; c < t.nk1; ++c, ++jc) {
        issue_next();
        asm volatile("cp.async.wait_group %0;\n" ::"n"(LA) : "memory");
        float* sA = sbase + (jc % S1) * stage_fl;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int kg = 2 * h + q;
          const int idx = ((kg * 16 + (row >> 3)) * 8 + (row & 7)) * 4;
          put_a(sA, row, kg, *reinterpret_cast<const float4*>(sA + idx));
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_arrive(&a_full[jc % S1]);
      }
      if (i >= 1) {                                // D2 of the previous task → destination states
        mbar_wait(&d2_full, (i - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        drain(tp);
      }
      mbar_wait(&d1_full, i & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      for (int c0 = 16 * h; c0 < t.n1; c0 += 32) {
        float w[16];
        tmem_ld16(tmem + lane_base + c0, w);
        float* ch = sA2 + (c0 / TC_KC) * 2 * 128 * TC_KC;
#pragma unroll
        for (int kg = 0; kg < 4; ++kg)
          put_a(ch, row, kg, make_float4(w[4 * kg], w[4 * kg + 1], w[4 * kg + 2], w[4 * kg + 3]));
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
      mbar_arrive(&a2_full);
      tp = t;
    }
    if (i >= 1) {
      mbar_wait(&d2_full, (i - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      drain(tp);
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(ncols));
}

// warp-specialised plan for one launch: ring stages S1 (3 … 8) of one 16-float K
// chunk (A hi|lo + B1 hi|lo), a 2-stage B2 ring and the phase-2 A region ≤ 220 KB
LrTcPlan m2l_tcw_plan(int n1max, int n2max) {
  LrTcPlan pl;
  pl.stage_fl = 2 * 128 * TC_KC + n1max * TC_KC * 2;
  pl.b2_fl = n2max * TC_KC * 2;
  const size_t a2 = (size_t)(n1max / TC_KC) * 2 * 128 * TC_KC;
  const size_t cap = (220 * 1024 - 1024) / 4 - 2 * (size_t)pl.b2_fl - a2;
  const int s = (int)(cap / pl.stage_fl);
  pl.stages = s >= 8 ? 8 : (s >= 6 ? 6 : (s >= 5 ? 5 : (s >= 4 ? 4 : 3)));
  pl.smem = ((size_t)pl.stages * pl.stage_fl + 2 * (size_t)pl.b2_fl + a2) * 4 + 1024;
  pl.ncols = tmem_cols(n1max + n2max);
  pl.n1max = n1max;
  return pl;
}
cudaError_t m2l_tcw_prepare() {
  cudaError_t e = cudaFuncSetAttribute(k_m2l_tcw<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_m2l_tcw<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_m2l_tcw<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_m2l_tcw<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_m2l_tcw<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  return e;
}
void launch_m2l_tcw(int ntask, const LrTcTask* tasks, const int64_t* src_off, const int64_t* dst_off,
                    const float* tcpool, const float2* src, float2* dst, const LrTcPlan& pl, int grid,
                    cudaStream_t s) {
  if (ntask <= 0) return;
#define TCW(S)                                                                                                   \
  k_m2l_tcw<S><<<grid, TCW_NT, pl.smem, s>>>(tasks, ntask, src_off, dst_off, tcpool, src, dst, pl.stage_fl, pl.b2_fl, \
                                          pl.n1max, pl.ncols)
  switch (pl.stages) {
    case 8: TCW(8); break;
    case 6: TCW(6); break;
    case 5: TCW(5); break;
    case 4: TCW(4); break;
    default: TCW(3); break;
  }
#undef TCW
}

// ---------------------------------------------------------------------------
// BF16x3 form of the fused factored M2L (k_m2l_bf; opt.lr_tensor_cores with opt.m2l_bf16):
// the roles and rings of k_m2l_tcw, with every operand split ONCE into bf16 hi / lo planes
// (x ≈ hi + lo, hi = bf16(x), lo = bf16(x − hi): 16 significant bits) and the products
// hi·hi + hi·lo + lo·hi on tcgen05 kind::f16 (K = 16 per MMA, fp32 accumulation in TMEM):
//  * the source states come pre-split (engine.cu: k_split_bf16 after the level's M2M), so the
//    row warps only issue 16-byte cp.async gathers straight into the canonical K-major bf16
//    layout — no in-shared-memory split pass (the LSU work that paced k_m2l_tcw);
//  * one ring job = 32 K elements (2 MMA k-steps); B1 / B2 (real forms of V̂ᵀ / Ûᵀ) are bf16
//    hi / lo tiles laid out on the device (k_tc_layout kind 2) and streamed by the TMA engine;
//  * phase 2's A operand is D1 read back from TMEM and split into bf16 hi / lo by the row warps.
// Error of a product: ≈ 2⁻¹⁶ relative (the dropped lo·lo term and the bf16 rounding of lo),
// i.e. ~1.5e-5 of the M2L contribution — below the FDA's own ε = 1e-4.
namespace {
constexpr int BK = 32;   // bf16 K elements per ring job
__device__ __forceinline__ uint32_t idesc_bf16(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// bf16 hi / lo of 8 floats packed as 4 + 4 32-bit words (element order = K order)
__device__ __forceinline__ void split8(const float* v, uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const __nv_bfloat16 h0 = __float2bfloat16_rn(v[2 * q]), h1 = __float2bfloat16_rn(v[2 * q + 1]);
    const __nv_bfloat16 l0 = __float2bfloat16_rn(v[2 * q] - __bfloat162float(h0));
    const __nv_bfloat16 l1 = __float2bfloat16_rn(v[2 * q + 1] - __bfloat162float(h1));
    h[q] = (uint32_t)__bfloat16_as_ushort(h0) | ((uint32_t)__bfloat16_as_ushort(h1) << 16);
    l[q] = (uint32_t)__bfloat16_as_ushort(l0) | ((uint32_t)__bfloat16_as_ushort(l1) << 16);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}
}  // namespace

__device__ int g_m2l_dbg = 0;   // FDA_M2L_DBG: per-role phase timers of CTA 0 (printf)
template <int S1>
__global__ void __launch_bounds__(TCW_NT, 1) k_m2l_bf(const LrTcTask* __restrict__ tasks, int ntask,
                                                   const int64_t* __restrict__ src_off,
                                                   const int64_t* __restrict__ dst_off,
                                                   const float* __restrict__ tcpool,
                                                   const __nv_bfloat16* __restrict__ shi,
                                                   const __nv_bfloat16* __restrict__ slo, float2* __restrict__ dst,
                                                   int stage_b, int b2_b, int n1max, uint32_t ncols) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sbase = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t a_full[S1], b_full[S1], empty[S1], b2_full[2], b2_empty[2];
  __shared__ uint64_t d1_full, a2_full, d2_full, y_free;
  __shared__ uint32_t tmem_base_sh;
  constexpr int LA = S1 >= 6 ? S1 - 3 : S1 - 2;
  constexpr int A_PL = 128 * BK * 2;               // bytes of one A plane (hi or lo) per job
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x;
  const bool dbg = g_m2l_dbg != 0 && blockIdx.x == 0;
  long long tp_e = 0, tp_b2 = 0, m_a = 0, m_b = 0, m_a2 = 0, m_y = 0, m_b2 = 0, r_e = 0, r_g = 0, r_d2 = 0, r_dr = 0,
            r_d1 = 0, r_is = 0, r_cv = 0, ntk = 0;
  const long long t_start = clock64();
  uint8_t* sB2 = sbase + S1 * stage_b;             // [2][b2_b]
  uint8_t* sA2 = sB2 + 2 * b2_b;                   // phase-2 A: (n1max / BK) jobs × [hi | lo] 128 × BK
  const uint8_t* pool8 = reinterpret_cast<const uint8_t*>(tcpool);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  if (tid == 0) {
    for (int q = 0; q < S1; ++q) {
      mbar_init(&a_full[q], 32 * TCW_RW);
      mbar_init(&b_full[q], 1);
      mbar_init(&empty[q], 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&b2_full[q], 1);
      mbar_init(&b2_empty[q], 1);
    }
    mbar_init(&d1_full, 1);
    mbar_init(&a2_full, 32 * TCW_RW);
    mbar_init(&d2_full, 1);
    mbar_init(&y_free, 32 * TCW_RW);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = tmem_base_sh;
  const uint32_t tY = tmem + (uint32_t)n1max;      // D2 region

  if (warp == TCW_RW + 1) {
    // ---------------- TMA producer: B1 per ring job, B2 per phase-2 job
    if (lane == 0) {
      int j = 0, b2j = 0;
      for (int ct = blockIdx.x; ct < ntask; ct += G) {
        const LrTcTask t = tasks[ct];
        const uint32_t bytes1 = (uint32_t)t.n1 * BK * 2 * 2;
        for (int c = 0; c < t.nk1; ++c, ++j) {
          const int st = j % S1;
          if (j >= S1) mbar_wait(&empty[st], ((j / S1) - 1) & 1);
          mbar_expect_tx(&b_full[st], bytes1);
          bulk_g2s(sbase + st * stage_b + 2 * A_PL, pool8 + 4 * t.b1_off + (int64_t)c * bytes1, bytes1, &b_full[st]);
        }
        const int nk2 = (t.n1 + BK - 1) / BK;
        const uint32_t bytes2 = (uint32_t)t.n2 * BK * 2 * 2;
        for (int c2 = 0; c2 < nk2; ++c2, ++b2j) {
          const int st = b2j & 1;
          if (b2j >= 2) mbar_wait(&b2_empty[st], ((b2j >> 1) - 1) & 1);
          mbar_expect_tx(&b2_full[st], bytes2);
          bulk_g2s(sB2 + st * b2_b, pool8 + 4 * t.b2_off + (int64_t)c2 * bytes2, bytes2, &b2_full[st]);
        }
      }
    }
  } else if (warp == TCW_RW) {
    // ---------------- MMA issuer
    if (lane == 0) {
      int j = 0, b2j = 0, i = 0;
      for (int ct = blockIdx.x; ct < ntask; ct += G, ++i) {
        const LrTcTask t = tasks[ct];
        const int N1 = t.n1, N2 = t.n2, K1 = 2 * t.T, nk2 = (N1 + BK - 1) / BK;
        const uint32_t idesc1 = idesc_bf16(N1);
        for (int c = 0; c < t.nk1; ++c, ++j) {
          const int st = j % S1;
          { const long long T0_ = dbg ? clock64() : 0; mbar_wait(&a_full[st], (j / S1) & 1); if (dbg) m_a += clock64() - T0_; }
          { const long long T0_ = dbg ? clock64() : 0; mbar_wait(&b_full[st], (j / S1) & 1); if (dbg) m_b += clock64() - T0_; }
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
          const uint8_t* sA = sbase + st * stage_b;
          const uint32_t a_hi = smem_u32(sA), a_lo = a_hi + A_PL;
          const uint32_t b_hi = smem_u32(sA + 2 * A_PL), b_lo = b_hi + N1 * BK * 2;
#pragma unroll
          for (int s = 0; s < BK / 16; ++s) {
            if (c * BK + 16 * s >= K1) break;
            const uint32_t ao = (uint32_t)(s * 2 * 16 * 128), bo = (uint32_t)(s * 2 * (N1 / 8) * 128);
            const uint64_t Ah = make_desc(a_hi + ao, 16 * 128, 128), Al = make_desc(a_lo + ao, 16 * 128, 128);
            const uint64_t Bh = make_desc(b_hi + bo, (N1 / 8) * 128, 128), Bl = make_desc(b_lo + bo, (N1 / 8) * 128, 128);
            mma_bf16(tmem, Ah, Bh, idesc1, (c > 0 || s > 0) ? 1u : 0u);
            mma_bf16(tmem, Ah, Bl, idesc1, 1u);
            mma_bf16(tmem, Al, Bh, idesc1, 1u);
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                           smem_u32(&empty[st]))
                       : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         smem_u32(&d1_full))
                     : "memory");
        { const long long T0_ = dbg ? clock64() : 0; mbar_wait(&a2_full, i & 1); if (dbg) m_a2 += clock64() - T0_; }
        if (i >= 1) { const long long T0_ = dbg ? clock64() : 0; mbar_wait(&y_free, (i - 1) & 1); if (dbg) m_y += clock64() - T0_; }
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        for (int c2 = 0; c2 < nk2; ++c2, ++b2j) {
          const int st = b2j & 1;
          { const long long T0_ = dbg ? clock64() : 0; mbar_wait(&b2_full[st], (b2j >> 1) & 1); if (dbg) m_b2 += clock64() - T0_; }
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
          const uint32_t b_hi = smem_u32(sB2 + st * b2_b), b_lo = b_hi + N2 * BK * 2;
          const uint32_t a_hi = smem_u32(sA2 + c2 * 2 * A_PL), a_lo = a_hi + A_PL;
#pragma unroll
          for (int s = 0; s < BK / 16; ++s) {
            if (c2 * BK + 16 * s >= N1) break;
            const uint32_t ao = (uint32_t)(s * 2 * 16 * 128), bo = (uint32_t)(s * 2 * (N2 / 8) * 128);
            const uint64_t Ah = make_desc(a_hi + ao, 16 * 128, 128), Al = make_desc(a_lo + ao, 16 * 128, 128);
            for (int n0 = 0; n0 < N2; n0 += 256) {
              const int nn = min(256, N2 - n0);
              const uint32_t idesc = idesc_bf16(nn);
              const uint32_t no = (uint32_t)((n0 / 8) * 128);
              const uint64_t Bh = make_desc(b_hi + bo + no, (N2 / 8) * 128, 128);
              const uint64_t Bl = make_desc(b_lo + bo + no, (N2 / 8) * 128, 128);
              mma_bf16(tY + n0, Ah, Bh, idesc, (c2 > 0 || s > 0) ? 1u : 0u);
              mma_bf16(tY + n0, Ah, Bl, idesc, 1u);
              mma_bf16(tY + n0, Al, Bh, idesc, 1u);
            }
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                           smem_u32(&b2_empty[st]))
                       : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         smem_u32(&d2_full))
                     : "memory");
      }
    }
  } else {
    // ---------------- row warps: thread (row = tid & 127, half h = tid >> 7); half h gathers the
    // k-groups {2h, 2h+1} (8 bf16 each) of each 32-element job from both planes and converts /
    // drains the 16-column TMEM blocks b ≡ h (mod 2)
    const int row = tid & 127, h = tid >> 7;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    int it = blockIdx.x, ic = 0, js = 0;
    LrTcTask ti = tasks[it];
    int64_t isp = row < ti.op_count ? 2 * src_off[ti.op_begin + row] : -1;   // bf16 element offset
    auto issue_next = [&]() {
      if (it < ntask) {
        const int st = js % S1;
        if (js >= S1) { const long long T0_ = dbg ? clock64() : 0; mbar_wait(&empty[st], ((js / S1) - 1) & 1); if (dbg) r_e += clock64() - T0_; }
        uint8_t* sA = sbase + st * stage_b;
        const int K2 = 2 * ti.T;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int kg = 2 * h + q;
          const int k = ic * BK + 8 * kg;
          const int nb = isp >= 0 ? 2 * min(8, max(0, K2 - k)) : 0;
          const int so = ((kg * 16 + (row >> 3)) * 8 + (row & 7)) * 16;
          cp16z(sA + so, nb ? (const void*)(shi + isp + k) : (const void*)shi, nb);
          cp16z(sA + A_PL + so, nb ? (const void*)(slo + isp + k) : (const void*)slo, nb);
        }
        ++js;
        if (++ic == ti.nk1) {
          ic = 0;
          it += G;
          if (it < ntask) {
            ti = tasks[it];
            isp = row < ti.op_count ? 2 * src_off[ti.op_begin + row] : -1;
          }
        }
      }
      asm volatile("cp.async.commit_group;\n" ::);
    };
    for (int q = 0; q < LA; ++q) issue_next();
    int jc = 0, i = 0;
    LrTcTask tp{};
    auto drain = [&](const LrTcTask& t) {
      float2* d = row < t.op_count ? dst + dst_off[t.op_begin + row] : nullptr;
      for (int c0 = 16 * h; c0 < t.n2; c0 += 32) {
        float w[16];
        tmem_ld16(tY + lane_base + c0, w);
        if (d) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int r = c0 / 2 + 2 * q;   // complex rows (r, r+1); r+1 = T is the padding slot
            if (r < t.T)
              atomicAdd(reinterpret_cast<float4*>(d + r), make_float4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]));
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
      mbar_arrive(&y_free);
    };
    for (int ct = blockIdx.x; ct < ntask; ct += G, ++i) {
      const LrTcTask t = tasks[ct];
      if (dbg) ++ntk;
      for (int c = 0; c < t.nk1; ++c, ++jc) {
        { const long long T1_ = dbg ? clock64() : 0; issue_next(); if (dbg) r_is += clock64() - T1_; }
        { const long long T0_ = dbg ? clock64() : 0;
          asm volatile("cp.async.wait_group %0;\n" ::"n"(LA) : "memory");
          if (dbg) r_g += clock64() - T0_; }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_arrive(&a_full[jc % S1]);
      }
      if (i >= 1) {                                // D2 of the previous task → destination states
        { const long long T0_ = dbg ? clock64() : 0; mbar_wait(&d2_full, (i - 1) & 1); if (dbg) r_d2 += clock64() - T0_; }
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        { const long long T0_ = dbg ? clock64() : 0; drain(tp); if (dbg) r_dr += clock64() - T0_; }
      }
      { const long long T0_ = dbg ? clock64() : 0; mbar_wait(&d1_full, i & 1); if (dbg) r_d1 += clock64() - T0_; }
      const long long T2_ = dbg ? clock64() : 0;
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      // D1 (fp32, row = op, columns = 2r interleaved) → bf16 hi / lo phase-2 A operand
      for (int c0 = 16 * h; c0 < t.n1; c0 += 32) {
        float w[16];
        tmem_ld16(tmem + lane_base + c0, w);
        uint8_t* ch = sA2 + (c0 / BK) * 2 * A_PL;
#pragma unroll
        for (int g8 = 0; g8 < 2; ++g8) {
          const int kg = ((c0 % BK) >> 3) + g8;
          uint4 hi, lo;
          split8(w + 8 * g8, hi, lo);
          const int so = ((kg * 16 + (row >> 3)) * 8 + (row & 7)) * 16;
          *reinterpret_cast<uint4*>(ch + so) = hi;
          *reinterpret_cast<uint4*>(ch + A_PL + so) = lo;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
      mbar_arrive(&a2_full);
      if (dbg) r_cv += clock64() - T2_;
      tp = t;
    }
    if (i >= 1) {
      mbar_wait(&d2_full, (i - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      drain(tp);
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  }
  if (dbg && lane == 0) {
    const long long tt = clock64() - t_start;
    if (warp == TCW_RW + 1) printf("[m2l_bf cta0] TMA: total %lld, wait empty %lld, wait b2_empty %lld\n", tt, tp_e, tp_b2);
    if (warp == TCW_RW)
      printf("[m2l_bf cta0] MMA: total %lld, wait a_full %lld, b_full %lld, a2_full %lld, y_free %lld, b2_full %lld\n", tt,
             m_a, m_b, m_a2, m_y, m_b2);
    if (warp == 0)
      printf("[m2l_bf cta0] ROW: tasks %lld total %lld, issue %lld (of which wait empty %lld), cp.async wait %lld, wait d2 %lld, "
             "drain %lld, wait d1 %lld, convert %lld\n", ntk, tt, r_is, r_e, r_g, r_d2, r_dr, r_d1, r_cv);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(ncols));
}

// plan of one k_m2l_bf launch: ring stages of one 32-element job (A hi|lo 16 KB + B1 hi|lo),
// a 2-stage B2 ring and the phase-2 A region, ≤ 220 KB
LrTcPlan m2l_bf_plan(int n1max, int n2max) {
  LrTcPlan pl;
  pl.stage_fl = (2 * 128 * BK * 2 + n1max * BK * 2 * 2) / 4;   // (in floats)
  pl.b2_fl = (n2max * BK * 2 * 2) / 4;
  const size_t a2 = (size_t)((n1max + BK - 1) / BK) * 2 * 128 * BK * 2 / 4;
  const size_t cap = (220 * 1024 - 1024) / 4 - 2 * (size_t)pl.b2_fl - a2;
  const int s = (int)(cap / pl.stage_fl);
  pl.stages = s >= 8 ? 8 : (s >= 6 ? 6 : (s >= 5 ? 5 : (s >= 4 ? 4 : 3)));
  pl.smem = ((size_t)pl.stages * pl.stage_fl + 2 * (size_t)pl.b2_fl + a2) * 4 + 1024;
  pl.ncols = tmem_cols(n1max + n2max);
  pl.n1max = n1max;
  return pl;
}
cudaError_t m2l_bf_prepare() {
  if (getenv("FDA_M2L_DBG")) {
    const int one = 1;
    cudaMemcpyToSymbol(g_m2l_dbg, &one, sizeof(int));
  }
  cudaError_t e = cudaFuncSetAttribute(k_m2l_bf<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_m2l_bf<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_m2l_bf<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_m2l_bf<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_m2l_bf<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  return e;
}
void launch_m2l_bf(int ntask, const LrTcTask* tasks, const int64_t* src_off, const int64_t* dst_off,
                   const float* tcpool, const __nv_bfloat16* shi, const __nv_bfloat16* slo, float2* dst,
                   const LrTcPlan& pl, int grid, cudaStream_t s) {
  if (ntask <= 0) return;
#define TBF(S)                                                                                                   \
  k_m2l_bf<S><<<grid, TCW_NT, pl.smem, s>>>(tasks, ntask, src_off, dst_off, tcpool, shi, slo, dst, pl.stage_fl * 4, \
                                         pl.b2_fl * 4, pl.n1max, pl.ncols)
  switch (pl.stages) {
    case 8: TBF(8); break;
    case 6: TBF(6); break;
    case 5: TBF(5); break;
    case 4: TBF(4); break;
    default: TBF(3); break;
  }
#undef TBF
}

// states → bf16 hi / lo planes (one thread per float; the planes share the states' offsets ×2)
__global__ void k_split_bf16(const float* __restrict__ x, int64_t n, __nv_bfloat16* __restrict__ hi,
                             __nv_bfloat16* __restrict__ lo) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float v = x[i];
  const __nv_bfloat16 h = __float2bfloat16_rn(v);
  hi[i] = h;
  lo[i] = __float2bfloat16_rn(v - __bfloat162float(h));
}
void launch_split_bf16(const float* x, int64_t n, __nv_bfloat16* hi, __nv_bfloat16* lo, cudaStream_t s) {
  if (n > 0) k_split_bf16<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, n, hi, lo);
}

// ---------------------------------------------------------------------------
// Dense translations in BF16x3 on tcgen05 (k_xlate_bf; SURVEY §8(a) a3-a5, M2M / L2L / dense
// M2L, Steps 2-3 P:458-499):  dst[:, op] += M · src[:, op]  for ≤ 128 ops sharing M (R × C).
// The ops are the M = 128 rows (TMEM lanes) and the matrix is the B operand, as in phase 1 of
// k_m2l_bf: D (128 × N) = S (128 × 2C) · A_Mᵀ, A_M = real interleaved 2R × 2C form of M (N =
// 2R padded to 16 ≤ 256), so each row of D is one op's interleaved complex result.
//  * A: the source states, pre-split into bf16 hi / lo planes (engine.cu: k_split_bf16 once per
//    level), gathered by the row warps with 16-byte cp.async straight into the canonical K-major
//    layout, S − 2 ring jobs (32 K elements each) ahead;
//  * B: A_Mᵀ as bf16 hi / lo tiles (k_tc_layout kind 2), streamed by the TMA engine (warp 9);
//  * MMA warp (8): per job 2 k-steps × (hi·hi + hi·lo + lo·hi), kind::f16, fp32 accumulation;
//  * two TMEM accumulator sets: the MMAs of task i+1 run while the row warps drain task i
//    (tcgen05.ld of the op's row → 16-byte vector atomics into the destination state).
// No phase 2 and no in-shared-memory split: the row warps only gather and drain.
template <int S>
__global__ void __launch_bounds__(TCW_NT, 1) k_xlate_bf(const XbfTask* __restrict__ tasks, int ntask,
                                                     const int64_t* __restrict__ src_off,
                                                     const int64_t* __restrict__ dst_off,
                                                     const float* __restrict__ tcpool,
                                                     const __nv_bfloat16* __restrict__ shi,
                                                     const __nv_bfloat16* __restrict__ slo, float2* __restrict__ dst,
                                                     int stage_b, int nmax, uint32_t ncols) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sbase = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t a_full[S], b_full[S], empty[S], d_full[2], d_free[2];
  __shared__ uint32_t tmem_base_sh;
  constexpr int LA = S >= 6 ? S - 3 : S - 2;
  constexpr int A_PL = 128 * BK * 2;               // bytes of one A plane (hi or lo) per job
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x;
  const uint8_t* pool8 = reinterpret_cast<const uint8_t*>(tcpool);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  if (tid == 0) {
    for (int q = 0; q < S; ++q) {
      mbar_init(&a_full[q], 32 * TCW_RW);
      mbar_init(&b_full[q], 1);
      mbar_init(&empty[q], 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&d_full[q], 1);
      mbar_init(&d_free[q], 32 * TCW_RW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = tmem_base_sh;

  if (warp == TCW_RW + 1) {
    // ---------------- TMA producer: the B tile of every ring job
    if (lane == 0) {
      int j = 0;
      for (int ct = blockIdx.x; ct < ntask; ct += G) {
        const XbfTask t = tasks[ct];
        const uint32_t bytes = (uint32_t)t.n * BK * 2 * 2;
        for (int c = 0; c < t.nk; ++c, ++j) {
          const int st = j % S;
          if (j >= S) mbar_wait(&empty[st], ((j / S) - 1) & 1);
          mbar_expect_tx(&b_full[st], bytes);
          bulk_g2s(sbase + st * stage_b + 2 * A_PL, pool8 + 4 * t.b_off + (int64_t)c * bytes, bytes, &b_full[st]);
        }
      }
    }
  } else if (warp == TCW_RW) {
    // ---------------- MMA issuer: task i accumulates into TMEM set i & 1
    if (lane == 0) {
      int j = 0, i = 0;
      for (int ct = blockIdx.x; ct < ntask; ct += G, ++i) {
        const XbfTask t = tasks[ct];
        const int N = t.n, K2 = 2 * t.C;
        const uint32_t idesc = idesc_bf16(N);
        const uint32_t td = tmem + (uint32_t)((i & 1) * nmax);
        if (i >= 2) mbar_wait(&d_free[i & 1], ((i - 2) >> 1) & 1);   // task i-2 drained
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        for (int c = 0; c < t.nk; ++c, ++j) {
          const int st = j % S;
          mbar_wait(&a_full[st], (j / S) & 1);
          mbar_wait(&b_full[st], (j / S) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
          const uint8_t* sA = sbase + st * stage_b;
          const uint32_t a_hi = smem_u32(sA), a_lo = a_hi + A_PL;
          const uint32_t b_hi = smem_u32(sA + 2 * A_PL), b_lo = b_hi + N * BK * 2;
#pragma unroll
          for (int s2 = 0; s2 < BK / 16; ++s2) {
            if (c * BK + 16 * s2 >= K2) break;
            const uint32_t ao = (uint32_t)(s2 * 2 * 16 * 128), bo = (uint32_t)(s2 * 2 * (N / 8) * 128);
            const uint64_t Ah = make_desc(a_hi + ao, 16 * 128, 128), Al = make_desc(a_lo + ao, 16 * 128, 128);
            const uint64_t Bh = make_desc(b_hi + bo, (N / 8) * 128, 128), Bl = make_desc(b_lo + bo, (N / 8) * 128, 128);
            mma_bf16(td, Ah, Bh, idesc, (c > 0 || s2 > 0) ? 1u : 0u);
            mma_bf16(td, Ah, Bl, idesc, 1u);
            mma_bf16(td, Al, Bh, idesc, 1u);
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                           smem_u32(&empty[st]))
                       : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         smem_u32(&d_full[i & 1]))
                     : "memory");
      }
    }
  } else {
    // ---------------- row warps: thread (row = tid & 127, half h = tid >> 7); half h gathers the
    // k-groups {2h, 2h+1} of each job from both planes and drains the 16-column TMEM blocks ≡ h (mod 2)
    const int row = tid & 127, h = tid >> 7;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    int it = blockIdx.x, ic = 0, js = 0;
    XbfTask ti = tasks[it];
    int64_t isp = row < ti.op_count ? 2 * src_off[ti.op_begin + row] : -1;   // bf16 element offset
    auto issue_next = [&]() {
      if (it < ntask) {
        const int st = js % S;
        if (js >= S) mbar_wait(&empty[st], ((js / S) - 1) & 1);
        uint8_t* sA = sbase + st * stage_b;
        const int K2 = 2 * ti.C;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int kg = 2 * h + q;
          const int k = ic * BK + 8 * kg;
          const int nb = isp >= 0 ? 2 * min(8, max(0, K2 - k)) : 0;
          const int so = ((kg * 16 + (row >> 3)) * 8 + (row & 7)) * 16;
          cp16z(sA + so, nb ? (const void*)(shi + isp + k) : (const void*)shi, nb);
          cp16z(sA + A_PL + so, nb ? (const void*)(slo + isp + k) : (const void*)slo, nb);
        }
        ++js;
        if (++ic == ti.nk) {
          ic = 0;
          it += G;
          if (it < ntask) {
            ti = tasks[it];
            isp = row < ti.op_count ? 2 * src_off[ti.op_begin + row] : -1;
          }
        }
      }
      asm volatile("cp.async.commit_group;\n" ::);
    };
    auto drain = [&](const XbfTask& t, int i) {
      mbar_wait(&d_full[i & 1], (i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      const uint32_t td = tmem + (uint32_t)((i & 1) * nmax);
      float2* d = row < t.op_count ? dst + dst_off[t.op_begin + row] : nullptr;
      for (int c0 = 16 * h; c0 < t.n; c0 += 32) {
        float w[16];
        tmem_ld16(td + lane_base + c0, w);
        if (d) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int r = c0 / 2 + 2 * q;   // complex rows (r, r+1); r+1 = R is the padding slot
            if (r < t.R)
              atomicAdd(reinterpret_cast<float4*>(d + r), make_float4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]));
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
      mbar_arrive(&d_free[i & 1]);
    };
    for (int q = 0; q < LA; ++q) issue_next();
    int jc = 0, i = 0;
    XbfTask tp{};
    for (int ct = blockIdx.x; ct < ntask; ct += G, ++i) {
      const XbfTask t = tasks[ct];
      for (int c = 0; c < t.nk; ++c, ++jc) {
        issue_next();
        asm volatile("cp.async.wait_group %0;\n" ::"n"(LA) : "memory");
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_arrive(&a_full[jc % S]);
      }
      if (i >= 1) drain(tp, i - 1);   // task i-1's accumulators while task i's MMAs run
      tp = t;
    }
    if (i >= 1) drain(tp, i - 1);
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(ncols));
}

// plan of one k_xlate_bf launch: S ring stages of one 32-element job (A hi|lo 16 KB + B hi|lo),
// ≤ 220 KB; two TMEM accumulator sets of nmax columns
LrTcPlan xlate_bf_plan(int nmax) {
  LrTcPlan pl;
  pl.stage_fl = (2 * 128 * BK * 2 + nmax * BK * 2 * 2) / 4;   // (in floats)
  const size_t cap = (220 * 1024 - 1024) / 4;
  const int s = (int)(cap / pl.stage_fl);
  pl.stages = s >= 8 ? 8 : (s >= 6 ? 6 : (s >= 5 ? 5 : (s >= 4 ? 4 : 3)));
  pl.smem = (size_t)pl.stages * pl.stage_fl * 4 + 1024;
  pl.ncols = tmem_cols(2 * nmax);
  pl.n1max = nmax;
  return pl;
}
cudaError_t xlate_bf_prepare() {
  cudaError_t e = cudaFuncSetAttribute(k_xlate_bf<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_xlate_bf<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_xlate_bf<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_xlate_bf<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_xlate_bf<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  return e;
}
void launch_xlate_bf(int ntask, const XbfTask* tasks, const int64_t* src_off, const int64_t* dst_off,
                     const float* tcpool, const __nv_bfloat16* shi, const __nv_bfloat16* slo, float2* dst,
                     const LrTcPlan& pl, int grid, cudaStream_t s) {
  if (ntask <= 0) return;
#define XBF(S)                                                                                                  \
  k_xlate_bf<S><<<grid, TCW_NT, pl.smem, s>>>(tasks, ntask, src_off, dst_off, tcpool, shi, slo, dst,            \
                                           pl.stage_fl * 4, pl.n1max, pl.ncols)
  switch (pl.stages) {
    case 8: XBF(8); break;
    case 6: XBF(6); break;
    case 5: XBF(5); break;
    case 4: XBF(4); break;
    default: XBF(3); break;
  }
#undef XBF
}

// ---------------------------------------------------------------------------
// Warp-specialised persistent form of the translation kernel (k_xlate_tcw):
// the same product (dst[:, op] += M · src[:, op] in interleaved real form,
// 3xTF32, N = 128 ops per task, TILES ≤ 2 row tiles) with the roles of
// k_m2l_tcw — row warps 0-7 gather the B operand (two threads per op, two
// k-groups each), split it in place and drain the accumulators; warp 8 issues
// the MMAs; warp 9 streams the A tiles with the TMA engine.  TMEM holds two
// accumulator sets (2 × TILES × 128 columns), so task i+1's MMAs run while
// the row warps drain task i: a warp reads 32 real rows × 16 ops per
// tcgen05.ld, pairs (Re, Im) of a complex row with one shuffle and adds them
// with 8-byte atomics, 16 lanes covering 16 consecutive complex rows of one op.
template <int S, int TILES>
__global__ void __launch_bounds__(TCW_NT, 1) k_xlate_tcw(const TcTask* __restrict__ tasks, int ntask,
                                                       const int64_t* __restrict__ src_off,
                                                       const int64_t* __restrict__ dst_off,
                                                       const float* __restrict__ tcpool,
                                                       const float2* __restrict__ src, float2* __restrict__ dst) {
  constexpr int N = 128;
  constexpr int A_FL = TILES * 2 * A_TILE;         // A floats per stage (hi | lo per tile)
  constexpr int STAGE_FL = A_FL + 2 * N * KC;      // + B hi | lo
  constexpr int LA = S >= 6 ? S - 3 : S - 2;
  constexpr uint32_t NCOLS = tmem_cols(2 * TILES * N);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  float* sbase = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t a_full[S], b_full[S], empty[S], d_full[2], y_free[2];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(NCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  if (tid == 0) {
    for (int q = 0; q < S; ++q) {
      mbar_init(&a_full[q], 1);
      mbar_init(&b_full[q], 32 * TCW_RW);
      mbar_init(&empty[q], 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&d_full[q], 1);
      mbar_init(&y_free[q], 32 * TCW_RW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = tmem_base_sh;

  if (warp == TCW_RW + 1) {
    // ---------------- TMA producer: the A tiles of every job
    if (lane == 0) {
      int j = 0;
      for (int ct = blockIdx.x; ct < ntask; ct += G) {
        const TcTask t = tasks[ct];
        for (int cg = t.kc0; cg < t.kc1; ++cg, ++j) {
          const int st = j % S;
          if (j >= S) mbar_wait(&empty[st], ((j / S) - 1) & 1);
          mbar_expect_tx(&a_full[st], (uint32_t)(TILES * 2 * A_TILE * 4));
#pragma unroll
          for (int ti = 0; ti < TILES; ++ti)
            bulk_g2s(sbase + st * STAGE_FL + ti * 2 * A_TILE, tcpool + t.a_off + ((int64_t)ti * t.nkc + cg) * 2 * A_TILE,
                     2 * A_TILE * 4, &a_full[st]);
        }
      }
    }
  } else if (warp == TCW_RW) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc<N>();
      int j = 0, i = 0;
      for (int ct = blockIdx.x; ct < ntask; ct += G, ++i) {
        const TcTask t = tasks[ct];
        const int b = i & 1;
        if (i >= 2) mbar_wait(&y_free[b], ((i >> 1) - 1) & 1);   // task i-2's accumulators drained
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        for (int cg = t.kc0; cg < t.kc1; ++cg, ++j) {
          const int st = j % S;
          mbar_wait(&a_full[st], (j / S) & 1);
          mbar_wait(&b_full[st], (j / S) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
          float* sA = sbase + st * STAGE_FL;
          const uint32_t b_hi = smem_u32(sA + A_FL), b_lo = b_hi + N * KC * 4;
#pragma unroll
          for (int s = 0; s < KC / 8; ++s) {
            const uint32_t bo = (uint32_t)(2 * s * (N / 8) * 128);
            const uint64_t Bh = make_desc(b_hi + bo, (N / 8) * 128, 128), Bl = make_desc(b_lo + bo, (N / 8) * 128, 128);
#pragma unroll
            for (int ti = 0; ti < TILES; ++ti) {
              const uint32_t a_hi = smem_u32(sA + ti * 2 * A_TILE), a_lo = a_hi + A_TILE * 4;
              const uint32_t ao = (uint32_t)(2 * s * 16 * 128);
              const uint64_t Ah = make_desc(a_hi + ao, 16 * 128, 128), Al = make_desc(a_lo + ao, 16 * 128, 128);
              const uint32_t d = tmem + (uint32_t)((b * TILES + ti) * N);
              mma_tf32(d, Ah, Bh, idesc, (cg > t.kc0 || s > 0) ? 1u : 0u);
              mma_tf32(d, Ah, Bl, idesc, 1u);
              mma_tf32(d, Al, Bh, idesc, 1u);
            }
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                           smem_u32(&empty[st]))
                       : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         smem_u32(&d_full[b]))
                     : "memory");
      }
    }
  } else {
    // ---------------- row warps: op = tid & 127, half h = tid >> 7 (k-groups 2h, 2h+1)
    const int op = tid & 127, h = tid >> 7;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    int it = blockIdx.x, js = 0;
    TcTask ti = tasks[it];
    int cg_i = ti.kc0;
    const float* isp = op < ti.op_count ? reinterpret_cast<const float*>(src) + 2 * src_off[ti.op_begin + op] : nullptr;
    auto issue_next = [&]() {
      if (it < ntask) {
        const int st = js % S;
        if (js >= S) mbar_wait(&empty[st], ((js / S) - 1) & 1);
        float* sB = sbase + st * STAGE_FL + A_FL;
        const int K2 = 2 * ti.C;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int kg = 2 * h + q;
          const int k = cg_i * KC + 4 * kg;
          const int nb = isp ? 4 * min(4, max(0, K2 - k)) : 0;
          cp16z(sB + ((kg * (N / 8) + (op >> 3)) * 8 + (op & 7)) * 4, nb ? (const void*)(isp + k) : (const void*)src, nb);
        }
        ++js;
        if (++cg_i == ti.kc1) {
          it += G;
          if (it < ntask) {
            ti = tasks[it];
            cg_i = ti.kc0;
            isp = op < ti.op_count ? reinterpret_cast<const float*>(src) + 2 * src_off[ti.op_begin + op] : nullptr;
          }
        }
      }
      asm volatile("cp.async.commit_group;\n" ::);
    };
    for (int q = 0; q < LA; ++q) issue_next();
    auto drain = [&](const TcTask& t, int b) {
      // lane = real row rr of the tile: complex row rr >> 1, Re (even) / Im (odd)
      for (int tt = 0; tt < t.ntile; ++tt)
        for (int c0 = 16 * h; c0 < N; c0 += 32) {
          float w[16];
          tmem_ld16(tmem + lane_base + (uint32_t)((b * TILES + tt) * N + c0), w);
          const int ci = (128 * tt + 32 * (warp & 3) + lane) >> 1;
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const float im = __shfl_xor_sync(0xffffffffu, w[q], 1);
            const int o = c0 + q;
            if ((lane & 1) == 0 && o < t.op_count && ci < t.R)
              atomicAdd(dst + dst_off[t.op_begin + o] + ci, make_float2(w[q], im));
          }
        }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
      mbar_arrive(&y_free[b]);
    };
    int jc = 0, i = 0;
    TcTask tp{};
    for (int ct = blockIdx.x; ct < ntask; ct += G, ++i) {
      const TcTask t = tasks[ct];
      for (int cg = t.kc0; cg < t.kc1; ++cg, ++jc) {
        issue_next();
        asm volatile("cp.async.wait_group %0;\n" ::"n"(LA) : "memory");
        float* sB = sbase + (jc % S) * STAGE_FL + A_FL;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int kg = 2 * h + q;
          const int idx = ((kg * (N / 8) + (op >> 3)) * 8 + (op & 7)) * 4;
          const float4 v = *reinterpret_cast<const float4*>(sB + idx);
          const float4 hv = tf32_hi4(v);
          *reinterpret_cast<float4*>(sB + idx) = hv;
          *reinterpret_cast<float4*>(sB + N * KC + idx) = make_float4(v.x - hv.x, v.y - hv.y, v.z - hv.z, v.w - hv.w);
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_arrive(&b_full[jc % S]);
      }
      if (i >= 1) {
        mbar_wait(&d_full[(i - 1) & 1], ((i - 1) >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        drain(tp, (i - 1) & 1);
      }
      tp = t;
    }
    if (i >= 1) {
      mbar_wait(&d_full[(i - 1) & 1], ((i - 1) >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      drain(tp, (i - 1) & 1);
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(NCOLS));
}

template <int S, int TILES>
size_t xlate_tcw_smem() {
  return (size_t)S * (TILES * 2 * A_TILE + 2 * 128 * KC) * 4 + 1024;
}
cudaError_t xlate_tcw_prepare() {
  cudaError_t e = cudaFuncSetAttribute(k_xlate_tcw<6, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)xlate_tcw_smem<6, 1>());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_xlate_tcw<4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xlate_tcw_smem<4, 2>());
  return e;
}
// persistent: grid = min(ntask, #SMs); tasks sorted longest first on the host
void launch_xlate_tcw(int tiles, int ntask, const TcTask* tasks, const int64_t* src_off, const int64_t* dst_off,
                      const float* tcpool, const float2* src, float2* dst, int grid, cudaStream_t s) {
  if (ntask <= 0) return;
  if (tiles == 1)
    k_xlate_tcw<6, 1><<<grid, TCW_NT, xlate_tcw_smem<6, 1>(), s>>>(tasks, ntask, src_off, dst_off, tcpool, src, dst);
  else
    k_xlate_tcw<4, 2><<<grid, TCW_NT, xlate_tcw_smem<4, 2>(), s>>>(tasks, ntask, src_off, dst_off, tcpool, src, dst);
}



// tensor-core operand layout (one CTA per matrix job): the real interleaved form of a
// complex matrix M (A[2i][2j] = Re M, A[2i][2j+1] = −Im M, A[2i+1][2j] = Im M,
// A[2i+1][2j+1] = Re M) split into TF32 hi = rna(x) and lo = rna(x − hi), written into the
// canonical K-major no-swizzle UMMA layout (core matrices of 8 rows × 16 B)
__device__ __forceinline__ float tf32_rna_dev(float x) {
  uint32_t u = __float_as_uint(x);
  if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;   // round to nearest, ties away
  return __uint_as_float(u);
}
__global__ void k_tc_layout(const TcLayoutJob* __restrict__ jobs, const float2* __restrict__ pool,
                            float* __restrict__ tcpool) {
  const TcLayoutJob jb = jobs[blockIdx.x];
  const float2* M = pool + jb.src;
  float* base = tcpool + jb.dst;
  if (jb.kind == 0) {
    const int64_t total = (int64_t)jb.a * jb.nkc * 128 * TC_KC;
    for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
      const int k = (int)(e % TC_KC), r = (int)((e / TC_KC) % 128);
      const int kc = (int)((e / (128 * TC_KC)) % jb.nkc), ti = (int)(e / ((int64_t)128 * TC_KC * jb.nkc));
      const int gr = 128 * ti + r, i = gr >> 1, gk = kc * TC_KC + k, j = gk >> 1;
      float x = 0.0f;
      if (i < jb.R && j < jb.C) {
        const float2 v = M[(int64_t)j * jb.R + i];
        x = (gr & 1) == 0 ? ((gk & 1) == 0 ? v.x : -v.y) : ((gk & 1) == 0 ? v.y : v.x);
      }
      const float h = tf32_rna_dev(x), l = tf32_rna_dev(x - h);
      float* hi = base + ((int64_t)ti * jb.nkc + kc) * 2 * 128 * TC_KC;
      const int idx = (((k >> 2) * 16 + (r >> 3)) * 8 + (r & 7)) * 4 + (k & 3);
      hi[idx] = h;
      hi[128 * TC_KC + idx] = l;
    }
  } else if (jb.kind == 2) {
    // bf16 B operand: per 32-element K chunk, per block of rb rows (jb.pad; 0 = all nrp rows),
    // [hi: nb × 32 | lo: nb × 32] (canonical K-major, core matrices of 8 rows × 16 B = 8 bf16)
    const int nrp = jb.a, rb = jb.pad > 0 ? jb.pad : jb.a;
    __nv_bfloat16* b16 = reinterpret_cast<__nv_bfloat16*>(base);
    const int64_t total = (int64_t)jb.nkc * nrp * 32;
    for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
      const int k = (int)(e % 32), gr = (int)((e / 32) % nrp), kc = (int)(e / ((int64_t)32 * nrp));
      const int i = gr >> 1, gk = kc * 32 + k, j = gk >> 1;
      if (gr >= 2 * jb.R || j >= jb.C) continue;
      const float2 v = M[(int64_t)j * jb.R + i];
      const float x = (gr & 1) == 0 ? ((gk & 1) == 0 ? v.x : -v.y) : ((gk & 1) == 0 ? v.y : v.x);
      const __nv_bfloat16 h = __float2bfloat16_rn(x), l = __float2bfloat16_rn(x - __bfloat162float(h));
      const int blk = gr / rb, lr = gr - blk * rb, nb = min(rb, nrp - blk * rb);
      __nv_bfloat16* hi = b16 + (int64_t)kc * 2 * nrp * 32 + (int64_t)blk * rb * 64;
      const int64_t idx = ((int64_t)((k >> 3) * (nb / 8) + (lr >> 3)) * 8 + (lr & 7)) * 8 + (k & 7);
      hi[idx] = h;
      hi[(int64_t)nb * 32 + idx] = l;
    }
  } else {
    const int nrp = jb.a;
    const int64_t total = (int64_t)jb.nkc * nrp * TC_KC;
    for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
      const int k = (int)(e % TC_KC), gr = (int)((e / TC_KC) % nrp), kc = (int)(e / ((int64_t)TC_KC * nrp));
      const int i = gr >> 1, gk = kc * TC_KC + k, j = gk >> 1;
      if (gr >= 2 * jb.R || j >= jb.C) continue;
      const float2 v = M[(int64_t)j * jb.R + i];
      const float x = (gr & 1) == 0 ? ((gk & 1) == 0 ? v.x : -v.y) : ((gk & 1) == 0 ? v.y : v.x);
      const float h = tf32_rna_dev(x), l = tf32_rna_dev(x - h);
      float* hi = base + (int64_t)kc * 2 * nrp * TC_KC;
      const int64_t idx = ((int64_t)((k >> 2) * (nrp / 8) + (gr >> 3)) * 8 + (gr & 7)) * 4 + (k & 3);
      hi[idx] = h;
      hi[(int64_t)nrp * TC_KC + idx] = l;
    }
  }
}
void launch_tc_layout(int njob, const TcLayoutJob* jobs, const float2* pool, float* tcpool, cudaStream_t s) {
  if (njob > 0) k_tc_layout<<<njob, 256, 0, s>>>(jobs, pool, tcpool);
}

namespace {
template <int N, int TILES, int S, int MB>
cudaError_t tc_attr() {
  return cudaFuncSetAttribute(k_xlate_tc<N, TILES, S, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)TcCfg<N, TILES, S>::SMEM);
}
}  // namespace

// variants (N, tiles, stages, CTAs per SM): 0 (128,1,3,1) 1 (128,2,3,1) 2 (128,3,3,1) 3 (256,1,3,1)
// 4 (256,2,3,1); 5 (128,1,2,3) 6 (128,2,2,2) — the latter two trade pipeline depth for CTAs per SM
#define TC_VARIANTS(X) X(0, 128, 1, 3, 1) X(1, 128, 2, 3, 1) X(2, 128, 3, 3, 1) X(3, 256, 1, 3, 1) \
  X(4, 256, 2, 3, 1) X(5, 128, 1, 2, 3) X(6, 128, 2, 2, 2)

cudaError_t tc_prepare() {
  cudaError_t e = cudaSuccess;
#define TC_ATTR(V, NN, TT, SS, MB) \
  if (e == cudaSuccess) e = tc_attr<NN, TT, SS, MB>();
  TC_VARIANTS(TC_ATTR)
#undef TC_ATTR
  return e;
}

int tc_variant(int n, int tiles, bool multi) {
  if (multi && n == 128 && tiles <= 2) return tiles == 1 ? 5 : 6;
  return n == 256 ? 2 + tiles : tiles - 1;
}
int tc_variant_ops(int v) { return (v == 3 || v == 4) ? 256 : 128; }

void launch_xlate_tc(int variant, int ntask, const TcTask* tasks, const int64_t* src_off, const int64_t* dst_off,
                     const float* tcpool, const float2* src, float2* dst, cudaStream_t s) {
  if (ntask <= 0) return;
#define TC_CASE(V, NN, TT, SS, MB)                                                                           \
  case V:                                                                                                   \
    k_xlate_tc<NN, TT, SS, MB><<<ntask, 128, TcCfg<NN, TT, SS>::SMEM, s>>>(tasks, src_off, dst_off, tcpool, src, \
                                                                          dst);                              \
    break;
  switch (variant) { TC_VARIANTS(TC_CASE) }
#undef TC_CASE
}

}  // namespace fda
