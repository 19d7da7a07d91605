// Tensor-core (tcgen05, sm_100a) grouped complex GEMM for the dense FDA
// translations (M2M, L2L, dense M2L).
//
// For one task (one matrix M, R × C complex, ≤ 64 complex rows of it and ≤ 64
// ops sharing it) the CTA computes D[:, n] = M_blk · S[:, n] and accumulates
// D into the destination states with vector atomics, exactly like k_xlate.
// Complex arithmetic is done on real planes:
//   A = [M_r; M_i] (128 × C, real),  P = A·S_r,  Q = A·S_i  (128 × 64, TMEM)
//   D_r = P_top - Q_bot,  D_i = Q_top + P_bot.
// fp32 accuracy from TF32 tensor cores by the 3-term split (3xTF32):
//   A·B ≈ A_hi·B_hi + A_hi·B_lo + A_lo·B_hi,  X_hi = tf32(X), X_lo = tf32(X - X_hi).
// A is pre-split and pre-laid-out on the host in the canonical K-major
// (no-swizzle) UMMA layout — core matrices of 8 rows × 16 bytes — per TC_KC-column
// chunk; the sources are pre-split once per tree level (k_split_states) into
// 16-byte-aligned planes, so the CTA streams both operands with 16-byte
// cp.async and only issues MMAs.  One thread issues the MMAs
// (tcgen05.mma.cta_group::1.kind::tf32, M = 128, N = 64, K = 8), completion is
// tracked by tcgen05.commit on an mbarrier, two shared-memory stages overlap
// the copy of chunk k+1 with the MMAs of chunk k.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"

namespace fda {

namespace {
constexpr int TC_N = 64;                     // ops per task (MMA N)
constexpr int A_TILE = 128 * TC_KC;          // floats per (chunk, hi|lo) A tile
constexpr int B_TILE = TC_N * TC_KC;         // floats per (chunk, plane) B tile
constexpr uint32_t TMEM_COLS = 2 * TC_N;     // P and Q accumulators

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// canonical K-major, no-swizzle UMMA shared-memory descriptor
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
  // base_offset = 0, lbo_mode = 0, layout_type = 0 (SWIZZLE_NONE)
  return d;
}

// instruction descriptor: kind::tf32, D = F32, A/B = TF32, both K-major, M = 128, N = TC_N
__host__ __device__ constexpr uint32_t make_idesc() {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TC_N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
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

__device__ __forceinline__ void cp16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(s)), "l"(g));
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
}  // namespace

// shared memory: 2 stages × (A hi, A lo, B r_hi, r_lo, i_hi, i_lo), 16-byte aligned
constexpr int TC_STAGE_FLOATS = 2 * A_TILE + 4 * B_TILE;
constexpr size_t TC_SMEM = (size_t)2 * TC_STAGE_FLOATS * sizeof(float) + 1024;

__global__ void __launch_bounds__(128, 3) k_xlate_tc(const TcTask* __restrict__ tasks,
                                                     const int64_t* __restrict__ src_off,
                                                     const int64_t* __restrict__ dst_off,
                                                     const float* __restrict__ tcpool,
                                                     const float* __restrict__ srcp, float2* __restrict__ dst) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  float* sbase = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t mbar[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ int64_t soff[TC_N];
  const TcTask t = tasks[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  for (int p = tid; p < TC_N; p += 128) soff[p] = p < t.op_count ? src_off[t.op_begin + p] : -1;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = tmem_base_sh;
  const uint32_t idesc = make_idesc();
  const int nkc = t.nkc;

  for (int kc = 0; kc < nkc; ++kc) {
    const int st = kc & 1;
    if (kc >= 2) mbar_wait(&mbar[st], ((kc - 2) >> 1) & 1);   // MMAs of chunk kc-2 released this stage
    float* sA = sbase + st * TC_STAGE_FLOATS;                 // [hi | lo], A_TILE each
    float* sB = sA + 2 * A_TILE;                              // [r_hi | r_lo | i_hi | i_lo], B_TILE each
    // A: contiguous 2 × A_TILE floats, pre-laid-out → 16-byte async copies
    const float* gA = tcpool + t.a_off + (int64_t)kc * 2 * A_TILE;
    for (int i = tid; i < 2 * A_TILE / 4; i += 128) cp16(sA + 4 * i, gA + 4 * i);
    asm volatile("cp.async.commit_group;\n" ::);
    // B: the sources were pre-split per state into 4 planes [r_hi | r_lo | i_hi | i_lo] of
    // Tp floats each (k_split_states); a core-matrix row (op n, k-group kg) is 16 contiguous
    // bytes of a plane → 16-byte async copies into ((kg·(N/8) + n/8)·8 + n%8)·4
    for (int i = tid; i < 4 * (TC_KC / 4) * TC_N; i += 128) {
      const int plane = i / ((TC_KC / 4) * TC_N), rem = i % ((TC_KC / 4) * TC_N);
      const int kg = rem / TC_N, n = rem % TC_N;
      float* dstp = sB + plane * B_TILE + ((kg * (TC_N / 8) + n / 8) * 8 + (n & 7)) * 4;
      const int64_t so = soff[n];
      if (so >= 0) cp16(dstp, srcp + so + (int64_t)plane * t.Tp + kc * TC_KC + 4 * kg);
      else *reinterpret_cast<float4*>(dstp) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      const uint32_t a_hi = smem_u32(sA), a_lo = smem_u32(sA + A_TILE);
      const uint32_t b0 = smem_u32(sB);
#pragma unroll
      for (int s = 0; s < TC_KC / 8; ++s) {
        // K = 8 per MMA: core-matrix k-groups 2s, 2s+1
        const uint32_t ao = (uint32_t)(2 * s * 16 * 128), bo = (uint32_t)(2 * s * (TC_N / 8) * 128);
        const uint64_t Ahi = make_desc(a_hi + ao, 16 * 128, 128), Alo = make_desc(a_lo + ao, 16 * 128, 128);
        const uint64_t Brh = make_desc(b0 + bo, (TC_N / 8) * 128, 128);
        const uint64_t Brl = make_desc(b0 + 4 * B_TILE + bo, (TC_N / 8) * 128, 128);
        const uint64_t Bih = make_desc(b0 + 8 * B_TILE + bo, (TC_N / 8) * 128, 128);
        const uint64_t Bil = make_desc(b0 + 12 * B_TILE + bo, (TC_N / 8) * 128, 128);
        const uint32_t acc = (kc > 0 || s > 0) ? 1u : 0u;
        mma_tf32(tmem, Ahi, Brh, idesc, acc);            // P = A · S_r
        mma_tf32(tmem, Ahi, Brl, idesc, 1u);
        mma_tf32(tmem, Alo, Brh, idesc, 1u);
        mma_tf32(tmem + TC_N, Ahi, Bih, idesc, acc);     // Q = A · S_i
        mma_tf32(tmem + TC_N, Ahi, Bil, idesc, 1u);
        mma_tf32(tmem + TC_N, Alo, Bih, idesc, 1u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                       smem_u32(&mbar[st]))
                   : "memory");
    }
  }
  mbar_wait(&mbar[(nkc - 1) & 1], ((nkc - 1) >> 1) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);

  // epilogue: warps 2,3 hold rows 64..127 (M_i·S) → shared; warps 0,1 combine and accumulate
  float* sE = sbase;  // [64 rows][2 (P,Q)][TC_N + 1]
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  if (warp >= 2) {
    const int row = (warp - 2) * 32 + lane;
    for (int c0 = 0; c0 < TC_N; c0 += 16) {
      float v[16];
      tmem_ld16(tmem + lane_base + c0, v);
#pragma unroll
      for (int j = 0; j < 16; ++j) sE[(row * 2 + 0) * (TC_N + 1) + c0 + j] = v[j];
      tmem_ld16(tmem + lane_base + TC_N + c0, v);
#pragma unroll
      for (int j = 0; j < 16; ++j) sE[(row * 2 + 1) * (TC_N + 1) + c0 + j] = v[j];
    }
  }
  __syncthreads();
  if (warp < 2) {
    const int row = warp * 32 + lane;       // complex row within the block
    const int grow = t.row0 + row;
    for (int c0 = 0; c0 < TC_N; c0 += 16) {
      float p[16], q[16];
      tmem_ld16(tmem + lane_base + c0, p);
      tmem_ld16(tmem + lane_base + TC_N + c0, q);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int n = c0 + j;
        if (n < t.op_count && grow < t.R) {
          const float pb = sE[(row * 2 + 0) * (TC_N + 1) + n], qb = sE[(row * 2 + 1) * (TC_N + 1) + n];
          atomicAdd(dst + dst_off[t.op_begin + n] + grow, make_float2(p[j] - qb, q[j] + pb));
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
}

size_t tc_smem_bytes() { return TC_SMEM; }

cudaError_t tc_prepare() {
  return cudaFuncSetAttribute(k_xlate_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TC_SMEM);
}

void launch_xlate_tc(int ntask, const TcTask* tasks, const int64_t* src_off, const int64_t* dst_off,
                     const float* tcpool, const float* srcp, float2* dst, cudaStream_t s) {
  if (ntask <= 0) return;
  k_xlate_tc<<<ntask, 128, TC_SMEM, s>>>(tasks, src_off, dst_off, tcpool, srcp, dst);
}

// Pre-split states [s0, s1) for the tensor-core operand B: state s (T complex at
// off[s]) → 4 planes of Tp floats at poff[s]: tf32 hi/lo of the real and the
// imaginary parts, zero-padded to Tp (a multiple of TC_KC).
__global__ void k_split_states(const float2* __restrict__ states, const int64_t* __restrict__ off,
                               const int64_t* __restrict__ poff, int T, int Tp, int64_t s0, int64_t s1,
                               float* __restrict__ planes) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t s = s0 + g / Tp;
  const int k = (int)(g % Tp);
  if (s >= s1) return;
  float2 v = k < T ? states[off[s] + k] : make_float2(0.f, 0.f);
  const uint32_t rh = to_tf32(v.x), ih = to_tf32(v.y);
  const uint32_t rl = to_tf32(v.x - __uint_as_float(rh)), il = to_tf32(v.y - __uint_as_float(ih));
  float* p = planes + poff[s];
  p[k] = __uint_as_float(rh);
  p[Tp + k] = __uint_as_float(rl);
  p[2 * Tp + k] = __uint_as_float(ih);
  p[3 * Tp + k] = __uint_as_float(il);
}

void launch_split_states(const float2* states, const int64_t* off, const int64_t* poff, int T, int Tp, int64_t s0,
                         int64_t s1, float* planes, cudaStream_t s) {
  if (s1 <= s0) return;
  const int64_t n = (s1 - s0) * Tp;
  k_split_states<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(states, off, poff, T, Tp, s0, s1, planes);
}

}  // namespace fda
