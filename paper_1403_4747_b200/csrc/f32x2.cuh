// Packed fp32 pairs for sm_100a: PTX add/sub/mul/fma .f32x2 → SASS FADD2 /
// FMUL2 / FFMA2.  One instruction carries two lanes of fp32 work, so a kernel
// limited by issue slots (not by the FMA pipe) does the same arithmetic in
// about half the instructions.  Measured on B200 (tools/ubench/ffma2.cu,
// profiles/r01_ubench_ffma2.jsonl): FFMA2 has the same per-lane FMA throughput
// as FFMA (≈65-71 TFLOP/s), i.e. it saves issue, not pipe, cycles.
// ptxas folds a scalar broadcast pack2(a, a) into the .F32 operand form and a
// pairwise negation pack2(-lo, -hi) into the operand's negate modifier.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fda {

struct f2x {
  uint64_t v;
};

__device__ __forceinline__ f2x pack2(float a, float b) {
  f2x r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ f2x bcast2(float a) { return pack2(a, a); }
__device__ __forceinline__ void unpack2(f2x x, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x.v));
}
__device__ __forceinline__ float lo2(f2x x) {
  float a, b;
  unpack2(x, a, b);
  (void)b;
  return a;
}
__device__ __forceinline__ float hi2(f2x x) {
  float a, b;
  unpack2(x, a, b);
  (void)a;
  return b;
}
__device__ __forceinline__ f2x neg2(f2x x) { return pack2(-lo2(x), -hi2(x)); }
__device__ __forceinline__ f2x add2(f2x a, f2x b) {
  f2x r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ f2x sub2(f2x a, f2x b) {
  f2x r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ f2x mul2(f2x a, f2x b) {
  f2x r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ f2x fma2(f2x a, f2x b, f2x c) {
  f2x r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
  return r;
}
__device__ __forceinline__ f2x zero2() { return pack2(0.f, 0.f); }

}  // namespace fda
