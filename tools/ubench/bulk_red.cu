// Microbenchmark: accumulating per-op rows into scattered destination states, the drain of the
// translation kernels.  Each "op" adds a row of W fp32 (2T floats of a complex state) into a
// destination row chosen at random among NS rows (the states).  Three forms:
//   red   : each thread owns one op row and issues W/4 red.global.add.v4.f32 (RED.128) — the
//           current drain of k_m2l_bf / k_xlate_bf
//   bulk  : each thread writes its row (in CH-float chunks) into its own shared-memory staging
//           slot and issues cp.reduce.async.bulk.global.shared::cta.add.f32 per chunk (TMA bulk
//           reduction; the LSU only sees shared stores)
//   store : plain st.global.v4 of the rows (no reduction; an upper bound)
// Reports payload GB/s (ops·W·4 bytes per second).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a bulk_red.cu -o bulk_red
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

constexpr int W = 240;    // floats per row (T = 120 complex)
constexpr int NT = 256;   // threads per CTA (one op row each per iteration)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ float val(int op, int c) { return 1e-3f * (float)((op * 7 + c) & 255); }

__global__ void __launch_bounds__(NT) k_red(float* __restrict__ st, const int* __restrict__ dst, int nops) {
  for (int op = blockIdx.x * NT + threadIdx.x; op < nops; op += gridDim.x * NT) {
    float* d = st + (int64_t)dst[op] * W;
#pragma unroll 4
    for (int c = 0; c < W; c += 4)
      atomicAdd(reinterpret_cast<float4*>(d + c), make_float4(val(op, c), val(op, c + 1), val(op, c + 2), val(op, c + 3)));
  }
}

__global__ void __launch_bounds__(NT) k_store(float* __restrict__ st, const int* __restrict__ dst, int nops) {
  for (int op = blockIdx.x * NT + threadIdx.x; op < nops; op += gridDim.x * NT) {
    float* d = st + (int64_t)dst[op] * W;
#pragma unroll 4
    for (int c = 0; c < W; c += 4)
      *reinterpret_cast<float4*>(d + c) = make_float4(val(op, c), val(op, c + 1), val(op, c + 2), val(op, c + 3));
  }
}

// two staging slots of CH floats per thread (double buffering over chunks)
template <int CH>
__global__ void __launch_bounds__(NT) k_bulk(float* __restrict__ st, const int* __restrict__ dst, int nops) {
  extern __shared__ __align__(128) float sbuf[];
  float* mine = sbuf + threadIdx.x * 2 * CH;
  int k = 0;
  for (int op = blockIdx.x * NT + threadIdx.x; op < nops; op += gridDim.x * NT) {
    float* d = st + (int64_t)dst[op] * W;
    for (int c0 = 0; c0 < W; c0 += CH, ++k) {
      float* b = mine + (k & 1) * CH;
      // the slot written two chunks ago must have been read by the bulk engine
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
#pragma unroll
      for (int c = 0; c < CH; c += 4)
        *reinterpret_cast<float4*>(b + c) = make_float4(val(op, c0 + c), val(op, c0 + c + 1), val(op, c0 + c + 2), val(op, c0 + c + 3));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;"
                   :: "l"(d + c0), "r"(smem_u32(b)), "r"(CH * 4) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int nops = 4 << 20;   // 4 M ops ≈ 4 GB of payload
  for (int ns : {100000, 1000000}) {   // 96 MB (L2-resident) and 960 MB of states
    std::vector<int> h(nops);
    uint64_t s = 12345;
    for (int i = 0; i < nops; ++i) { s = s * 6364136223846793005ull + 1442695040888963407ull; h[i] = (int)((s >> 33) % ns); }
    int* d_dst; float* d_st;
    CK(cudaMalloc(&d_dst, sizeof(int) * nops));
    CK(cudaMalloc(&d_st, sizeof(float) * (size_t)ns * W));
    CK(cudaMemcpy(d_dst, h.data(), sizeof(int) * nops, cudaMemcpyHostToDevice));
    CK(cudaMemset(d_st, 0, sizeof(float) * (size_t)ns * W));
    CK(cudaFuncSetAttribute(k_bulk<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_bulk<24>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_bulk<48>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_bulk<80>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto timeit = [&](const char* name, int ch, int per_sm, auto launch) {
      const int nop = per_sm == 0 ? nops / 16 : nops;
      launch();
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      ms /= 5;
      printf("{\"form\": \"%s\", \"chunk_B\": %d, \"states\": %d, \"ctas_per_sm\": %d, \"ms\": %.3f, \"payload_GBps\": %.1f}\n",
             name, ch * 4, ns, per_sm, ms, (double)nop * W * 4 / ms * 1e-6);
    };
    // per-SM rates without the L2 saturated: 8 SMs, one CTA each
    {
      const int grid = 8, per_sm = 0;
      timeit("red128_8sm", 16, per_sm, [&]() { k_red<<<grid, NT>>>(d_st, d_dst, nops / 16); });
      timeit("bulk_reduce_8sm", 16, per_sm, [&]() { k_bulk<16><<<grid, NT, NT * 2 * 16 * 4>>>(d_st, d_dst, nops / 16); });
      timeit("bulk_reduce_8sm", 24, per_sm, [&]() { k_bulk<24><<<grid, NT, NT * 2 * 24 * 4>>>(d_st, d_dst, nops / 16); });
      timeit("bulk_reduce_8sm", 48, per_sm, [&]() { k_bulk<48><<<grid, NT, NT * 2 * 48 * 4>>>(d_st, d_dst, nops / 16); });
      timeit("bulk_reduce_8sm", 80, per_sm, [&]() { k_bulk<80><<<grid, NT, NT * 2 * 80 * 4>>>(d_st, d_dst, nops / 16); });
    }
    for (int per_sm : {2, 4}) {
      const int grid = nsm * per_sm;
      timeit("red128", 16, per_sm, [&]() { k_red<<<grid, NT>>>(d_st, d_dst, nops); });
      timeit("store", 16, per_sm, [&]() { k_store<<<grid, NT>>>(d_st, d_dst, nops); });
      timeit("bulk_reduce", 16, per_sm, [&]() { k_bulk<16><<<grid, NT, NT * 2 * 16 * 4>>>(d_st, d_dst, nops); });
      timeit("bulk_reduce", 24, per_sm, [&]() { k_bulk<24><<<grid, NT, NT * 2 * 24 * 4>>>(d_st, d_dst, nops); });
      timeit("bulk_reduce", 48, per_sm, [&]() { k_bulk<48><<<grid, NT, NT * 2 * 48 * 4>>>(d_st, d_dst, nops); });
      if (per_sm == 2) timeit("bulk_reduce", 80, per_sm, [&]() { k_bulk<80><<<grid, NT, NT * 2 * 80 * 4>>>(d_st, d_dst, nops); });
    }
    // correctness of the bulk form: states after one bulk run == after one red run
    std::vector<float> a((size_t)ns * W), b((size_t)ns * W);
    CK(cudaMemset(d_st, 0, sizeof(float) * (size_t)ns * W));
    k_red<<<nsm * 4, NT>>>(d_st, d_dst, nops);
    CK(cudaMemcpy(a.data(), d_st, a.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemset(d_st, 0, sizeof(float) * (size_t)ns * W));
    k_bulk<48><<<nsm * 2, NT, NT * 2 * 48 * 4>>>(d_st, d_dst, nops);
    CK(cudaMemcpy(b.data(), d_st, b.size() * 4, cudaMemcpyDeviceToHost));
    double md = 0, mx = 0;
    for (size_t i = 0; i < a.size(); ++i) { md = std::max(md, (double)fabsf(a[i] - b[i])); mx = std::max(mx, (double)fabsf(a[i])); }
    printf("{\"check\": \"bulk vs red\", \"states\": %d, \"max_abs_diff\": %.3e, \"max_abs\": %.3e}\n", ns, md, mx);
    cudaFree(d_dst); cudaFree(d_st);
  }
  return 0;
}
