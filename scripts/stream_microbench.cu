// Streaming-kernel shapes for the direct step (2 reads + 2 writes per element):
// SIMT grid-stride loops at several unroll / occupancy points vs a TMA bulk
// pipeline (cp.async.bulk global->smem, compute, cp.async.bulk smem->global).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/stream_mb scripts/stream_microbench.cu
//   ./scripts/stream_mb [n_floats]
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s -> %s (%d)\n", #x, cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint4 ldv(const void* p) {
  uint4 v;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void stv(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void stv_cs(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
union V4 { uint4 r; float f[4]; };

template <int U, int MINB, bool CS>
__global__ void __launch_bounds__(256, MINB)
simt(const float* __restrict__ g, float* __restrict__ w, float* __restrict__ u, float lr, long long nv) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  for (long long base = tid; base < nv; base += nth * U) {
    V4 x[U], y[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      long long v = base + k * nth;
      if (v < nv) { x[k].r = ldv(g + v * 4); y[k].r = ldv(w + v * 4); }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      long long v = base + k * nth;
      if (v < nv) {
        V4 o;
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          o.f[l] = __fadd_rn(0.0f, x[k].f[l]);
          y[k].f[l] = __fsub_rn(y[k].f[l], __fmul_rn(lr, o.f[l]));
        }
        if (CS) { stv_cs(u + v * 4, o.r); stv_cs(w + v * 4, y[k].r); }
        else { stv(u + v * 4, o.r); stv(w + v * 4, y[k].r); }
      }
    }
  }
}

// ---- TMA bulk pipeline
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* b, unsigned parity) {
  unsigned ok;
  asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
  return ok;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(dst), "r"(smem_u32(src)), "r"(bytes) : "memory");
}

// per stage: g, w in; u, w out (in place over the inputs) -- 2 buffers of CH bytes
template <int CH, int ST>
__global__ void __launch_bounds__(256, 1)
tma_pipe(const float* __restrict__ g, float* __restrict__ w, float* __restrict__ u, float lr, long long n) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) unsigned long long full[ST];
  const long long nch = n * 4 / CH;   // full chunks only (bench sizes are multiples)
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < ST; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  long long first = blockIdx.x, step = gridDim.x;
  // prologue
  int it = 0;
  auto issue = [&](long long c, int s) {
    char* bg = sm + (size_t)s * 2 * CH;
    char* bw = bg + CH;
    mbar_expect_tx(&full[s], 2 * CH);
    bulk_g2s(bg, (const char*)g + c * CH, CH, &full[s]);
    bulk_g2s(bw, (const char*)w + c * CH, CH, &full[s]);
  };
  if (tid == 0) {
    for (int k = 0; k < ST; ++k) {
      long long c = first + (long long)k * step;
      if (c < nch) issue(c, k);
    }
  }
  for (long long c = first; c < nch; c += step, ++it) {
    const int s = it % ST;
    const unsigned parity = (it / ST) & 1;
    while (!mbar_try_wait(&full[s], parity)) {}
    float* bg = (float*)(sm + (size_t)s * 2 * CH);
    float* bw = bg + CH / 4;
    for (int i = tid * 4; i < CH / 4; i += 256 * 4) {
      float4 x = *(float4*)(bg + i), y = *(float4*)(bw + i);
      float4 o;
      o.x = __fadd_rn(0.f, x.x); o.y = __fadd_rn(0.f, x.y); o.z = __fadd_rn(0.f, x.z); o.w = __fadd_rn(0.f, x.w);
      y.x = __fsub_rn(y.x, __fmul_rn(lr, o.x)); y.y = __fsub_rn(y.y, __fmul_rn(lr, o.y));
      y.z = __fsub_rn(y.z, __fmul_rn(lr, o.z)); y.w = __fsub_rn(y.w, __fmul_rn(lr, o.w));
      *(float4*)(bg + i) = o;
      *(float4*)(bw + i) = y;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      bulk_s2g((char*)u + c * CH, bg, CH);
      bulk_s2g((char*)w + c * CH, bw, CH);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      // refill this stage once its stores have read the smem
      long long cn = c + (long long)ST * step;
      if (cn < nch) {
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        issue(cn, s);
      }
    }
    __syncthreads();
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  long long n = argc > 1 ? atoll(argv[1]) : 25559040;  // multiple of 16 KiB / 4
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float *g, *w, *u, *flush;
  CK(cudaMalloc(&g, n * 4));
  CK(cudaMalloc(&w, n * 4));
  CK(cudaMalloc(&u, n * 4));
  CK(cudaMalloc(&flush, 256 << 20));
  CK(cudaMemset(g, 0, n * 4));
  CK(cudaMemset(w, 0, n * 4));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const double bytes = 16.0 * n;
  auto run = [&](const char* name, auto launch) {
    float best = 1e30f, sum = 0;
    for (int rep = 0; rep < 12; ++rep) {
      CK(cudaMemsetAsync(flush, rep, 256 << 20));
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (rep >= 2) { sum += ms; if (ms < best) best = ms; }
    }
    CK(cudaGetLastError());
    printf("%-34s best %7.1f us (%6.0f GB/s)  mean %7.1f us (%6.0f GB/s)\n", name, best * 1e3,
           bytes / (best * 1e-3) / 1e9, sum / 10 * 1e3, bytes / (sum / 10 * 1e-3) / 1e9);
  };
  const long long nv = n / 4;
  run("simt U4 minB3 (current)", [&] { simt<4, 3, false><<<sms * 3, 256>>>(g, w, u, 0.1f, nv); });
  run("simt U4 minB3 st.cs", [&] { simt<4, 3, true><<<sms * 3, 256>>>(g, w, u, 0.1f, nv); });
  run("simt U2 minB4", [&] { simt<2, 4, false><<<sms * 4, 256>>>(g, w, u, 0.1f, nv); });
  run("simt U2 minB6", [&] { simt<2, 6, false><<<sms * 6, 256>>>(g, w, u, 0.1f, nv); });
  run("simt U2 minB8", [&] { simt<2, 8, false><<<sms * 8, 256>>>(g, w, u, 0.1f, nv); });
  run("simt U1 minB8", [&] { simt<1, 8, false><<<sms * 8, 256>>>(g, w, u, 0.1f, nv); });
  run("simt U4 minB4", [&] { simt<4, 4, false><<<sms * 4, 256>>>(g, w, u, 0.1f, nv); });
  run("simt U1 minB8 many blocks", [&] { simt<1, 8, false><<<(int)((nv + 255) / 256), 256>>>(g, w, u, 0.1f, nv); });
  run("simt U2 minB8 st.cs", [&] { simt<2, 8, true><<<sms * 8, 256>>>(g, w, u, 0.1f, nv); });
  {
    constexpr int CH = 8192, ST = 6;
    size_t sm = (size_t)ST * 2 * CH;
    CK(cudaFuncSetAttribute(tma_pipe<CH, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    run("tma 8K x6 stages, 1 CTA/SM", [&] { tma_pipe<CH, ST><<<sms, 256, sm>>>(g, w, u, 0.1f, n); });
    run("tma 8K x6 stages, 2 CTA/SM", [&] { tma_pipe<CH, ST><<<sms * 2, 256, sm>>>(g, w, u, 0.1f, n); });
  }
  {
    constexpr int CH = 16384, ST = 4;
    size_t sm = (size_t)ST * 2 * CH;
    CK(cudaFuncSetAttribute(tma_pipe<CH, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    run("tma 16K x4 stages, 1 CTA/SM", [&] { tma_pipe<CH, ST><<<sms, 256, sm>>>(g, w, u, 0.1f, n); });
  }
  {
    constexpr int CH = 4096, ST = 8;
    size_t sm = (size_t)ST * 2 * CH;
    CK(cudaFuncSetAttribute(tma_pipe<CH, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    run("tma 4K x8 stages, 2 CTA/SM", [&] { tma_pipe<CH, ST><<<sms * 2, 256, sm>>>(g, w, u, 0.1f, n); });
    run("tma 4K x8 stages, 3 CTA/SM", [&] { tma_pipe<CH, ST><<<sms * 3, 256, sm>>>(g, w, u, 0.1f, n); });
  }
  return 0;
}
