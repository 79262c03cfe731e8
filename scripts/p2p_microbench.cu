// Peer-memory copy microbenchmark over NVLink (two GPUs, one process).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_mb scripts/p2p_microbench.cu
//   ./p2p_mb [bytes]
//
// Measures GB/s per direction for: SM pull (ld.global.cg.v4 from the peer),
// SM push (st.global.v4 to the peer), TMA bulk pull (cp.async.bulk peer->smem
// ->local), each with both GPUs moving data at once (the allreduce pattern),
// over a range of CTA counts.  Informs the engine's data-phase design.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1); } } while (0)

template <int U>
__global__ void pull_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, long long nv) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  for (long long base = tid; base < nv; base += nth * U) {
    uint4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long long v = base + u * nth;
      if (v < nv) asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                               : "=r"(x[u].x), "=r"(x[u].y), "=r"(x[u].z), "=r"(x[u].w) : "l"(src + v));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long long v = base + u * nth;
      if (v < nv) dst[v] = x[u];
    }
  }
}

template <int U>
__global__ void push_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, long long nv) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  for (long long base = tid; base < nv; base += nth * U) {
    uint4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long long v = base + u * nth;
      if (v < nv) x[u] = src[v];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long long v = base + u * nth;
      if (v < nv) asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};"
                               :: "l"(dst + v), "r"(x[u].x), "r"(x[u].y), "r"(x[u].z), "r"(x[u].w) : "memory");
    }
  }
}

// TMA 1-D bulk: peer -> shared (mbarrier complete_tx) -> local global (bulk store)
#define CHUNK 16384
#define STAGES 4
__global__ void tma_pull_kernel(const char* __restrict__ src, char* __restrict__ dst, long long nbytes) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) unsigned long long bar[STAGES];
  const long long nchunks = nbytes / CHUNK;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      unsigned a = (unsigned)__cvta_generic_to_shared(&bar[s]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(a));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  unsigned phase[STAGES] = {0};
  long long my = 0;
  // issue the first STAGES loads
  long long c0 = blockIdx.x;
  for (int s = 0; s < STAGES; ++s) {
    long long c = c0 + (long long)s * gridDim.x;
    if (c >= nchunks) break;
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    unsigned d = (unsigned)__cvta_generic_to_shared(smem + s * CHUNK);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(CHUNK) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(d), "l"(src + c * CHUNK), "r"(CHUNK), "r"(b) : "memory");
  }
  for (long long c = c0, k = 0; c < nchunks; c += gridDim.x, ++k) {
    int s = k % STAGES;
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    unsigned d = (unsigned)__cvta_generic_to_shared(smem + s * CHUNK);
    // wait data
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                 " @!p bra W;\n}" :: "r"(b), "r"(phase[s]) : "memory");
    phase[s] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(dst + c * CHUNK), "r"(d), "r"(CHUNK) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    long long cn = c + (long long)STAGES * gridDim.x;
    if (cn < nchunks) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(CHUNK) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(d), "l"(src + cn * CHUNK), "r"(CHUNK), "r"(b) : "memory");
    }
    ++my;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  long long bytes = argc > 1 ? atoll(argv[1]) : (256ll << 20);
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) { printf("need 2 GPUs\n"); return 1; }
  char *buf[2][2];
  cudaStream_t st[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&buf[d][0], bytes));
    CK(cudaMalloc(&buf[d][1], bytes));
    CK(cudaMemset(buf[d][0], d + 1, bytes));
    CK(cudaStreamCreate(&st[d]));
    CK(cudaFuncSetAttribute(tma_pull_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, STAGES * CHUNK));
  }
  const long long nv = bytes / 16;
  const char* names[] = {"pull_ld_cg_U4", "push_st_U4", "tma_bulk_pull"};
  int grids[] = {16, 32, 64, 96, 128, 148, 296};
  for (int m = 0; m < 3; ++m) {
    for (int gi = 0; gi < 7; ++gi) {
      int grid = grids[gi];
      cudaEvent_t e0[2], e1[2];
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        for (int d = 0; d < 2; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaEventCreate(&e0[d]));
          CK(cudaEventCreate(&e1[d]));
        }
        for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
        for (int d = 0; d < 2; ++d) {
          CK(cudaSetDevice(d));
          const char* peer_src = buf[1 - d][0];
          char* local_dst = buf[d][1];
          const char* local_src = buf[d][0];
          char* peer_dst = buf[1 - d][1];
          CK(cudaEventRecord(e0[d], st[d]));
          if (m == 0) pull_kernel<4><<<grid, 256, 0, st[d]>>>((const uint4*)peer_src, (uint4*)local_dst, nv);
          else if (m == 1) push_kernel<4><<<grid, 256, 0, st[d]>>>((const uint4*)local_src, (uint4*)peer_dst, nv);
          else tma_pull_kernel<<<grid, 32, STAGES * CHUNK, st[d]>>>(peer_src, local_dst, bytes);
          CK(cudaEventRecord(e1[d], st[d]));
        }
        float ms = 0;
        for (int d = 0; d < 2; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaEventSynchronize(e1[d]));
          float x;
          CK(cudaEventElapsedTime(&x, e0[d], e1[d]));
          if (x > ms) ms = x;
          CK(cudaGetLastError());
        }
        if (rep > 0 && ms < best) best = ms;
      }
      printf("%-16s grid %4d  %7.1f GB/s per direction (both GPUs at once)\n", names[m], grid,
             bytes / (best * 1e-3) / 1e9);
    }
  }
  return 0;
}
