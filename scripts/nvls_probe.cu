// NVLS (NVSwitch multicast + in-switch reduction) probe, one process, all GPUs.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/nvls_probe scripts/nvls_probe.cu -lcuda
//   ./scripts/nvls_probe [bytes]
//
// 1. checks CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, creates a multicast object
//    over every GPU, binds one physical allocation per GPU, maps the multicast
//    and unicast views;
// 2. correctness: multimem.ld_reduce of (dev+1) patterns, multimem.st broadcast;
// 3. bandwidth of an NVLS allreduce (each GPU ld_reduces its 1/P shard and
//    multimem.st-s it back to everyone) vs the bus-bytes formula 2(P-1)/P * S.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

#define CU(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); \
  printf("CU %s -> %s (%s:%d)\n", #x, s, __FILE__, __LINE__); exit(1); } } while (0)
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s -> %s (%d)\n", #x, cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__global__ void fill(float* p, long long n, float v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) p[i] = v;
}

// owner of [v0, v1) (16-byte vectors): reduce through the switch, broadcast the result
__global__ void nvls_allreduce(float* mc_in, float* mc_out, long long v0, long long v1, float inv) {
  for (long long v = v0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; v < v1;
       v += (long long)gridDim.x * blockDim.x) {
    float a, b, c, d;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(mc_in + 4 * v) : "memory");
    a *= inv; b *= inv; c *= inv; d *= inv;
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(mc_out + 4 * v), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
  }
}

int main(int argc, char** argv) {
  long long bytes = argc > 1 ? atoll(argv[1]) : (100ll << 20);
  CU(cuInit(0));
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  printf("devices: %d\n", ndev);
  for (int d = 0; d < ndev; ++d) {
    CUdevice dev;
    CU(cuDeviceGet(&dev, d));
    int mc = 0, fab = 0;
    CU(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
    printf("dev %d multicast_supported=%d fabric_handles=%d\n", d, mc, fab);
  }
  CUmulticastObjectProp prop = {};
  prop.numDevices = ndev;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  prop.size = 2 * bytes;
  CU(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  size_t size = ((2 * bytes + gran - 1) / gran) * gran;
  prop.size = size;
  printf("granularity %zu size %zu\n", gran, size);
  CUmemGenericAllocationHandle mch;
  CU(cuMulticastCreate(&mch, &prop));
  for (int d = 0; d < ndev; ++d) {
    CUdevice dev;
    CU(cuDeviceGet(&dev, d));
    CU(cuMulticastAddDevice(mch, dev));
  }
  std::vector<float*> uc(ndev), mcp(ndev);
  std::vector<CUcontext> ctx(ndev);
  for (int d = 0; d < ndev; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaFree(0));
    CU(cuCtxGetCurrent(&ctx[d]));
    CUmemAllocationProp p = {};
    p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    p.location.id = d;
    p.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t g2 = 0;
    CU(cuMemGetAllocationGranularity(&g2, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    CUmemGenericAllocationHandle ph;
    CU(cuMemCreate(&ph, size, &p, 0));
    CU(cuMulticastBindMem(mch, 0, ph, 0, size, 0));
    CUdeviceptr a;
    CU(cuMemAddressReserve(&a, size, gran, 0, 0));
    CU(cuMemMap(a, size, 0, ph, 0));
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = d;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CU(cuMemSetAccess(a, size, &acc, 1));
    uc[d] = (float*)a;
    CUdeviceptr m;
    CU(cuMemAddressReserve(&m, size, gran, 0, 0));
    CU(cuMemMap(m, size, 0, mch, 0));
    CU(cuMemSetAccess(m, size, &acc, 1));
    mcp[d] = (float*)m;
  }
  const long long n = bytes / 4, nv = n / 4;
  for (int d = 0; d < ndev; ++d) {
    CK(cudaSetDevice(d));
    fill<<<296, 256>>>(uc[d], n, (float)(d + 1));
    CK(cudaDeviceSynchronize());
  }
  // correctness: everyone reduces its shard and broadcasts
  float inv = 1.0f / ndev;
  for (int d = 0; d < ndev; ++d) {
    CK(cudaSetDevice(d));
    nvls_allreduce<<<148, 512>>>(mcp[d], mcp[d] + n, nv * d / ndev, nv * (d + 1) / ndev, inv);
  }
  for (int d = 0; d < ndev; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
  float want = 0;
  for (int d = 0; d < ndev; ++d) want += d + 1;
  want *= inv;
  for (int d = 0; d < ndev; ++d) {
    std::vector<float> h(4);
    CK(cudaSetDevice(d));
    CK(cudaMemcpy(h.data(), uc[d] + n, 16, cudaMemcpyDeviceToHost));
    float last[4];
    CK(cudaMemcpy(last, uc[d] + n + (nv - 1) * 4, 16, cudaMemcpyDeviceToHost));
    printf("dev %d result[0]=%f last=%f want %f\n", d, h[0], last[3], want);
  }
  // bandwidth
  for (int grid : {32, 64, 148, 296}) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      std::vector<cudaEvent_t> e0(ndev), e1(ndev);
      for (int d = 0; d < ndev; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceSynchronize());
        CK(cudaEventCreate(&e0[d]));
        CK(cudaEventCreate(&e1[d]));
      }
      for (int d = 0; d < ndev; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventRecord(e0[d]));
        nvls_allreduce<<<grid, 512>>>(mcp[d], mcp[d] + n, nv * d / ndev, nv * (d + 1) / ndev, inv);
        CK(cudaEventRecord(e1[d]));
      }
      float ms = 0;
      for (int d = 0; d < ndev; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventSynchronize(e1[d]));
        float x;
        CK(cudaEventElapsedTime(&x, e0[d], e1[d]));
        if (x > ms) ms = x;
      }
      if (rep && ms < best) best = ms;
    }
    double bus = 2.0 * (ndev - 1) / ndev * bytes;
    printf("NVLS allreduce %lld B grid %d: %.1f us  busbw %.1f GB/s\n", bytes, grid, best * 1e3,
           bus / (best * 1e-3) / 1e9);
  }
  return 0;
}
