// Host side of the eagercoll_b200 C ABI: communicator, IPC peer mapping,
// request ring, waits and launches.  See include/eagercoll_b200.h.
#include <cuda.h>
#include <cuda_runtime.h>
#include <errno.h>
#include <immintrin.h>
#include <sched.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include <atomic>
#include <chrono>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/eagercoll_b200.h"
#include "ec_common.cuh"

// launchers (ec_kernels.cu)
cudaError_t launch_engine(int dtype, const EcDesc* d_descs, int n_local, int blocks_per_rank,
                          unsigned long long epoch, int smem_bytes, cudaStream_t s);
cudaError_t launch_fold(int dtype, void* stash, const void* grad, long long n, int mode,
                        unsigned int* nonfinite, cudaStream_t s, int gated);
cudaError_t launch_update(int dtype, void* w, const void* u, double lr, long long n, cudaStream_t s);
cudaError_t launch_momentum(int dtype, void* w, void* buf, const void* u, double lr, double mu,
                            long long n, cudaStream_t s);
cudaError_t launch_reduce(int dtype, const void* const* srcs, int p, unsigned long long has,
                          void* dst, long long n, int div, cudaStream_t s);
cudaError_t launch_post(EcLocal* L, unsigned long long seq1, unsigned int type, unsigned int flags,
                        long long t, long long arg, cudaStream_t s);
int engine_blocks_per_sm(int dtype, int smem_bytes);
cudaError_t launch_set_generation(EcLocal* L, EcHostCtl* H, long long gen, int stash_pending,
                                  long long contributed_round, cudaStream_t s);
cudaError_t launch_stream_barrier(unsigned long long* count, unsigned long long target,
                                  EcHostCtl* H, unsigned long long timeout_ns, cudaStream_t s);
cudaError_t launch_fold_auto(int dtype, void* stash, const void* grad, long long n, EcLocal* L,
                             unsigned long long seq1, unsigned flags, long long t, int zero_copy,
                             cudaStream_t s);
cudaError_t launch_wait_gen(EcLocal* L, EcHostCtl* H, long long t, int R, int lead,
                            unsigned long long timeout_ns, cudaStream_t s);
cudaError_t launch_wait_done(EcLocal* L, EcHostCtl* H, long long t, unsigned long long timeout_ns,
                             cudaStream_t s);
cudaError_t launch_update_gen(int dtype, void* w, void* mom, const char* ring, long long slot_bytes,
                              int R, EcLocal* L, double lr, double mu, long long n, EcHostCtl* H,
                              long long t, unsigned long long timeout_ns, unsigned long long seq1,
                              void* stash, const void* gbuf, const EcDesc* dp, int progressive,
                              int share, cudaStream_t s);
cudaError_t launch_write_u64(unsigned long long* p, unsigned long long v, cudaStream_t s);
cudaError_t launch_direct_step(int dtype, const EcDesc* d_desc, unsigned long long seq,
                               unsigned int flags, void* w, void* mom, const void* ring,
                               long long slot_bytes, const void* src0, const void* src1,
                               double lr, double mu, long long n, long long t,
                               unsigned long long timeout_ns, cudaStream_t s,
                               cudaStream_t ps, cudaEvent_t pev);
cudaError_t launch_direct(int dtype, const EcDesc* d_desc, long long nvec, unsigned long long seq,
                          unsigned int type, unsigned int flags, long long t, long long arg,
                          cudaStream_t s);
cudaError_t launch_spin(unsigned long long ns, cudaStream_t s);
cudaError_t preload_kernels();
extern unsigned long long g_ec_launches;

#define EC_VERSION 10000
#define BLOB_MAGIC 0x45434231u  // "ECB1"

static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(EC_E_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                            \
  } while (0)

static inline unsigned long long now_ns() {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (unsigned long long)ts.tv_sec * 1000000000ull + ts.tv_nsec;
}

template <typename T>
static inline T aload(const T* p) { return __atomic_load_n(p, __ATOMIC_ACQUIRE); }
template <typename T>
static inline void astore(T* p, T v) { __atomic_store_n(p, v, __ATOMIC_RELEASE); }

// Spin, then back off: tight for the first ~50 us (latency of a round), then yield.
struct Backoff {
  unsigned long long t0 = now_ns();
  unsigned it = 0;
  void pause() {
    ++it;
    if (it < 2000) {
      _mm_pause();
    } else if (it < 20000) {
      sched_yield();
    } else {
      struct timespec ts = {0, 20000};
      nanosleep(&ts, nullptr);
    }
  }
  bool expired(int timeout_ms) const {
    return timeout_ms >= 0 && now_ns() - t0 > (unsigned long long)timeout_ms * 1000000ull;
  }
};

struct EcRankHost {
  int rank = -1;
  EcCtrl* ctrl = nullptr;
  char* send = nullptr;
  char* ring = nullptr;
  char* gbuf = nullptr;        // registered gradient buffer (zero-copy offers)
  EcHostCtl* h = nullptr;      // host view
  EcHostCtl* hd = nullptr;     // device view of the same pinned page
  EcLocal* local = nullptr;
  unsigned long long* forced = nullptr;
  long long n_forced = 0;
  unsigned long long next_seq = 0;
  unsigned long long last_update_ns = 0;  // device-timed update of the last reconciled async step
  unsigned long long bar_epoch = 0;       // ec_stream_barrier calls so far
  // the last stream-ordered pin release (ec_set_pin ordered): a new host pin
  // waits for it, so an older queued unpin can never clear a newer pin
  cudaEvent_t unpin_ev = nullptr;
  bool unpin_pending = false;
  std::mutex mu;
  std::mutex pin_mu;
};

struct BlobV1 {
  unsigned magic;
  int rank;
  long long n;
  int dtype, R;
  cudaIpcMemHandle_t ctrl, send, ring, gbuf;
};

struct ec_comm {
  int P = 0, rank_lo = 0, n_local = 0, device = 0, dtype = 0, flavor = 0, R = 2, W = 0;
  int w_step = 0;   // workers of rounds with progressive step updates (EcDesc::w_step)
  bool W_default = true;
  long long n = 0, slot_bytes = 0;
  int elem = 4;
  unsigned long long timeout_ns = 60ull * 1000000000ull;
  std::vector<EcRankHost*> L;
  std::vector<EcCtrl*> ctrl;
  std::vector<char*> send, ring, gbuf;
  std::vector<int> opened;  // 1 = IPC-opened peer
  EcDesc* d_descs = nullptr;
  cudaStream_t es = nullptr;
  bool running = false;
  bool direct = false;          // world of one rank: no persistent kernel (see ec_kernels.cu)
  void* last_stream = nullptr;  // direct mode orders host-posted requests on it
  cudaStream_t pub_s = nullptr;  // direct mode: the steps' publication stream
  cudaEvent_t pub_ev = nullptr;
  cudaEvent_t pub_join_ev = nullptr;
  bool pub_used = false;         // a step published on pub_s
  // the last host-posted request's kernels (direct mode): a step issued on
  // another stream is ordered behind them, so its publication never waits
  cudaEvent_t req_ev = nullptr;
  cudaStream_t req_stream = nullptr;
  bool req_pending = false;
  unsigned long long epoch = 0;
  int mode = 0, chv = 256, stages = 4, smem_bytes = 0;  // data phase (see EcDesc)
  int lead = 1;                                        // rounds in flight (EcDesc::lead)
  int quorum = 0;                                      // majority quorum (EcDesc::quorum)
  double budget = 0.0;                                 // SMs' worth of engine CTAs held
  // NVLS (reduction_mode "fast"): multicast object over every rank's GPU
  CUmemGenericAllocationHandle mc_handle = 0, mc_phys = 0;
  bool mc_created = false, mc_attached = false, mc_phys_made = false;
  CUdeviceptr mc_va = 0, uc_va = 0;
  size_t mc_size = 0;
  char* ring_cuda = nullptr;  // the cudaMalloc'd ring, restored when NVLS is torn down
  // idle park (see watcher_main): the engine exits on its own after
  // EC_IDLE_PARK_MS without work, so device-wide syncs in user code return;
  // any post relaunches it, and a watcher relaunches it for remote peers
  std::recursive_mutex live_mu;        // posts, starts, pauses, the watcher's park/relaunch
  std::thread watcher;
  std::atomic<bool> quit{false};
  std::atomic<bool> parked_auto{false};
  std::atomic<unsigned long long> last_api_ns{0};
  unsigned long long idle_ns = 0;      // 0: never park on idleness
  unsigned long long* poll_buf = nullptr;   // pinned: peers' words, read while parked
  cudaStream_t ws = nullptr;           // watcher's copy stream
  unsigned long long idle_parks = 0, idle_wakes = 0;
};

static int check_li(ec_comm_t* c, int li) {
  if (!c) return fail(EC_E_ARG, "null communicator");
  if (li < 0 || li >= c->n_local) return fail(EC_E_ARG, "local index %d out of range", li);
  return EC_OK;
}

// a stream for host-visible publications, highest priority: its one-warp
// kernels are scheduled ahead of the next step's queued CTAs
static int make_pub_stream(ec_comm_t* c, cudaStream_t* s, cudaEvent_t* ev) {
  int lo_pri = 0, hi_pri = 0;
  CK(cudaSetDevice(c->device));
  CK(cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri));
  CK(cudaStreamCreateWithPriority(s, cudaStreamNonBlocking, hi_pri));
  CK(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
  return EC_OK;
}



static int device_error(EcRankHost* r) {
  unsigned long long e = aload(&r->h->error);
  if (e) {
    return fail(EC_E_DEVICE, "engine error %llu (info 0x%llx) at rank %d", e,
                aload(&r->h->error_info), r->rank);
  }
  return EC_OK;
}


// ---- NVLS: NVSwitch multicast objects through the driver API ----------------
// (entry points fetched at run time: the library must load where no driver is
// installed, e.g. the build container)
typedef CUresult (*PFN_mcCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*);
typedef CUresult (*PFN_mcAddDevice)(CUmemGenericAllocationHandle, CUdevice);
typedef CUresult (*PFN_mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t, unsigned long long);
typedef CUresult (*PFN_mcGran)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags);
typedef CUresult (*PFN_memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
typedef CUresult (*PFN_memRelease)(CUmemGenericAllocationHandle);
typedef CUresult (*PFN_addrReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
typedef CUresult (*PFN_addrFree)(CUdeviceptr, size_t);
typedef CUresult (*PFN_memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
typedef CUresult (*PFN_memUnmap)(CUdeviceptr, size_t);
typedef CUresult (*PFN_setAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
typedef CUresult (*PFN_export)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long);
typedef CUresult (*PFN_import)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType);
typedef CUresult (*PFN_devGet)(CUdevice*, int);
typedef CUresult (*PFN_devAttr)(int*, CUdevice_attribute, CUdevice);
typedef CUresult (*PFN_mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);

struct DrvApi {
  PFN_mcCreate mcCreate = nullptr;
  PFN_mcAddDevice mcAddDevice = nullptr;
  PFN_mcBindMem mcBindMem = nullptr;
  PFN_mcGran mcGran = nullptr;
  PFN_memCreate memCreate = nullptr;
  PFN_memRelease memRelease = nullptr;
  PFN_addrReserve addrReserve = nullptr;
  PFN_addrFree addrFree = nullptr;
  PFN_memMap memMap = nullptr;
  PFN_memUnmap memUnmap = nullptr;
  PFN_setAccess setAccess = nullptr;
  PFN_export exportH = nullptr;
  PFN_import importH = nullptr;
  PFN_devGet devGet = nullptr;
  PFN_devAttr devAttr = nullptr;
  PFN_mcUnbind mcUnbind = nullptr;
  bool ok = false;
};

static DrvApi& drv() {
  static DrvApi d;
  static bool tried = false;
  if (tried) return d;
  tried = true;
  auto get = [](const char* name, void** fn) -> bool {
    cudaDriverEntryPointQueryResult q;
    return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
           q == cudaDriverEntryPointSuccess && *fn;
  };
  d.ok = get("cuMulticastCreate", (void**)&d.mcCreate) && get("cuMulticastAddDevice", (void**)&d.mcAddDevice) &&
         get("cuMulticastBindMem", (void**)&d.mcBindMem) && get("cuMulticastGetGranularity", (void**)&d.mcGran) &&
         get("cuMemCreate", (void**)&d.memCreate) && get("cuMemRelease", (void**)&d.memRelease) &&
         get("cuMemAddressReserve", (void**)&d.addrReserve) && get("cuMemAddressFree", (void**)&d.addrFree) &&
         get("cuMemMap", (void**)&d.memMap) && get("cuMemUnmap", (void**)&d.memUnmap) &&
         get("cuMemSetAccess", (void**)&d.setAccess) &&
         get("cuMemExportToShareableHandle", (void**)&d.exportH) &&
         get("cuMemImportFromShareableHandle", (void**)&d.importH) && get("cuDeviceGet", (void**)&d.devGet) &&
         get("cuDeviceGetAttribute", (void**)&d.devAttr) && get("cuMulticastUnbind", (void**)&d.mcUnbind);
  return d;
}

#define DRV(call)                                                                 \
  do {                                                                            \
    CUresult r_ = (call);                                                         \
    if (r_ != CUDA_SUCCESS) return fail(EC_E_CUDA, "%s failed (%d)", #call, (int)r_); \
  } while (0)

static size_t nvls_size(ec_comm_t* c, size_t gran) {
  const size_t want = (size_t)c->slot_bytes * (1 + c->R);  // staging + result ring
  return ((want + gran - 1) / gran) * gran;
}

// POSIX file descriptors (passed between the ranks' processes over a Unix
// socket) work without IMEX channels; fabric handles are plain bytes but need them
static CUmemAllocationHandleType nvls_handle_type() {
  const char* e = getenv("EC_NVLS_HANDLE");
  return (e && strcmp(e, "fabric") == 0) ? CU_MEM_HANDLE_TYPE_FABRIC
                                         : CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
}

static int nvls_prop(ec_comm_t* c, CUmulticastObjectProp* prop, size_t* gran) {
  DrvApi& D = drv();
  memset(prop, 0, sizeof(*prop));
  prop->numDevices = c->P;
  prop->handleTypes = nvls_handle_type();
  prop->size = (size_t)c->slot_bytes * (1 + c->R);
  DRV(D.mcGran(gran, prop, CU_MULTICAST_GRANULARITY_MINIMUM));
  prop->size = nvls_size(c, *gran);
  return EC_OK;
}

static void nvls_teardown(ec_comm_t* c) {
  DrvApi& D = drv();
  if (!D.ok) return;
  if (c->mode == 2 && c->ring_cuda) {
    c->L[0]->ring = c->ring_cuda;
    c->ring[c->rank_lo] = c->ring_cuda;
    c->mode = 0;
  }
  if (c->mc_va) {
    D.memUnmap(c->mc_va, c->mc_size);
    D.addrFree(c->mc_va, c->mc_size);
    c->mc_va = 0;
  }
  if (c->uc_va) {
    D.memUnmap(c->uc_va, c->mc_size);
    D.addrFree(c->uc_va, c->mc_size);
    c->uc_va = 0;
  }
  if (c->mc_phys_made) {
    CUdevice dev;
    if (D.devGet(&dev, c->device) == CUDA_SUCCESS) D.mcUnbind(c->mc_handle, dev, 0, c->mc_size);
    D.memRelease(c->mc_phys);
    c->mc_phys_made = false;
  }
  if (c->mc_created || c->mc_attached) {
    D.memRelease(c->mc_handle);
    c->mc_created = c->mc_attached = false;
  }
}

// Every engine is a cooperative grid that must be co-resident with every other
// running engine on the device (a CTA that never gets an SM would stall its
// rank forever).  Each communicator reserves its CTAs' share of the SMs at
// creation; a communicator created when others hold most of the device gets
// fewer worker CTAs or fails loudly.
static std::mutex g_budget_mu;
static std::map<int, double> g_budget_used;

static int budget_engine(ec_comm_t* c, bool w_default) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  const int k = engine_blocks_per_sm(c->dtype, c->smem_bytes);
  if (sms <= 0 || k <= 0) return fail(EC_E_CUDA, "engine occupancy query failed");
  std::lock_guard<std::mutex> g(g_budget_mu);
  const double left = sms - 1 - g_budget_used[c->device];   // one SM of slack
  auto need = [&](int W) { return (double)c->n_local * (1 + W) / k; };
  if (need(c->W) > left) {
    if (!w_default && !getenv("EC_WORKERS_SHRINK"))
      return fail(EC_E_STATE, "no room for another engine on device %d (%.0f of %d SMs held by "
                  "other collectives): close or release them", c->device,
                  g_budget_used[c->device], sms);
    const int W = (int)(left * k / c->n_local) - 1;
    if (W < 4)
      return fail(EC_E_STATE, "no room for another engine on device %d (%.0f of %d SMs held by "
                  "other collectives): close or release them", c->device,
                  g_budget_used[c->device], sms);
    c->W = W;
  }
  c->budget = need(c->W);
  g_budget_used[c->device] += c->budget;
  return EC_OK;
}

static void budget_release(ec_comm_t* c) {
  std::lock_guard<std::mutex> g(g_budget_mu);
  g_budget_used[c->device] -= c->budget;
  c->budget = 0.0;
}

extern "C" int ec_nvls_supported(int device) {
  DrvApi& D = drv();
  if (!D.ok) return 0;
  CUdevice dev;
  if (D.devGet(&dev, device) != CUDA_SUCCESS) return 0;
  int mc = 0, fab = 0;
  D.devAttr(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  D.devAttr(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
  return mc && fab;
}

extern "C" int ec_nvls_create(ec_comm_t* c, void* blob, size_t cap, size_t* len) {
  if (!c) return fail(EC_E_ARG, "null communicator");
  if (c->n_local != 1 || c->dtype != EC_F32 || c->P < 2)
    return fail(EC_E_ARG, "NVLS needs one fp32 rank per GPU and P >= 2");
  if (cap < sizeof(CUmemFabricHandle)) return fail(EC_E_ARG, "blob too small");
  DrvApi& D = drv();
  if (!D.ok) return fail(EC_E_STATE, "driver multicast API unavailable");
  CK(cudaSetDevice(c->device));
  CUmulticastObjectProp prop;
  size_t gran = 0;
  int rc = nvls_prop(c, &prop, &gran);
  if (rc) return rc;
  DRV(D.mcCreate(&c->mc_handle, &prop));
  c->mc_created = true;
  c->mc_size = prop.size;
  if (nvls_handle_type() == CU_MEM_HANDLE_TYPE_FABRIC) {
    CUmemFabricHandle fh;
    DRV(D.exportH(&fh, c->mc_handle, CU_MEM_HANDLE_TYPE_FABRIC, 0));
    memcpy(blob, &fh, sizeof(fh));
    if (len) *len = sizeof(fh);
  } else {
    int fd = -1;  // the caller passes this descriptor to the other ranks (SCM_RIGHTS)
    DRV(D.exportH(&fd, c->mc_handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
    memcpy(blob, &fd, sizeof(fd));
    if (len) *len = sizeof(fd);
  }
  return EC_OK;
}

extern "C" int ec_nvls_attach(ec_comm_t* c, const void* blob, size_t len) {
  if (!c) return fail(EC_E_ARG, "null communicator");
  DrvApi& D = drv();
  if (!D.ok) return fail(EC_E_STATE, "driver multicast API unavailable");
  CK(cudaSetDevice(c->device));
  if (!c->mc_created) {
    if (nvls_handle_type() == CU_MEM_HANDLE_TYPE_FABRIC) {
      if (len < sizeof(CUmemFabricHandle)) return fail(EC_E_ARG, "blob too short");
      CUmemFabricHandle fh;
      memcpy(&fh, blob, sizeof(fh));
      DRV(D.importH(&c->mc_handle, &fh, CU_MEM_HANDLE_TYPE_FABRIC));
    } else {
      if (len < sizeof(int)) return fail(EC_E_ARG, "blob too short");
      int fd;
      memcpy(&fd, blob, sizeof(fd));  // a descriptor valid in THIS process
      DRV(D.importH(&c->mc_handle, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
    }
    c->mc_attached = true;
    CUmulticastObjectProp prop;
    size_t gran = 0;
    int rc = nvls_prop(c, &prop, &gran);
    if (rc) return rc;
    c->mc_size = prop.size;
  }
  CUdevice dev;
  DRV(D.devGet(&dev, c->device));
  DRV(D.mcAddDevice(c->mc_handle, dev));
  return EC_OK;
}

extern "C" int ec_nvls_bind(ec_comm_t* c) {
  if (!c) return fail(EC_E_ARG, "null communicator");
  if (c->running) return fail(EC_E_STATE, "bind NVLS before the engine starts");
  DrvApi& D = drv();
  if (!D.ok || !(c->mc_created || c->mc_attached)) return fail(EC_E_STATE, "attach first");
  CK(cudaSetDevice(c->device));
  CUmemAllocationProp p;
  memset(&p, 0, sizeof(p));
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = c->device;
  p.requestedHandleTypes = nvls_handle_type();
  DRV(D.memCreate(&c->mc_phys, c->mc_size, &p, 0));
  c->mc_phys_made = true;
  DRV(D.mcBindMem(c->mc_handle, 0, c->mc_phys, 0, c->mc_size, 0));
  CUmemAccessDesc acc;
  memset(&acc, 0, sizeof(acc));
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = c->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  const size_t align = 2ull << 20;
  DRV(D.addrReserve(&c->uc_va, c->mc_size, align, 0, 0));
  DRV(D.memMap(c->uc_va, c->mc_size, 0, c->mc_phys, 0));
  DRV(D.setAccess(c->uc_va, c->mc_size, &acc, 1));
  DRV(D.addrReserve(&c->mc_va, c->mc_size, align, 0, 0));
  DRV(D.memMap(c->mc_va, c->mc_size, 0, c->mc_handle, 0));
  DRV(D.setAccess(c->mc_va, c->mc_size, &acc, 1));
  CK(cudaMemset((void*)c->uc_va, 0, c->mc_size));
  CK(cudaDeviceSynchronize());
  // the result ring now lives in the multicast-bound region (after the staging slot)
  EcRankHost* r = c->L[0];
  c->ring_cuda = r->ring;
  r->ring = (char*)c->uc_va + c->slot_bytes;
  c->ring[c->rank_lo] = r->ring;
  c->mode = 2;
  // the switch round trip is long: the NVLS data phase wants more CTAs
  // (measured P=4, 1 GiB: W=64 363 GB/s, W=128 558, W=144 561 busbw)
  if (c->W_default && c->n_local == 1) {
    budget_release(c);
    c->W = 128;
    int rc = budget_engine(c, true);
    if (rc) return rc;
  }
  return EC_OK;
}

extern "C" {

int ec_version(void) { return EC_VERSION; }
uint64_t ec_launch_count(void) { return __atomic_load_n(&g_ec_launches, __ATOMIC_RELAXED); }
const char* ec_last_error(void) { return g_err.c_str(); }

int ec_comm_create(int world_size, int rank_lo, int n_local, int device, int64_t n_elems,
                   int dtype, int flavor, int ring_slots, int workers_per_rank, ec_comm_t** out) {
  if (!out) return fail(EC_E_ARG, "out is null");
  *out = nullptr;
  if (world_size < 1 || world_size > EC_MAX_P)
    return fail(EC_E_ARG, "world_size must be in [1, %d]", EC_MAX_P);
  if (n_local < 1 || rank_lo < 0 || rank_lo + n_local > world_size)
    return fail(EC_E_ARG, "bad local rank range [%d, %d)", rank_lo, rank_lo + n_local);
  if (n_elems < 1) return fail(EC_E_ARG, "n_elems must be >= 1");
  if (dtype < EC_F32 || dtype > EC_I64) return fail(EC_E_ARG, "bad dtype %d", dtype);
  if (flavor < EC_SYNC || flavor > EC_MAJORITY) return fail(EC_E_ARG, "bad flavor %d", flavor);
  if (ring_slots < 2) return fail(EC_E_ARG, "ring_slots must be >= 2");
  CK(cudaSetDevice(device));
  CK(preload_kernels());
  ec_comm* c = new ec_comm();
  c->P = world_size;
  c->rank_lo = rank_lo;
  c->n_local = n_local;
  c->device = device;
  c->dtype = dtype;
  c->flavor = flavor;
  c->R = ring_slots;
  c->n = n_elems;
  c->elem = dtype == EC_F32 ? 4 : 8;
  c->slot_bytes = ((n_elems * c->elem + 255) / 256) * 256;
  if (workers_per_rank <= 0) {
    const char* env = getenv("EC_WORKERS");
    workers_per_rank = env ? atoi(env) : 0;
  }
  const bool w_default = workers_per_rank <= 0;
  if (workers_per_rank <= 0) {
    if (n_local == 1) {
      // 128 worker CTAs: with two rounds in flight plain 100 MB rounds run at
      // 665-677 GB/s vs 616-636 with 80-96 (profiles/r2_geom4.json,
      // r2_geom2.json); at P >= 3 a round carrying progressive step updates
      // uses EcDesc::w_step = 80 of them (the step beside its update kernel:
      // 14,146 vs 13,583 steps/s), at P = 2 all 128 (9,747 vs 9,586 with 96)
      workers_per_rank = 128;
    } else {  // emulated world: all ranks' CTA groups share one GPU
      workers_per_rank = (144 / n_local) - 1;
      if (workers_per_rank > 16) workers_per_rank = 16;
      if (workers_per_rank < 1) workers_per_rank = 1;
    }
  }
  c->W_default = w_default;
  c->W = workers_per_rank;
  {
    const char* e = getenv("EC_WORKERS_STEP");
    const int ws = e ? atoi(e) : (world_size >= 3 && n_local == 1 ? 80 : workers_per_rank);
    c->w_step = ws > 0 && ws < workers_per_rank ? ws : workers_per_rank;
  }
  c->direct = world_size == 1 && !getenv("EC_FORCE_ENGINE");
  // Data phase: fused TMA (default) or two-phase ld.cg pull (EC_DATA=ldg).
  // TMA geometry: P source slices + 1 output slice per stage, `stages` deep,
  // within ~150 KB of shared memory.
  c->mode = (getenv("EC_DATA") && strcmp(getenv("EC_DATA"), "ldg") == 0) ? 1 : 0;
  {
    int chb = world_size <= 12 ? 16384 : 1024;
    if (const char* e = getenv("EC_CHUNK")) chb = atoi(e);
    int st = (150 * 1024) / ((world_size + 1) * chb);
    if (st > 4) st = 4;
    if (const char* e = getenv("EC_STAGES")) st = atoi(e);
    if (st < 2) st = 2;
    if (st > 8) st = 8;
    // stay inside the opt-in shared-memory limit (227 KB per CTA, minus static)
    while (st > 2 && (long long)st * (world_size + 1) * chb > 200 * 1024) --st;
    while (chb > 1024 && (long long)st * (world_size + 1) * chb > 200 * 1024) chb /= 2;
    c->chv = chb / 16;
    c->stages = st;
    // one-shot for small messages (each rank pulls every slice and reduces
    // the whole vector into its own slot): no push / remote completion on the
    // round's critical path
    if (c->mode == 0 && world_size > 1) {
      // measured (profiles/r2_p2_oneshot.json, r2_sweep4_lead2.json): at P=2
      // one-shot wins up to ~1 MB (14.4 vs 16.4 us at 256 KB), at P=4 up to
      // 64 KB; beyond, the two-shot's split work (and progressive updates) win
      const char* e = getenv("EC_ONESHOT_BYTES");
      const long long lim = e ? atoll(e) : (world_size == 2 ? (1ll << 20) : 65536);
      if (n_elems * c->elem <= lim) c->mode = 3;
    }
    c->smem_bytes = (c->mode == 0 || c->mode == 3) ? st * (world_size + 1) * chb : 0;
  }
  if (!c->direct) {
    const int brc = budget_engine(c, w_default);
    if (brc) {
      delete c;
      return brc;
    }
  }
  if (const char* env = getenv("EC_TIMEOUT_S")) c->timeout_ns = (unsigned long long)(atof(env) * 1e9);
  {
    const char* env = getenv("EC_IDLE_PARK_MS");
    const double ms = env ? atof(env) : 100.0;
    c->idle_ns = ms > 0 ? (unsigned long long)(ms * 1e6) : 0ull;
  }
  c->ctrl.assign(world_size, nullptr);
  c->send.assign(world_size, nullptr);
  c->ring.assign(world_size, nullptr);
  c->gbuf.assign(world_size, nullptr);
  c->opened.assign(world_size, 0);
  for (int i = 0; i < n_local; ++i) {
    EcRankHost* r = new EcRankHost();
    r->rank = rank_lo + i;
    c->L.push_back(r);
    cudaError_t e;
    if ((e = cudaMalloc(&r->ctrl, sizeof(EcCtrl))) != cudaSuccess ||
        (e = cudaMalloc(&r->send, c->slot_bytes)) != cudaSuccess ||
        (e = cudaMalloc(&r->ring, c->slot_bytes * c->R)) != cudaSuccess ||
        (e = cudaMalloc(&r->gbuf, c->slot_bytes)) != cudaSuccess ||
        (e = cudaMemset(r->gbuf, 0, c->slot_bytes)) != cudaSuccess ||
        (e = cudaMalloc(&r->local, sizeof(EcLocal))) != cudaSuccess ||
        (e = cudaMemset(r->ctrl, 0, sizeof(EcCtrl))) != cudaSuccess ||
        (e = cudaMemset(r->send, 0, c->slot_bytes)) != cudaSuccess ||
        (e = cudaMemset(r->ring, 0, c->slot_bytes * c->R)) != cudaSuccess ||
        (e = cudaHostAlloc(&r->h, sizeof(EcHostCtl), cudaHostAllocMapped | cudaHostAllocPortable)) != cudaSuccess) {
      ec_comm_destroy(c);
      return fail(EC_E_NOMEM, "allocation failed: %s", cudaGetErrorString(e));
    }
    memset((void*)r->h, 0, sizeof(EcHostCtl));
    r->h->pin_lo = ~0ull;
    if ((e = cudaHostGetDevicePointer((void**)&r->hd, r->h, 0)) != cudaSuccess) {
      ec_comm_destroy(c);
      return fail(EC_E_CUDA, "cudaHostGetDevicePointer: %s", cudaGetErrorString(e));
    }
    std::unique_ptr<EcLocal> initp(new EcLocal());   // ~100 KB: not on the stack
    EcLocal& init = *initp;
    memset(&init, 0, sizeof(init));
    init.hold_from = EC_INF_GEN;
    init.contributed_round = -1;
    init.stash_null = 1;
    init.pin_dev = ~0ull;
    init.guard_tau = EC_INF_GEN;
    init.pend_lo = EC_INF_GEN;
    init.last_off = -1;
    if ((e = cudaMemcpy(r->local, &init, sizeof(init), cudaMemcpyHostToDevice)) != cudaSuccess) {
      ec_comm_destroy(c);
      return fail(EC_E_CUDA, "init local: %s", cudaGetErrorString(e));
    }
    c->ctrl[r->rank] = r->ctrl;
    c->send[r->rank] = r->send;
    c->ring[r->rank] = r->ring;
    c->gbuf[r->rank] = r->gbuf;
  }
  if (cudaMalloc(&c->d_descs, sizeof(EcDesc) * n_local) != cudaSuccess) {
    ec_comm_destroy(c);
    return fail(EC_E_NOMEM, "descriptor allocation failed");
  }
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if (cudaStreamCreateWithPriority(&c->es, cudaStreamNonBlocking, hi) != cudaSuccess) {
    ec_comm_destroy(c);
    return fail(EC_E_CUDA, "engine stream creation failed");
  }
  // the direct steps' publication stream (a world of one has no engine)
  if (c->direct && make_pub_stream(c, &c->pub_s, &c->pub_ev) != EC_OK) {
    ec_comm_destroy(c);
    return fail(EC_E_CUDA, "publication stream creation failed");
  }
  *out = c;
  return EC_OK;
}

int ec_comm_set_quorum(ec_comm_t* c, int min_arrivals) {
  if (!c) return fail(EC_E_ARG, "null communicator");
  if (c->running) return fail(EC_E_STATE, "set the quorum before the engine starts");
  if (min_arrivals < 0 || min_arrivals > c->P) return fail(EC_E_ARG, "quorum out of range");
  c->quorum = min_arrivals;
  return EC_OK;
}

int ec_comm_export(ec_comm_t* c, int li, void* blob, size_t cap, size_t* len) {
  int rc = check_li(c, li);
  if (rc) return rc;
  if (!blob || cap < sizeof(BlobV1)) return fail(EC_E_ARG, "blob buffer too small (%zu)", sizeof(BlobV1));
  EcRankHost* r = c->L[li];
  BlobV1 b;
  memset(&b, 0, sizeof(b));
  b.magic = BLOB_MAGIC;
  b.rank = r->rank;
  b.n = c->n;
  b.dtype = c->dtype;
  b.R = c->R;
  CK(cudaSetDevice(c->device));
  CK(cudaIpcGetMemHandle(&b.ctrl, r->ctrl));
  CK(cudaIpcGetMemHandle(&b.send, r->send));
  CK(cudaIpcGetMemHandle(&b.ring, r->ring));
  CK(cudaIpcGetMemHandle(&b.gbuf, r->gbuf));
  memcpy(blob, &b, sizeof(b));
  if (len) *len = sizeof(b);
  return EC_OK;
}

int ec_comm_import(ec_comm_t* c, int peer, const void* blob, size_t len) {
  if (!c) return fail(EC_E_ARG, "null communicator");
  if (peer < 0 || peer >= c->P) return fail(EC_E_ARG, "peer %d out of range", peer);
  if (peer >= c->rank_lo && peer < c->rank_lo + c->n_local) return EC_OK;  // local rank
  if (!blob || len < sizeof(BlobV1)) return fail(EC_E_ARG, "blob too short");
  BlobV1 b;
  memcpy(&b, blob, sizeof(b));
  if (b.magic != BLOB_MAGIC || b.rank != peer)
    return fail(EC_E_ARG, "blob is not rank %d's (magic %x rank %d)", peer, b.magic, b.rank);
  if (b.n != c->n || b.dtype != c->dtype || b.R != c->R)
    return fail(EC_E_ARG, "peer %d geometry mismatch (n %lld/%lld dtype %d/%d R %d/%d)", peer,
                b.n, c->n, b.dtype, c->dtype, b.R, c->R);
  if (c->opened[peer]) return EC_OK;
  CK(cudaSetDevice(c->device));
  void *pc = nullptr, *ps = nullptr, *pr = nullptr, *pg = nullptr;
  CK(cudaIpcOpenMemHandle(&pc, b.ctrl, cudaIpcMemLazyEnablePeerAccess));
  CK(cudaIpcOpenMemHandle(&ps, b.send, cudaIpcMemLazyEnablePeerAccess));
  CK(cudaIpcOpenMemHandle(&pr, b.ring, cudaIpcMemLazyEnablePeerAccess));
  CK(cudaIpcOpenMemHandle(&pg, b.gbuf, cudaIpcMemLazyEnablePeerAccess));
  c->ctrl[peer] = (EcCtrl*)pc;
  c->send[peer] = (char*)ps;
  c->ring[peer] = (char*)pr;
  c->gbuf[peer] = (char*)pg;
  c->opened[peer] = 1;
  return EC_OK;
}

int ec_comm_set_replay(ec_comm_t* c, int li, const uint64_t* masks, int64_t n) {
  int rc = check_li(c, li);
  if (rc) return rc;
  if (c->running) return fail(EC_E_STATE, "set_replay while the engine runs");
  if (c->direct) return fail(EC_E_STATE, "replay needs the persistent engine (world_size > 1)");
  EcRankHost* r = c->L[li];
  CK(cudaSetDevice(c->device));
  if (r->forced) {
    cudaFree(r->forced);
    r->forced = nullptr;
  }
  r->n_forced = 0;
  if (n > 0) {
    CK(cudaMalloc(&r->forced, sizeof(unsigned long long) * n));
    CK(cudaMemcpy(r->forced, masks, sizeof(unsigned long long) * n, cudaMemcpyHostToDevice));
    r->n_forced = n;
  }
  return EC_OK;
}

static int upload_descs(ec_comm_t* c) {
  for (int q = 0; q < c->P; ++q)
    if (!c->ctrl[q]) return fail(EC_E_STATE, "rank %d's buffers are not mapped (import first)", q);
  CK(cudaSetDevice(c->device));
  std::vector<EcDesc> d(c->n_local);
  const int V = 16 / c->elem;
  for (int i = 0; i < c->n_local; ++i) {
    EcRankHost* r = c->L[i];
    EcDesc& x = d[i];
    memset(&x, 0, sizeof(x));
    x.rank = r->rank;
    x.P = c->P;
    x.flavor = c->flavor;
    x.dtype = c->dtype;
    x.R = c->R;
    x.W = c->W;
    x.w_step = c->w_step < c->W ? c->w_step : c->W;   // W may have shrunk to the budget
    // arrival words of progressive updates: < 0 (default) geometric, after
    // 1/2, 3/4, 7/8, ... of a worker's chunks (P=4 step: 14.37k vs 14.28k
    // steps/s with ~4 evenly spaced words, profiles/r2_signal_n4.log);
    // 0: ~4 evenly spaced; k > 0: one word per k chunks
    x.sig_every = getenv("EC_SIGNAL_EVERY") ? atoi(getenv("EC_SIGNAL_EVERY")) : -1;
    if (x.sig_every < 0) x.sig_every = -1;
    x.replay = r->forced != nullptr;
    x.vec = V;
    x.n = c->n;
    x.nvec = c->n / V;
    x.slot_bytes = c->slot_bytes;
    x.n_forced = r->n_forced;
    x.timeout_ns = c->timeout_ns;
    x.mode = c->mode;
    x.chv = c->chv;
    x.stages = c->stages;
    x.smem_bytes = c->smem_bytes;
    // two rounds in flight (the next one's snapshot overlaps this one's data
    // phase) need the fused TMA pipeline and a third result slot for readers
    c->lead = ((c->mode == 0 || c->mode == 3) && c->R >= 3 && !getenv("EC_NO_LEAD")) ? 2 : 1;
    x.lead = c->lead;
    x.quorum = c->flavor == EC_MAJORITY ? c->quorum : 0;
    x.idle_sleep_ns = getenv("EC_IDLE_SLEEP_NS") ? (unsigned)atoi(getenv("EC_IDLE_SLEEP_NS")) : 512u;
    if (x.idle_sleep_ns < 32) x.idle_sleep_ns = 32;
    for (int q = 0; q < c->P; ++q) {
      x.ctrl[q] = c->ctrl[q];
      x.send[q] = c->send[q];
      x.ring[q] = c->ring[q];
      x.gbuf[q] = c->gbuf[q];
    }
    if (c->mode == 2) {
      x.mc_stage = (char*)c->mc_va;
      x.mc_ring = (char*)c->mc_va + c->slot_bytes;
      x.uc_stage = (char*)c->uc_va;
    }
    x.hctl = r->hd;
    x.local = r->local;
    x.park_votes = &c->L[0]->local->park_votes;
    x.n_local = c->n_local;
    x.forced = r->forced;
    astore(&r->h->stop, 0ull);
  }
  CK(cudaMemcpy(c->d_descs, d.data(), sizeof(EcDesc) * c->n_local, cudaMemcpyHostToDevice));
  return EC_OK;
}

// direct mode: a host-posted request is answered by kernels on the caller's
// stream, which must follow every step publication already queued on the
// publication stream (replies and done generations are written in order)
static int order_after_pub(ec_comm_t* c, cudaStream_t s) {
  if (!c->pub_used) return EC_OK;
  if (!c->pub_join_ev) CK(cudaEventCreateWithFlags(&c->pub_join_ev, cudaEventDisableTiming));
  CK(cudaEventRecord(c->pub_join_ev, c->pub_s));
  CK(cudaStreamWaitEvent(s, c->pub_join_ev, 0));
  return EC_OK;
}

// direct mode: remember where a host-posted request's kernels went
static int note_request(ec_comm_t* c, cudaStream_t s) {
  if (!c->req_ev) CK(cudaEventCreateWithFlags(&c->req_ev, cudaEventDisableTiming));
  CK(cudaEventRecord(c->req_ev, s));
  c->req_stream = s;
  c->req_pending = true;
  return EC_OK;
}

static inline void touch(ec_comm_t* c) { c->last_api_ns.store(now_ns(), std::memory_order_relaxed); }

// (re)launch the persistent engine for a new epoch; caller holds live_mu
static int launch_epoch(ec_comm_t* c) {
  CK(cudaSetDevice(c->device));
  for (EcRankHost* r : c->L) astore(&r->h->stop, 0ull);
  c->epoch += 1;
  // the launch's park-vote counter starts from zero (stream-ordered before it)
  CK(cudaMemsetAsync(&c->L[0]->local->park_votes, 0, sizeof(unsigned long long), c->es));
  CK(launch_engine(c->dtype, c->d_descs, c->n_local, 1 + c->W, c->epoch, c->smem_bytes, c->es));
  c->parked_auto.store(false);
  return EC_OK;
}

// Every posting entry point runs under live_mu and calls this first: a
// communicator the watcher parked for idleness is relaunched before the post.
static int ensure_live(ec_comm_t* c) {
  touch(c);
  if (c->running && c->parked_auto.load()) {
    c->idle_wakes += 1;
    return launch_epoch(c);
  }
  return EC_OK;
}

// True when every local rank's engine has exited launch `epoch`.
static bool all_exited(ec_comm_t* c) {
  for (EcRankHost* r : c->L)
    if (aload(&r->h->exited) != c->epoch) return false;
  return true;
}

// Idle park.  A persistent engine makes every device-wide synchronisation
// (torch.cuda.synchronize, cudaFree in the caching allocator, cuDNN's RNN
// setup, lazy module loads) wait for it.  This thread parks the engine once
// the communicator has had no API call and completed no round for idle_ns and
// nothing is outstanding (every reserved request processed, no snapshot
// pending publication): it asks the controllers to exit if idle (stop = 2;
// the local controllers vote and exit together), so user syncs return.  The
// next post relaunches the engine (ensure_live).  While parked, a rank with
// remote peers polls its control block for their activation / snapshot /
// arrival words of its next generation and relaunches when one appears (the
// peers' round needs this rank's snapshot and owner shard).
static void watcher_main(ec_comm_t* c) {
  cudaSetDevice(c->device);
  unsigned long long last_done = ~0ull, last_change = now_ns();
  const bool remote = c->P > c->n_local;
  while (!c->quit.load()) {
    const bool parked = c->parked_auto.load();
    std::this_thread::sleep_for(std::chrono::microseconds(parked && remote ? 100 : 1000));
    std::unique_lock<std::recursive_mutex> lk(c->live_mu);
    if (c->quit.load() || !c->running) continue;
    const unsigned long long now = now_ns();
    if (!c->parked_auto.load()) {
      unsigned long long dsum = 0;
      for (EcRankHost* r : c->L) dsum += aload(&r->h->done_gen1);
      if (dsum != last_done) {
        last_done = dsum;
        last_change = now;
      }
      const unsigned long long api = c->last_api_ns.load(std::memory_order_relaxed);
      const unsigned long long last = api > last_change ? api : last_change;
      if (now - last < c->idle_ns) continue;
      bool idle = true;
      for (EcRankHost* r : c->L)
        idle = idle && aload(&r->h->req_done) == r->next_seq &&
               aload(&r->h->snap_gen1) == aload(&r->h->done_gen1) && !aload(&r->h->error);
      if (!idle) continue;
      for (EcRankHost* r : c->L) astore(&r->h->stop, 2ull);
      Backoff bo;
      while (!all_exited(c) && !bo.expired(20)) bo.pause();
      if (!all_exited(c)) {
        // not idle after all (a peer's round arrived): withdraw; a park the
        // controllers had already committed to still completes
        for (EcRankHost* r : c->L) astore(&r->h->stop, 0ull);
        Backoff b2;
        bool any = false;
        while (!b2.expired(2)) b2.pause();
        for (EcRankHost* r : c->L) any = any || aload(&r->h->exited) == c->epoch;
        if (!any) {
          last_change = now_ns();
          continue;
        }
        while (!all_exited(c)) std::this_thread::sleep_for(std::chrono::microseconds(50));
      }
      cudaStreamSynchronize(c->es);
      for (EcRankHost* r : c->L) astore(&r->h->stop, 0ull);
      c->parked_auto.store(true);
      c->idle_parks += 1;
    } else if (remote) {
      bool wake = false;
      for (EcRankHost* r : c->L) {
        const unsigned long long g1 = aload(&r->h->done_gen1) + 1;   // next generation + 1
        const size_t words = (size_t)3 * EC_MAX_P;
        if (cudaMemcpyAsync(c->poll_buf, r->ctrl, words * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, c->ws) != cudaSuccess ||
            cudaStreamSynchronize(c->ws) != cudaSuccess)
          break;
        const unsigned long long* act = c->poll_buf;
        const unsigned long long* snap = c->poll_buf + EC_MAX_P;
        for (int q = 0; q < c->P && !wake; ++q)
          wake = act[q] >= g1 || (snap[q] >> EC_SNAP_SHIFT) >= g1;
        if (!wake) {   // arrive_from sits after rsdone_from in EcCtrl
          if (cudaMemcpyAsync(c->poll_buf, r->ctrl->arrive_from, EC_MAX_P * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, c->ws) == cudaSuccess &&
              cudaStreamSynchronize(c->ws) == cudaSuccess)
            for (int q = 0; q < c->P && !wake; ++q) wake = c->poll_buf[q] >= g1;
        }
        if (wake) break;
      }
      if (wake) {
        c->idle_wakes += 1;
        launch_epoch(c);
        last_change = now_ns();
      }
    }
  }
}

int ec_comm_start(ec_comm_t* c) {
  if (!c) return fail(EC_E_ARG, "null communicator");
  std::lock_guard<std::recursive_mutex> lk(c->live_mu);
  touch(c);
  if (c->running) return ensure_live(c);
  int rc = upload_descs(c);
  if (rc) return rc;
  if (c->direct) {
    c->running = true;
    return EC_OK;
  }
  if ((rc = launch_epoch(c))) return rc;
  c->running = true;
  if (c->idle_ns && !c->watcher.joinable()) {
    if (!c->poll_buf && cudaHostAlloc((void**)&c->poll_buf, 3 * EC_MAX_P * sizeof(unsigned long long),
                                      cudaHostAllocDefault) != cudaSuccess)
      return fail(EC_E_NOMEM, "watcher buffer");
    if (!c->ws) CK(cudaStreamCreateWithFlags(&c->ws, cudaStreamNonBlocking));
    c->watcher = std::thread(watcher_main, c);
  }
  return EC_OK;
}

int ec_comm_pause(ec_comm_t* c, int timeout_ms) {
  if (!c) return fail(EC_E_ARG, "null communicator");
  std::lock_guard<std::recursive_mutex> lk(c->live_mu);
  if (!c->running) return EC_OK;
  if (c->direct) {
    c->running = false;
    return EC_OK;
  }
  if (c->parked_auto.load()) {     // already parked by the idle watcher
    c->running = false;
    c->parked_auto.store(false);
    return EC_OK;
  }
  for (EcRankHost* r : c->L) astore(&r->h->stop, 1ull);
  Backoff bo;
  for (EcRankHost* r : c->L) {
    while (aload(&r->h->exited) != c->epoch) {
      if (bo.expired(timeout_ms))
        return fail(EC_E_TIMEOUT, "engine of rank %d did not park within %d ms", r->rank, timeout_ms);
      bo.pause();
    }
  }
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->es));
  c->running = false;
  for (EcRankHost* r : c->L) astore(&r->h->stop, 0ull);
  return EC_OK;
}

int ec_comm_destroy(ec_comm_t* c) {
  if (!c) return EC_OK;
  int rc = EC_OK;
  c->quit.store(true);
  if (c->watcher.joinable()) c->watcher.join();
  cudaSetDevice(c->device);
  if (c->running) rc = ec_comm_pause(c, 10000);
  if (c->running) {
    // the engine did not park: do not free memory a live kernel still touches
    return fail(EC_E_STATE, "engine still running; communicator leaked");
  }
  for (int q = 0; q < c->P; ++q) {
    if (c->opened[q]) {
      cudaIpcCloseMemHandle(c->ctrl[q]);
      cudaIpcCloseMemHandle(c->send[q]);
      cudaIpcCloseMemHandle(c->ring[q]);
      cudaIpcCloseMemHandle(c->gbuf[q]);
    }
  }
  nvls_teardown(c);
  if (c->pub_s) {
    cudaStreamSynchronize(c->pub_s);   // a step's publication may still run
    cudaStreamDestroy(c->pub_s);
    cudaEventDestroy(c->pub_ev);
    if (c->pub_join_ev) cudaEventDestroy(c->pub_join_ev);
    if (c->req_ev) cudaEventDestroy(c->req_ev);
  }
  for (EcRankHost* r : c->L) {
    if (r->ctrl) cudaFree(r->ctrl);
    if (r->send) cudaFree(r->send);
    if (r->ring) cudaFree(r->ring);
    if (r->gbuf) cudaFree(r->gbuf);
    if (r->local) cudaFree(r->local);
    if (r->forced) cudaFree(r->forced);
    if (r->unpin_ev) cudaEventDestroy(r->unpin_ev);

    if (r->h) cudaFreeHost(r->h);
    delete r;
  }
  if (c->d_descs) cudaFree(c->d_descs);
  if (c->es) cudaStreamDestroy(c->es);
  if (c->ws) cudaStreamDestroy(c->ws);
  if (c->poll_buf) cudaFreeHost(c->poll_buf);
  budget_release(c);
  delete c;
  return rc;
}

int ec_comm_error(ec_comm_t* c, int li, uint64_t* code, uint64_t* info) {
  int rc = check_li(c, li);
  if (rc) return rc;
  if (code) *code = aload(&c->L[li]->h->error);
  if (info) *info = aload(&c->L[li]->h->error_info);
  return EC_OK;
}

void* ec_send_ptr(ec_comm_t* c, int li) {
  if (check_li(c, li)) return nullptr;
  return c->L[li]->send;
}

void* ec_grad_ptr(ec_comm_t* c, int li) {
  if (check_li(c, li)) return nullptr;
  return c->L[li]->gbuf;
}

void* ec_slot_ptr(ec_comm_t* c, int li, int64_t gen) {
  if (check_li(c, li) || gen < 0) return nullptr;
  return c->L[li]->ring + (gen % c->R) * c->slot_bytes;
}

int64_t ec_n_elems(ec_comm_t* c) { return c ? c->n : -1; }
int ec_comm_set_generation(ec_comm_t* c, int li, int64_t gen, int stash_pending,
                           int64_t contributed_round) {
  int rc = check_li(c, li);
  if (rc) return rc;
  if (c->running) return fail(EC_E_STATE, "pause the engine before re-basing its generation");
  if (gen < 0) return fail(EC_E_ARG, "generation must be >= 0");
  EcRankHost* r = c->L[li];
  CK(cudaSetDevice(c->device));
  if (c->pub_s) CK(cudaStreamSynchronize(c->pub_s));   // no step publication still queued
  // the engine's own stream is idle while it is parked
  cudaError_t e = launch_set_generation(r->local, r->hd, gen, stash_pending ? 1 : 0,
                                        contributed_round, c->es);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->es);
  if (e != cudaSuccess) return fail(EC_E_CUDA, "set generation: %s", cudaGetErrorString(e));
  return EC_OK;
}

int ec_stream_barrier(ec_comm_t* c, int li, void* stream) {
  int rc = check_li(c, li);
  if (rc) return rc;
  if (!c->ctrl[0]) return fail(EC_E_STATE, "rank 0's control block is not mapped (import first)");
  EcRankHost* r = c->L[li];
  // every rank's epoch advances in lockstep: the k-th barrier completes at k*P
  const unsigned long long epoch = ++r->bar_epoch;
  CK(launch_stream_barrier(&c->ctrl[0]->bar_count, epoch * (unsigned long long)c->P, r->hd,
                           c->timeout_ns, (cudaStream_t)stream));
  return EC_OK;
}

int ec_comm_progressive(ec_comm_t* c) {
  return c ? (!c->direct && c->mode == 0 && (c->w_step < c->W ? c->w_step : c->W) <= EC_PROG_W &&
               c->dtype != EC_I64) : -1;
}

int ec_fold(ec_comm_t* c, int li, const void* grad, int mode, void* stream) {
  int rc = check_li(c, li);
  if (rc) return rc;
  if (!grad) return fail(EC_E_ARG, "null gradient");
  EcRankHost* r = c->L[li];
  // into a pending stash: check first, so a non-finite gradient is refused
  // (EC_R_POISONED at the post) without touching the gradients it holds
  CK(launch_fold(c->dtype, r->send, grad, c->n, mode, &r->local->poison, (cudaStream_t)stream,
                 mode == EC_FOLD_ADD));
  return EC_OK;
}

int ec_copy_in(ec_comm_t* c, int li, const void* src, void* stream) {
  int rc = check_li(c, li);
  if (rc) return rc;
  EcRankHost* r = c->L[li];
  if (src != r->send)
    CK(cudaMemcpyAsync(r->send, src, c->n * c->elem, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return EC_OK;
}

static int reserve_seq(ec_comm_t* c, EcRankHost* r, unsigned long long* seq) {
  Backoff bo;
  while (r->next_seq - aload(&r->h->req_done) >= EC_REQ_RING) {
    if (bo.expired(60000)) return fail(EC_E_TIMEOUT, "request ring full at rank %d", r->rank);
    int e = device_error(r);
    if (e) return e;
    bo.pause();
  }
  *seq = r->next_seq++;
  (void)c;
  return EC_OK;
}

static int host_post(ec_comm_t* c, int li, unsigned type, unsigned flags, long long t, long long arg,
                     uint64_t* seq_out) {
  int rc = check_li(c, li);
  if (rc) return rc;
  EcRankHost* r = c->L[li];
  std::lock_guard<std::recursive_mutex> live(c->live_mu);
  if ((rc = ensure_live(c))) return rc;
  std::lock_guard<std::mutex> g(r->mu);
  unsigned long long seq;
  if ((rc = reserve_seq(c, r, &seq))) return rc;
  if (c->direct) {
    if (!c->running && (rc = ec_comm_start(c))) return rc;
    if ((rc = order_after_pub(c, (cudaStream_t)c->last_stream))) return rc;
    CK(launch_direct(c->dtype, c->d_descs + li, c->n / (16 / c->elem), seq, type, flags, t, arg,
                     (cudaStream_t)c->last_stream));
    if ((rc = note_request(c, (cudaStream_t)c->last_stream))) return rc;
    if (seq_out) *seq_out = seq;
    return EC_OK;
  }
  EcReq* q = &r->h->req[seq % EC_REQ_RING];
  q->type = type;
  q->flags = flags;
  q->t = t;
  q->arg = arg;
  __atomic_thread_fence(__ATOMIC_SEQ_CST);
  astore(&q->seq1, seq + 1);
  if (seq_out) *seq_out = seq;
  return EC_OK;
}

int ec_post_contribute(ec_comm_t* c, int li, int64_t t, uint32_t flags, void* stream, uint64_t* seq_out) {
  int rc = check_li(c, li);
  if (rc) return rc;
  EcRankHost* r = c->L[li];
  std::lock_guard<std::recursive_mutex> live(c->live_mu);
  if ((rc = ensure_live(c))) return rc;
  std::lock_guard<std::mutex> g(r->mu);
  unsigned long long seq;
  if ((rc = reserve_seq(c, r, &seq))) return rc;
  if (c->direct) {
    if (!c->running && (rc = ec_comm_start(c))) return rc;
    c->last_stream = stream;
    if ((rc = order_after_pub(c, (cudaStream_t)stream))) return rc;
    CK(launch_direct(c->dtype, c->d_descs + li, c->n / (16 / c->elem), seq, EC_REQ_CONTRIB,
                     flags & 7u, t, 0, (cudaStream_t)stream));
    if ((rc = note_request(c, (cudaStream_t)stream))) return rc;
    if (seq_out) *seq_out = seq;
    return EC_OK;
  }
  CK(launch_post(r->local, seq + 1, EC_REQ_CONTRIB, flags & 7u, t, 0, (cudaStream_t)stream));
  if (seq_out) *seq_out = seq;
  return EC_OK;
}

int ec_post_activate(ec_comm_t* c, int li, int64_t t, uint64_t* seq) {
  return host_post(c, li, EC_REQ_ACTIVATE, 0, t, 0, seq);
}

int ec_post_hold(ec_comm_t* c, int li, int64_t hold_from, uint64_t* seq) {
  return host_post(c, li, EC_REQ_HOLD, 0, 0, hold_from, seq);
}

int ec_post_guard(ec_comm_t* c, int li, int64_t tau, int64_t pending_lo, uint64_t* seq) {
  return host_post(c, li, EC_REQ_GUARD, 0, pending_lo, tau, seq);
}

int ec_reply(ec_comm_t* c, int li, uint64_t seq, int timeout_ms, int* status) {
  int rc = check_li(c, li);
  if (rc) return rc;
  touch(c);
  EcRankHost* r = c->L[li];
  Backoff bo;
  while (true) {
    unsigned long long v = aload(&r->h->reply[seq % EC_REQ_RING]);
    if ((v >> 8) == seq + 1) {
      if (status) *status = (int)(v & 0xff);
      return EC_OK;
    }
    if (timeout_ms == 0) {
      if (status) *status = EC_R_PENDING;
      return EC_OK;
    }
    if ((rc = device_error(r))) return rc;
    if (bo.expired(timeout_ms))
      return fail(EC_E_TIMEOUT, "rank %d: no reply to request %llu within %d ms", r->rank,
                  (unsigned long long)seq, timeout_ms);
    bo.pause();
  }
}

int ec_done_gen(ec_comm_t* c, int li, int64_t* gen) {
  int rc = check_li(c, li);
  if (rc) return rc;
  if (gen) *gen = (int64_t)aload(&c->L[li]->h->done_gen1) - 1;
  return EC_OK;
}

int ec_gen_info(ec_comm_t* c, int li, int64_t gen, uint64_t* mask, uint64_t* has, int* nap) {
  int rc = check_li(c, li);
  if (rc) return rc;
  EcRankHost* r = c->L[li];
  if (gen < 0 || (long long)aload(&r->h->done_gen1) <= gen)
    return fail(EC_E_STATE, "generation %lld has not completed", (long long)gen);
  EcLog* lg = &r->h->log[gen % EC_LOG_RING];
  unsigned long long g1 = aload(&lg->gen1);
  unsigned long long m = aload(&lg->mask), hm = aload(&lg->has), np = aload(&lg->nap);
  __atomic_thread_fence(__ATOMIC_ACQUIRE);
  if (aload(&lg->gen1) != g1 || g1 != (unsigned long long)gen + 1) {
    if (g1 > (unsigned long long)gen + 1 || (long long)aload(&r->h->done_gen1) > gen + EC_LOG_RING)
      return fail(EC_E_STATE, "generation %lld fell out of the %d-entry log", (long long)gen, EC_LOG_RING);
    // done says the entry exists: its stores are in flight (never observed
    // since the tag moved before the publisher's fence; kept as a guard)
    Backoff bo;
    while (aload(&lg->gen1) != (unsigned long long)gen + 1) {
      if (bo.expired(1000))
        return fail(EC_E_STATE, "generation %lld: log entry not published", (long long)gen);
      bo.pause();
    }
    __atomic_thread_fence(__ATOMIC_ACQUIRE);
    m = aload(&lg->mask);
    hm = aload(&lg->has);
    np = aload(&lg->nap);
  }
  if (mask) *mask = m;
  if (has) *has = hm;
  if (nap) *nap = (int)np;
  return EC_OK;
}

int ec_gen_times(ec_comm_t* c, int li, int64_t gen, uint64_t* t5) {
  int rc = check_li(c, li);
  if (rc) return rc;
  EcRankHost* r = c->L[li];
  if (gen < 0 || (long long)aload(&r->h->done_gen1) <= gen)
    return fail(EC_E_STATE, "generation %lld has not completed", (long long)gen);
  EcLog* lg = &r->h->log[gen % EC_LOG_RING];
  {
    // done says the entry exists; wait out stores still in flight (guard)
    Backoff bo;
    while (aload(&lg->gen1) < (unsigned long long)gen + 1 && !bo.expired(1000)) bo.pause();
  }
  unsigned long long g1 = aload(&lg->gen1);
  t5[0] = aload(&lg->t_snap);
  t5[1] = aload(&lg->t_cmd);
  t5[2] = aload(&lg->t_rs);
  t5[3] = aload(&lg->t_done);
  t5[4] = aload(&lg->t_req);
  __atomic_thread_fence(__ATOMIC_ACQUIRE);
  if (aload(&lg->gen1) != g1 || g1 != (unsigned long long)gen + 1)
    return fail(EC_E_STATE, "generation %lld fell out of the log", (long long)gen);
  return EC_OK;
}

int ec_wait(ec_comm_t* c, int li, int64_t t, int timeout_ms, int pin, int64_t* gen_out,
            uint64_t* mask, int* nap) {
  int rc = check_li(c, li);
  if (rc) return rc;
  touch(c);
  EcRankHost* r = c->L[li];
  Backoff bo;
  unsigned long long d1;
  while ((d1 = aload(&r->h->done_gen1)) < (unsigned long long)t + 1) {
    if ((rc = device_error(r))) return rc;
    if (bo.expired(timeout_ms))
      return fail(EC_E_TIMEOUT, "rank %d round %lld did not complete", r->rank, (long long)t);
    bo.pause();
  }
  long long G = (long long)d1 - 1;
  std::unique_lock<std::mutex> pin_lock(r->pin_mu, std::defer_lock);
  if (pin && !c->direct) {
    // A stream-ordered unpin of an earlier read may still be queued (e.g.
    // behind that read's clone): let it land first, or it would clear this pin
    // after the handshake below and the engine could reuse the slot under us.
    pin_lock.lock();
    if (r->unpin_pending) {
      CK(cudaEventSynchronize(r->unpin_ev));
      r->unpin_pending = false;
    }
    // Pin handshake with the controller's pre-snapshot check (ec_kernels.cu):
    // publish the pin, wait until the controller has acknowledged seeing it
    // (it refreshes the host pin every few us), then make sure the engine had
    // not already passed the check for the round that would reuse G's slot.
    while (true) {
      __atomic_store_n(&r->h->pin_lo, (unsigned long long)G, __ATOMIC_SEQ_CST);
      const unsigned long long ps = __atomic_add_fetch(&r->h->pin_seq, 1ull, __ATOMIC_SEQ_CST);
      Backoff ab;
      // a parked engine (paused, or parked for idleness) re-reads the pin at start
      while (c->running && !c->parked_auto.load() && aload(&r->h->pin_ack) < ps) {
        if ((rc = device_error(r))) return rc;
        if (ab.expired(timeout_ms < 0 ? 10000 : timeout_ms))
          return fail(EC_E_TIMEOUT, "rank %d: engine did not acknowledge the pin", r->rank);
        ab.pause();
      }
      long long D = (long long)aload(&r->h->done_gen1) - 1;
      if (D < G + c->R - c->lead) break;   // no snapshot of G + R yet (see wait_and_pin)
      G = D;
    }
  }
  if (gen_out) *gen_out = G;
  if (mask || nap) {
    uint64_t m = 0;
    int np = 0;
    if ((rc = ec_gen_info(c, li, G, &m, nullptr, &np))) return rc;
    if (mask) *mask = m;
    if (nap) *nap = np;
  }
  return EC_OK;
}

// ---- kernel-duration instrumentation for ec_step (bench.py roofline) --------
struct EcTimedLaunch {
  int kind;  // 0 fold, 1 update
  cudaEvent_t a, b;
};
static std::mutex g_prof_mu;
static int g_prof_on = 0;
static std::vector<EcTimedLaunch> g_prof;
static std::vector<cudaEvent_t> g_ev_pool;

static cudaEvent_t prof_event() {
  if (!g_ev_pool.empty()) {
    cudaEvent_t e = g_ev_pool.back();
    g_ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

struct ProfScope {
  int kind;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  ProfScope(int k, void* stream) : kind(k), s((cudaStream_t)stream) {
    if (!__atomic_load_n(&g_prof_on, __ATOMIC_RELAXED)) return;
    std::lock_guard<std::mutex> g(g_prof_mu);
    a = prof_event();
    cudaEventRecord(a, s);
  }
  ~ProfScope() {
    if (!a) return;
    std::lock_guard<std::mutex> g(g_prof_mu);
    cudaEvent_t b = prof_event();
    cudaEventRecord(b, s);
    g_prof.push_back({kind, a, b});
  }
};

int ec_step_update_ns(ec_comm_t* c, int li, uint64_t* ns) {
  int rc = check_li(c, li);
  if (rc) return rc;
  *ns = c->L[li]->last_update_ns;
  return EC_OK;
}

int ec_profile_enable(int on) {
  __atomic_store_n(&g_prof_on, on ? 1 : 0, __ATOMIC_RELAXED);
  return EC_OK;
}

int ec_profile_read(double* ms_sum, int64_t* counts) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  ms_sum[0] = ms_sum[1] = 0.0;
  counts[0] = counts[1] = 0;
  for (auto& x : g_prof) {
    float ms = 0.f;
    cudaEventSynchronize(x.b);
    if (cudaEventElapsedTime(&ms, x.a, x.b) == cudaSuccess) {
      ms_sum[x.kind] += ms;
      counts[x.kind] += 1;
    }
    g_ev_pool.push_back(x.a);
    g_ev_pool.push_back(x.b);
  }
  g_prof.clear();
  return EC_OK;
}

int ec_round(ec_comm_t* c, int li, int64_t t, uint32_t flags, void* stream, int timeout_ms,
             int* status, int64_t* gen, uint64_t* mask, int* nap) {
  uint64_t seq;
  int rc = ec_post_contribute(c, li, t, flags, stream, &seq);
  if (rc) return rc;
  int st = 0;
  if ((rc = ec_reply(c, li, seq, timeout_ms, &st))) return rc;
  if (status) *status = st;
  if (st == EC_R_POISONED || st == EC_R_ERROR) return EC_OK;
  return ec_wait(c, li, t, timeout_ms, 0, gen, mask, nap);
}

int ec_round_async(ec_comm_t* c, int li, int64_t t, uint32_t flags, void* stream, uint64_t* seq) {
  int rc = ec_post_contribute(c, li, t, flags, stream, seq);
  if (rc) return rc;
  EcRankHost* r = c->L[li];
  CK(launch_wait_done(r->local, r->hd, t, c->timeout_ns, (cudaStream_t)stream));
  return EC_OK;
}

int ec_step(ec_comm_t* c, int li, int64_t t, const void* grad, int fold_mode, uint32_t flags,
            void* w, void* mom, double lr, double mu, void* stream, int timeout_ms,
            int* status, int64_t* gen, uint64_t* mask, int* nap) {
  int rc = check_li(c, li);
  if (rc) return rc;
  if (!w) return fail(EC_E_ARG, "null weights");
  if (grad) {
    ProfScope ps(0, stream);
    if ((rc = ec_fold(c, li, grad, fold_mode, stream))) return rc;
  }
  uint64_t seq;
  if ((rc = ec_post_contribute(c, li, t, flags, stream, &seq))) return rc;
  int st = 0;
  if ((rc = ec_reply(c, li, seq, timeout_ms, &st))) return rc;
  if (status) *status = st;
  if (st == EC_R_POISONED || st == EC_R_ERROR) return EC_OK;
  int64_t G;
  if ((rc = ec_wait(c, li, t, timeout_ms, 1, &G, mask, nap))) return rc;
  if (gen) *gen = G;
  const void* u = ec_slot_ptr(c, li, G);
  {
    ProfScope ps(1, stream);
    if (mom && mu != 0.0) rc = ec_momentum_update(w, mom, u, lr, mu, c->n, c->dtype, stream);
    else rc = ec_sgd_update(w, u, lr, c->n, c->dtype, stream);
  }
  if (rc) return rc;
  return ec_set_pin(c, li, ~0ull, 1, stream);
}

int ec_step_async(ec_comm_t* c, int li, int64_t t, const void* grad, uint32_t flags, void* w,
                  void* mom, double lr, double mu, void* stream, uint64_t* seq_out) {
  int rc = check_li(c, li);
  if (rc) return rc;
  if (!w || !grad) return fail(EC_E_ARG, "null weights or gradient");
  if (c->dtype == EC_I64) return fail(EC_E_ARG, "eager-SGD step needs a float dtype");
  EcRankHost* r = c->L[li];
  cudaStream_t s = (cudaStream_t)stream;
  {
    // every step carries a fresh request sequence number and generation in
    // its launch arguments: a captured graph would replay stale ones
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(s, &cap));
    if (cap != cudaStreamCaptureStatusNone)
      return fail(EC_E_STATE, "ec_step_async cannot be captured into a CUDA graph");
  }
  // reservation and launches under live_mu: the idle watcher never parks with
  // a reserved request outstanding
  std::lock_guard<std::recursive_mutex> live(c->live_mu);
  if (!c->running && (rc = ec_comm_start(c))) return rc;
  if ((rc = ensure_live(c))) return rc;
  unsigned long long seq;
  {
    std::lock_guard<std::mutex> g(r->mu);
    if ((rc = reserve_seq(c, r, &seq))) return rc;
  }
  const bool zero_copy = grad == r->gbuf;
  // progressive update: the update kernel behind this offer consumes the
  // round's chunks as they land (owners publish arrival words to us)
  const void* mom_eff = (mom && mu != 0.0) ? mom : nullptr;
  const bool prog = !c->direct && ec_comm_progressive(c) == 1 && !getenv("EC_NO_PROGRESSIVE") &&
                    ((((uintptr_t)w) | ((uintptr_t)mom_eff)) & 15) == 0;
  if (!(c->direct && zero_copy)) {
    // fold (+ the offer's post, fused into the fold's last CTA, engine mode).
    // A world of one offering its registered buffer needs no fold launch: the
    // step kernel offers it in place, or folds it into a pending stash in-pass
    ProfScope ps(0, stream);
    CK(launch_fold_auto(c->dtype, r->send, grad, c->n, r->local, c->direct ? 0 : seq + 1,
                        (flags & 7u) | (prog ? EC_CF_STEP : 0u), t, zero_copy ? 1 : 0, s));
  }
  if (c->direct) {
    // decide + round + update in one launch (see ec_direct_step_kernel); its
    // publication on the communicator's publication stream (not while the
    // caller captures a graph: then behind it, on the same stream)
    c->last_stream = stream;
    const bool side = !getenv("EC_PUBLISH_SAME_STREAM");
    if (side && !c->pub_s && (rc = make_pub_stream(c, &c->pub_s, &c->pub_ev))) return rc;
    if (side) c->pub_used = true;
    if (c->req_pending && c->req_stream != s) CK(cudaStreamWaitEvent(s, c->req_ev, 0));
    c->req_pending = false;
    ProfScope ps(1, stream);
    CK(launch_direct_step(c->dtype, c->d_descs + li, seq,
                          (flags & 7u) | (grad == r->gbuf ? EC_CF_SRC_GRAD_AUTO : 0u), w,
                          (mom && mu != 0.0) ? mom : nullptr, r->ring, c->slot_bytes, r->send,
                          r->gbuf, lr, mu, c->n, t, c->timeout_ns, s, side ? c->pub_s : nullptr,
                          c->pub_ev));
    if (seq_out) *seq_out = seq;
    return EC_OK;
  }
  {
    // device wait for a generation >= t + pin, update, unpin: one launch
    ProfScope ps(1, stream);
    CK(launch_update_gen(c->dtype, w, (mom && mu != 0.0) ? mom : nullptr, r->ring, c->slot_bytes, c->R,
                         r->local, lr, mu, c->n, r->hd, t, c->timeout_ns, seq + 1, r->send,
                         r->gbuf, c->d_descs + li, prog ? 1 : 0, c->n_local, s));
  }
  if (seq_out) *seq_out = seq;
  return EC_OK;
}

int ec_step_result(ec_comm_t* c, int li, uint64_t seq, int64_t t, int timeout_ms, int* status,
                   int64_t* gen, uint64_t* mask, int* nap) {
  int rc = check_li(c, li);
  if (rc) return rc;
  touch(c);
  EcRankHost* r = c->L[li];
  if ((rc = ec_reply(c, li, seq, timeout_ms, status))) return rc;
  if (status && (*status == EC_R_POISONED || *status == EC_R_ERROR)) return EC_OK;
  Backoff bo;
  while (aload(&r->h->steptag[t % EC_REQ_RING]) != (unsigned long long)t + 1) {
    if ((rc = device_error(r))) return rc;
    if (bo.expired(timeout_ms))
      return fail(EC_E_TIMEOUT, "rank %d step %lld did not complete", r->rank, (long long)t);
    bo.pause();
  }
  const int64_t G = (int64_t)aload(&r->h->stepgen[t % EC_REQ_RING]) - 1;
  if (gen) *gen = G;
  // the device mirror of done runs ahead of the host-visible log: wait for it
  while ((int64_t)aload(&r->h->done_gen1) <= G) {
    if ((rc = device_error(r))) return rc;
    if (bo.expired(timeout_ms)) return fail(EC_E_TIMEOUT, "rank %d log of generation %lld", r->rank, (long long)G);
    bo.pause();
  }
  r->last_update_ns = aload(&r->h->stepns[t % EC_REQ_RING]);
  if (status && aload(&r->h->stepbad[t % EC_REQ_RING])) *status = EC_R_POISONED;
  if (mask || nap) {
    uint64_t m = 0;
    int np = 0;
    if ((rc = ec_gen_info(c, li, G, &m, nullptr, &np))) return rc;
    if (mask) *mask = m;
    if (nap) *nap = np;
  }
  return EC_OK;
}

int ec_set_pin(ec_comm_t* c, int li, uint64_t pin_lo, int ordered, void* stream) {
  int rc = check_li(c, li);
  if (rc) return rc;
  EcRankHost* r = c->L[li];
  if (ordered) {
    std::lock_guard<std::mutex> g(r->pin_mu);
    CK(cudaSetDevice(c->device));
    CK(launch_write_u64(&r->hd->pin_lo, pin_lo, (cudaStream_t)stream));
    if (!r->unpin_ev) CK(cudaEventCreateWithFlags(&r->unpin_ev, cudaEventDisableTiming));
    CK(cudaEventRecord(r->unpin_ev, (cudaStream_t)stream));
    r->unpin_pending = true;
  } else {
    std::lock_guard<std::mutex> g(r->pin_mu);
    __atomic_store_n(&r->h->pin_lo, (unsigned long long)pin_lo, __ATOMIC_SEQ_CST);
  }
  return EC_OK;
}

int ec_fold_raw(void* stash, const void* grad, int64_t n, int dtype, int mode, uint32_t* nonfinite,
                void* stream) {
  if (!stash || !grad || n < 0) return fail(EC_E_ARG, "bad fold arguments");
  if (dtype < EC_F32 || dtype > EC_I64) return fail(EC_E_ARG, "bad dtype");
  if (n == 0) return EC_OK;
  CK(launch_fold(dtype, stash, grad, n, mode, nonfinite, (cudaStream_t)stream, 0));
  return EC_OK;
}

int ec_sgd_update(void* w, const void* u, double lr, int64_t n, int dtype, void* stream) {
  if (!w || !u || n < 0) return fail(EC_E_ARG, "bad update arguments");
  if (dtype != EC_F32 && dtype != EC_F64) return fail(EC_E_ARG, "update needs a float dtype");
  if (n == 0) return EC_OK;
  CK(launch_update(dtype, w, u, lr, n, (cudaStream_t)stream));
  return EC_OK;
}

int ec_momentum_update(void* w, void* buf, const void* u, double lr, double mu, int64_t n, int dtype,
                       void* stream) {
  if (!w || !buf || !u || n < 0) return fail(EC_E_ARG, "bad momentum arguments");
  if (dtype != EC_F32 && dtype != EC_F64) return fail(EC_E_ARG, "momentum needs a float dtype");
  if (n == 0) return EC_OK;
  CK(launch_momentum(dtype, w, buf, u, lr, mu, n, (cudaStream_t)stream));
  return EC_OK;
}

int ec_local_reduce(const void* const* srcs, int p, uint64_t has, void* dst, int64_t n, int dtype,
                    int divide, void* stream) {
  if (!srcs || !dst || p < 1 || p > EC_MAX_P || n < 0) return fail(EC_E_ARG, "bad reduce arguments");
  if (dtype < EC_F32 || dtype > EC_I64) return fail(EC_E_ARG, "bad dtype");
  if (n == 0) return EC_OK;
  CK(launch_reduce(dtype, srcs, p, has, dst, n, divide, (cudaStream_t)stream));
  return EC_OK;
}

int ec_spin(uint64_t ns, void* stream) {
  CK(launch_spin(ns, (cudaStream_t)stream));
  return EC_OK;
}

/* Diagnostics: host-visible words, the engine stream's status and a copy of
 * the engine's private state (read on a side stream while the engine runs).
 * out[0..15]: done_gen1, req_done, error, error_info, exited, snap_gen1, stop,
 * pin_lo, stream_status, L.g, L.snapped, L.contrib, L.internal_act,
 * L.cmd_seq, L.round_done, L.next_req */
int ec_debug_state(ec_comm_t* c, int li, int64_t* out) {
  int rc = check_li(c, li);
  if (rc) return rc;
  EcRankHost* r = c->L[li];
  out[0] = aload(&r->h->done_gen1);
  out[1] = aload(&r->h->req_done);
  out[2] = aload(&r->h->error);
  out[3] = aload(&r->h->error_info);
  out[4] = aload(&r->h->exited);
  out[5] = aload(&r->h->snap_gen1);
  out[6] = aload(&r->h->stop);
  out[7] = aload(&r->h->pin_lo);
  out[8] = c->es ? (int64_t)cudaStreamQuery(c->es) : -1;
  EcLocal loc;
  cudaStream_t s;
  CK(cudaSetDevice(c->device));
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaError_t e = cudaMemcpyAsync(&loc, r->local, sizeof(loc), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (e != cudaSuccess) return fail(EC_E_CUDA, "debug copy: %s", cudaGetErrorString(e));
  out[9] = loc.g;
  out[10] = loc.snapped;
  out[11] = loc.contrib;
  out[12] = loc.internal_act;
  out[13] = (int64_t)loc.cmd_seq;
  out[14] = (int64_t)loc.round_done;
  out[15] = (int64_t)loc.next_req;
  return EC_OK;
}

int ec_step_times(ec_comm_t* c, int li, int64_t t, uint64_t* t3) {
  int rc = check_li(c, li);
  if (rc) return rc;
  if (t < 0 || !t3) return fail(EC_E_ARG, "bad step");
  EcRankHost* r = c->L[li];
  cudaStream_t s;
  CK(cudaSetDevice(c->device));
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaError_t e = cudaMemcpyAsync(t3, &r->local->tl[t & 63][0], 4 * sizeof(unsigned long long),
                                  cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (e != cudaSuccess) return fail(EC_E_CUDA, "step times copy: %s", cudaGetErrorString(e));
  return EC_OK;
}

// checked build: the controller's 16 iteration starts before it saw step t's
// offer (t one of the last 8); zeros in the production build
int ec_step_iterations(ec_comm_t* c, int li, int64_t t, uint64_t* t16) {
  // t16: 16 iteration starts, then 16 x 4 section stamps (80 words)
  int rc = check_li(c, li);
  if (rc) return rc;
  if (t < 0 || !t16) return fail(EC_E_ARG, "bad step");
  EcRankHost* r = c->L[li];
  cudaStream_t s;
  CK(cudaSetDevice(c->device));
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaError_t e = cudaMemcpyAsync(t16, &r->local->tl_it[t & 7][0], 16 * sizeof(unsigned long long),
                                  cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(t16 + 16, &r->local->tl_sec[t & 7][0][0], 64 * sizeof(unsigned long long),
                        cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (e != cudaSuccess) return fail(EC_E_CUDA, "iterations copy: %s", cudaGetErrorString(e));
  return EC_OK;
}

int ec_comm_traffic(ec_comm_t* c, int li, uint64_t* rx_bytes, uint64_t* tx_bytes) {
  int rc = check_li(c, li);
  if (rc) return rc;
  EcRankHost* r = c->L[li];
  unsigned long long v[2] = {0, 0};
  cudaStream_t s;
  CK(cudaSetDevice(c->device));
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaError_t e = cudaMemcpyAsync(v, &r->local->nv_rx, sizeof(v), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (e != cudaSuccess) return fail(EC_E_CUDA, "traffic copy: %s", cudaGetErrorString(e));
  if (rx_bytes) *rx_bytes = v[0];
  if (tx_bytes) *tx_bytes = v[1];
  return EC_OK;
}

int ec_comm_idle_stats(ec_comm_t* c, uint64_t* parks, uint64_t* wakes, int* parked) {
  if (!c) return fail(EC_E_ARG, "null communicator");
  std::lock_guard<std::recursive_mutex> lk(c->live_mu);
  if (parks) *parks = c->idle_parks;
  if (wakes) *wakes = c->idle_wakes;
  if (parked) *parked = c->parked_auto.load() ? 1 : 0;
  return EC_OK;
}

}  // extern "C"
