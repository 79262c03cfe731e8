// sm_100a kernels of the eager-SGD partial-collective path.
//
//   ec_engine<T>        persistent per-rank collective engine (controller CTA +
//                       worker CTAs): activation / snapshot protocol, two-shot
//                       peer-memory reduction in tree order, result publish.
//   ec_fold_kernel      GradientBuffer.fold          (eagersgd.py:55-57)
//   ec_update_kernel    w = w - lr*u                 (eagersgd.py:165)
//   ec_momentum_kernel  opt-in SGD momentum
//   ec_reduce_kernel    tree_order_sum of local vectors (collectives.py:385-403)
//   ec_post_kernel      stream-ordered request doorbell
//   ec_spin_kernel      device imbalance injection   (transport.py:137-149)
//
// All bulk traffic moves in 16-byte vectors; the engine reads peer and reused
// buffers with ld.global.cg so it never serves a stale L1 line.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "ec_common.cuh"
#include "ec_ops.cuh"

// ---------------------------------------------------------------------------
// engine: reduce-scatter (pull) of this rank's shard

template <typename T, int P, int U>
__device__ __forceinline__ void rs_fixed(const EcDesc& d, const char* const* sp,
                                         unsigned long long has, long long v0,
                                         long long v1, char* dst, long long start,
                                         long long stride, T inv, bool pow2) {
  constexpr int V = Ops<T>::V;
  const char* src[P];
#pragma unroll
  for (int q = 0; q < P; ++q) src[q] = sp[q];
  for (long long base = v0 + start; base < v1; base += stride * U) {
    Vec16<T> x[U][P];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long long v = base + (long long)u * stride;
#pragma unroll
      for (int q = 0; q < P; ++q) {
        if (v < v1 && ((has >> q) & 1ull))
          x[u][q].raw = ld_cg_v4(src[q] + v * 16);
        else
          x[u][q].raw = make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long long v = base + (long long)u * stride;
      if (v < v1) {
        Vec16<T> o;
#pragma unroll
        for (int l = 0; l < V; ++l) {
          T c[P];
#pragma unroll
          for (int q = 0; q < P; ++q) c[q] = Ops<T>::canon(x[u][q].e[l]);
          o.e[l] = Ops<T>::divp(tree_sum<T, P>(c), d.P, inv, pow2);
        }
        st_v4(dst + v * 16, o.raw);
      }
    }
  }
}

template <typename T>
__device__ void rs_dyn(const EcDesc& d, const char* const* sp, unsigned long long has, long long v0,
                       long long v1, char* dst, long long start, long long stride, T inv, bool pow2) {
  constexpr int V = Ops<T>::V;
  for (long long v = v0 + start; v < v1; v += stride) {
    Vec16<T> o;
#pragma unroll
    for (int l = 0; l < V; ++l) {
      auto leaf = [&](int q) -> T {
        if (!((has >> q) & 1ull)) return Ops<T>::zero();
        Vec16<T> x;
        x.raw = ld_cg_v4(sp[q] + v * 16);
        return Ops<T>::canon(x.e[l]);
      };
      o.e[l] = Ops<T>::divp(tree_sum_dyn<T>(d.P, leaf), d.P, inv, pow2);
    }
    st_v4(dst + v * 16, o.raw);
  }
}

template <typename T>
__device__ void rs_shard(const EcDesc& d, const char* const* sp, unsigned long long has,
                         long long v0, long long v1, char* dst, long long start, long long stride) {
  const bool pow2 = (d.P & (d.P - 1)) == 0;
  const T inv = (T)1 / (T)d.P;  // exact for powers of two
  switch (d.P) {
    case 1: rs_fixed<T, 1, 4>(d, sp, has, v0, v1, dst, start, stride, inv, pow2); break;
    case 2: rs_fixed<T, 2, 4>(d, sp, has, v0, v1, dst, start, stride, inv, pow2); break;
    case 3: rs_fixed<T, 3, 2>(d, sp, has, v0, v1, dst, start, stride, inv, pow2); break;
    case 4: rs_fixed<T, 4, 2>(d, sp, has, v0, v1, dst, start, stride, inv, pow2); break;
    case 5: rs_fixed<T, 5, 2>(d, sp, has, v0, v1, dst, start, stride, inv, pow2); break;
    case 6: rs_fixed<T, 6, 2>(d, sp, has, v0, v1, dst, start, stride, inv, pow2); break;
    case 7: rs_fixed<T, 7, 2>(d, sp, has, v0, v1, dst, start, stride, inv, pow2); break;
    case 8: rs_fixed<T, 8, 2>(d, sp, has, v0, v1, dst, start, stride, inv, pow2); break;
    default: rs_dyn<T>(d, sp, has, v0, v1, dst, start, stride, inv, pow2); break;
  }
}

// scalar tail (n % V elements) -- reduced by the last owner
template <typename T>
__device__ void rs_tail(const EcDesc& d, const char* const* sp, unsigned long long has, char* dst,
                        int lane) {
  const long long e0 = d.nvec * Ops<T>::V;
  const long long e = e0 + lane;
  if (e >= d.n) return;
  const bool pow2 = (d.P & (d.P - 1)) == 0;
  const T inv = (T)1 / (T)d.P;
  auto leaf = [&](int q) -> T {
    if (!((has >> q) & 1ull)) return Ops<T>::zero();
    const volatile T* s = reinterpret_cast<const volatile T*>(sp[q]);
    return Ops<T>::canon(s[e]);
  };
  reinterpret_cast<T*>(dst)[e] = Ops<T>::divp(tree_sum_dyn<T>(d.P, leaf), d.P, inv, pow2);
}

__device__ __forceinline__ long long shard_lo(long long nvec, int q, int P) {
  return (long long)(((unsigned long long)nvec * (unsigned long long)q) / (unsigned long long)P);
}

// ---------------------------------------------------------------------------
// TMA helpers (1-D bulk copies; peer addresses work through the UVA window)

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* b, unsigned parity) {
  unsigned ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
               " selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void tma_load(void* sdst, const void* gsrc, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_store(void* gdst, const void* ssrc, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               :: "l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void tma_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory");
}
// allow the n most recent store groups to still be reading shared memory
__device__ __forceinline__ void tma_wait_read_n(int n) {
  switch (n) {
    case 0: tma_wait_read<0>(); break;
    case 1: tma_wait_read<1>(); break;
    case 2: tma_wait_read<2>(); break;
    case 3: tma_wait_read<3>(); break;
    case 4: tma_wait_read<4>(); break;
    case 5: tma_wait_read<5>(); break;
    case 6: tma_wait_read<6>(); break;
    default: tma_wait_read<7>(); break;
  }
}
__device__ __forceinline__ void tma_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// TMA data phase geometry (host and device agree): chunks of `chv` 16-byte
// vectors, `stages` deep, P source slices + 1 output slice per stage.
__device__ __forceinline__ long long chunk_lo(long long nch, int q, int P) {
  return (long long)(((unsigned long long)nch * (unsigned long long)q) / (unsigned long long)P);
}

template <typename T, int P>
__device__ __forceinline__ bool reduce_chunk_smem(const char* src, char* out, int nvv, int chb,
                                                  unsigned long long has, int p, T inv, bool pow2) {
  constexpr int V = Ops<T>::V;
  bool bad = false;
  for (int i = threadIdx.x; i < nvv; i += blockDim.x) {
    Vec16<T> x[P];
#pragma unroll
    for (int q = 0; q < P; ++q)
      x[q].raw = ((has >> q) & 1ull) ? *reinterpret_cast<const uint4*>(src + (size_t)q * chb + i * 16)
                                     : make_uint4(0, 0, 0, 0);
    Vec16<T> o;
#pragma unroll
    for (int l = 0; l < V; ++l) {
      T c[P];
#pragma unroll
      for (int q = 0; q < P; ++q) c[q] = Ops<T>::canon(x[q].e[l]);
      o.e[l] = Ops<T>::divp(tree_sum<T, P>(c), p, inv, pow2);
      bad |= !Ops<T>::finite(o.e[l]);
    }
    *reinterpret_cast<uint4*>(out + i * 16) = o.raw;
  }
  return bad;
}

template <typename T>
__device__ bool reduce_chunk_smem_dyn(const char* src, char* out, int nvv, int chb,
                                      unsigned long long has, int p, T inv, bool pow2) {
  constexpr int V = Ops<T>::V;
  bool bad = false;
  for (int i = threadIdx.x; i < nvv; i += blockDim.x) {
    Vec16<T> o;
#pragma unroll
    for (int l = 0; l < V; ++l) {
      auto leaf = [&](int q) -> T {
        if (!((has >> q) & 1ull)) return Ops<T>::zero();
        Vec16<T> x;
        x.raw = *reinterpret_cast<const uint4*>(src + (size_t)q * chb + i * 16);
        return Ops<T>::canon(x.e[l]);
      };
      o.e[l] = Ops<T>::divp(tree_sum_dyn<T>(p, leaf), p, inv, pow2);
      bad |= !Ops<T>::finite(o.e[l]);
    }
    *reinterpret_cast<uint4*>(out + i * 16) = o.raw;
  }
  return bad;
}

// returns whether this thread produced a non-finite reduced value
template <typename T>
__device__ __forceinline__ bool reduce_chunk(const char* src, char* out, int nvv, int chb,
                                             unsigned long long has, int p) {
  const bool pow2 = (p & (p - 1)) == 0;
  const T inv = (T)1 / (T)p;
  switch (p) {
    case 1: return reduce_chunk_smem<T, 1>(src, out, nvv, chb, has, p, inv, pow2);
    case 2: return reduce_chunk_smem<T, 2>(src, out, nvv, chb, has, p, inv, pow2);
    case 3: return reduce_chunk_smem<T, 3>(src, out, nvv, chb, has, p, inv, pow2);
    case 4: return reduce_chunk_smem<T, 4>(src, out, nvv, chb, has, p, inv, pow2);
    case 5: return reduce_chunk_smem<T, 5>(src, out, nvv, chb, has, p, inv, pow2);
    case 6: return reduce_chunk_smem<T, 6>(src, out, nvv, chb, has, p, inv, pow2);
    case 7: return reduce_chunk_smem<T, 7>(src, out, nvv, chb, has, p, inv, pow2);
    case 8: return reduce_chunk_smem<T, 8>(src, out, nvv, chb, has, p, inv, pow2);
    default: return reduce_chunk_smem_dyn<T>(src, out, nvv, chb, has, p, inv, pow2);
  }
}

// One round of the fused TMA data phase for CTA w of this rank:
//   for each chunk of MY shard: bulk-load the chunk from every contributing
//   rank's send buffer (peer memory, NVLink) into shared memory, reduce it in
//   tree order, then bulk-store the result into EVERY rank's result slot
//   (reduce-scatter pull and all-gather push, pipelined per chunk).
// arrival words for fused updates: after the stores of this worker's first k
// chunks completed, tell every rank that applies an update this round
__device__ __forceinline__ void signal_chunks(const EcDesc& d, int w, long long g,
                                              unsigned long long updm, long long k) {
  fence_proxy_async_global();   // completed async-proxy stores -> generic release below
  fence_acq_rel_sys();
  const unsigned long long v = (((unsigned long long)g + 1) << EC_PROG_SHIFT) | (unsigned long long)k;
  for (unsigned long long m = updm; m; m &= m - 1) {
    const int q = __ffsll((long long)m) - 1;
    st_relaxed_sys(&d.ctrl[q]->prog[d.rank][w], v);
  }
}

//
// One-shot (mode 3, small messages): every rank's workers take ALL chunks,
// pull every contributing rank's slice and store the reduced chunk into the
// rank's OWN slot only -- no push to peers and no remote-store completion on
// the critical path.  The done word then means "my reads of everyone's
// buffers and my own slot are complete", which is what both the peers (their
// send buffers are free) and this rank (its result is in) wait for.
template <typename T>
__device__ void round_tma(const EcDesc& d, const char* const* sp, int w, long long g,
                          unsigned long long has, char* smem, unsigned long long* full,
                          unsigned long long& it, bool& bad, unsigned long long updm,
                          bool oneshot, int wact) {
  // wact: the worker CTAs this round uses (all W, or the step's count in a
  // round with progressive updates -- the update kernel maps chunks with it)
  const int P = d.P, r = d.rank, S = d.stages;
  const int chv = d.chv, chb = d.chv * 16;
  const long long nch = (d.nvec + chv - 1) / chv;
  const long long c0 = oneshot ? 0 : chunk_lo(nch, r, P), c1 = oneshot ? nch : chunk_lo(nch, r + 1, P);
  if (oneshot) updm = 0;
  EC_ASSERT(0 <= c0 && c0 <= c1 && c1 <= nch && g >= 0);
  const long long mine = (w < wact && c1 - c0 > w) ? (c1 - c0 - w + wact - 1) / wact : 0;
  const long long off = (g % d.R) * d.slot_bytes;
  const size_t stage_bytes = (size_t)(P + 1) * chb;
  const unsigned npop = (unsigned)__popcll(has);
  // arrival words for progressive updates: ~4 per worker per round by default.
  // Each costs a full-completion wait and proxy + sys fences on the issuing
  // thread (P=4, 100 MB step: data phase 248.7 us without, 253.9 with one
  // final word, 260.9 with one per 8 chunks, 266.2 per 4); fewer words leave
  // more of the update after the round (done->offer 46 us with one)
  const long long sig = d.sig_every > 0 ? d.sig_every : (mine + 3) / 4 > 1 ? (mine + 3) / 4 : 1;
  // sig_every < 0 (EC_SIGNAL_EVERY=-1): a geometric schedule instead -- words
  // after 1/2, 3/4, 7/8, ... of the worker's chunks, so what the update has
  // left once the round is over shrinks to about the last chunk
  const bool geo = d.sig_every < 0;
  auto signal_at = [&](long long done_chunks) -> bool {   // chunks < done_chunks landed
    if (!geo) return ((done_chunks) % sig) == 0;
    for (int j = 1; j <= 5; ++j)
      if (done_chunks == mine - (mine >> j) && (mine >> j) > 0) return true;
    return false;
  };
  // bytes this worker moves to / from OTHER ranks (the NVLink traffic it
  // issues; EcLocal::nv_rx / nv_tx, read by ec_comm_traffic)
  unsigned long long nv_rx = 0, nv_tx = 0;
  auto issue = [&](long long k) {  // thread 0: loads of my k-th chunk
    const int s = (int)((it + k) % S);
    const long long c = c0 + w + k * wact;
    const long long v0 = c * chv;
    const unsigned bytes = (unsigned)(min((long long)chv, d.nvec - v0) * 16);
    char* st = smem + s * stage_bytes;
    EC_ASSERT(c >= c0 && c < c1 && v0 < d.nvec && bytes > 0 && bytes <= (unsigned)chb);
    EC_ASSERT((size_t)(s + 1) * stage_bytes <= (size_t)d.smem_bytes);
    mbar_expect_tx(&full[s], npop * bytes);
    for (int q = 0; q < P; ++q)
      if ((has >> q) & 1ull) {
        tma_load(st + (size_t)q * chb, sp[q] + v0 * 16, bytes, &full[s]);
        if (q != r) nv_rx += bytes;
      }
  };
  if (threadIdx.x == 0) {
    fence_proxy_async_global();  // peers' generic writes (acquired via flags) -> async-proxy reads
    for (long long k = 0; k < mine && k < S; ++k) issue(k);
  }
  for (long long k = 0; k < mine; ++k) {
    const int s = (int)((it + k) % S);
    const unsigned parity = (unsigned)(((it + k) / S) & 1ull);
    const long long c = c0 + w + k * wact;
    const long long v0 = c * chv;
    const int nvv = (int)min((long long)chv, d.nvec - v0);
    char* st = smem + s * stage_bytes;
    char* out = st + (size_t)P * chb;
    // the out slice of stage s was last stored from S chunks ago; the S-1 newer
    // store groups may still be in flight
    if (threadIdx.x == 0) tma_wait_read_n(S - 1);
    while (!mbar_try_wait(&full[s], parity)) {
    }
    __syncthreads();
    bad |= reduce_chunk<T>(st, out, nvv, chb, has, P);
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      EC_ASSERT(off + (v0 + nvv) * 16 <= (long long)d.R * d.slot_bytes && nvv > 0);
      for (int j = 0; j < (oneshot ? 1 : P); ++j) {
        const int q = (r + j) % P;  // own slot first, then peers round-robin
        tma_store(d.ring[q] + off + v0 * 16, out, (unsigned)nvv * 16);
      }
      if (!oneshot) nv_tx += (unsigned long long)(P - 1) * nvv * 16;
      tma_commit();
      if (k + S < mine) issue(k + S);
      if (updm && k >= 2 && signal_at(k - 1)) {
        // all but the 2 newest store groups have fully landed: chunks < k - 1
        // (one signal per sig_every chunks: each costs a sys fence)
        asm volatile("cp.async.bulk.wait_group 2;" ::: "memory");
        signal_chunks(d, w, g, updm, k - 1);
      }
    }
  }
  it += (unsigned long long)mine;
  if (threadIdx.x == 0) {
    tma_wait_all();
    fence_proxy_async_global();
    if (updm) signal_chunks(d, w, g, updm, mine);
    if (nv_rx) atomicAdd(&d.local->nv_rx, nv_rx);
    if (nv_tx) atomicAdd(&d.local->nv_tx, nv_tx);
  }
}

// scalar tail (n % V elements): reduced by the last owner, pushed to every slot
template <typename T>
__device__ void tail_push(const EcDesc& d, const char* const* sp, unsigned long long has,
                          long long g, bool oneshot = false) {
  const long long e = d.nvec * Ops<T>::V + threadIdx.x;
  if (threadIdx.x >= Ops<T>::V || e >= d.n) return;
  const bool pow2 = (d.P & (d.P - 1)) == 0;
  const T inv = (T)1 / (T)d.P;
  auto leaf = [&](int q) -> T {
    if (!((has >> q) & 1ull)) return Ops<T>::zero();
    const volatile T* s = reinterpret_cast<const volatile T*>(sp[q]);
    return Ops<T>::canon(s[e]);
  };
  const T u = Ops<T>::divp(tree_sum_dyn<T>(d.P, leaf), d.P, inv, pow2);
  const long long off = (g % d.R) * d.slot_bytes;
  unsigned long long rx = 0;
  for (int q = 0; q < d.P; ++q) rx += (q != d.rank && ((has >> q) & 1ull)) ? sizeof(T) : 0;
  atomicAdd(&d.local->nv_rx, rx);
  if (oneshot) {
    reinterpret_cast<volatile T*>(d.ring[d.rank] + off)[e] = u;
    return;
  }
  for (int q = 0; q < d.P; ++q) reinterpret_cast<volatile T*>(d.ring[q] + off)[e] = u;
  atomicAdd(&d.local->nv_tx, (unsigned long long)(d.P - 1) * sizeof(T));
}

// Two-phase pull data path (ld.global.cg): reduce-scatter, then all-gather.
template <typename T>
__device__ void round_ldg(const EcDesc& d, const char* const* sp, int w, long long g,
                          unsigned long long has, unsigned long long seen) {
  EcLocal* L = d.local;
  EcCtrl* C = d.ctrl[d.rank];
  const int tid = threadIdx.x;
  const long long bt = blockDim.x;
  char* my_slot = d.ring[d.rank] + (g % d.R) * d.slot_bytes;
  const long long off = (g % d.R) * d.slot_bytes;
  {
    const long long v0 = shard_lo(d.nvec, d.rank, d.P), v1 = shard_lo(d.nvec, d.rank + 1, d.P);
    rs_shard<T>(d, sp, has, v0, v1, my_slot, (long long)w * bt + tid, (long long)d.W * bt);
    if (d.rank == d.P - 1 && w == 0 && tid < Ops<T>::V) rs_tail<T>(d, sp, has, my_slot, tid);
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    unsigned long long old = atomicAdd(&L->rs_count, 1ull);
    if (old + 1 == (unsigned long long)d.W * seen) {
      fence_acq_rel_sys();
      for (int q = 0; q < d.P; ++q) st_release_sys(&d.ctrl[q]->rsdone_from[d.rank], (unsigned long long)g + 1);
      L->t_rs4[(seen - 1) & 3] = globaltimer_ns();
    }
    const unsigned long long t0 = globaltimer_ns();
    for (int q = 0; q < d.P; ++q) {
      while (ld_acquire_sys(&C->rsdone_from[q]) < (unsigned long long)g + 1) {
        if (globaltimer_ns() - t0 > d.timeout_ns) {
          st_release_sys(&d.hctl->error_info, 0x100 + q);
          st_release_sys(&d.hctl->error, EC_DERR_TIMEOUT);
          break;
        }
      }
    }
  }
  __syncthreads();
  constexpr int U = 4;
  const long long start = (long long)w * bt + tid, stride = (long long)d.W * bt;
  for (int k = 1; k < d.P; ++k) {
    const int q = (d.rank + k) % d.P;
    const char* src = d.ring[q] + off;
    const long long v0 = shard_lo(d.nvec, q, d.P), v1 = shard_lo(d.nvec, q + 1, d.P);
    for (long long base = v0 + start; base < v1; base += stride * U) {
      uint4 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        long long v = base + (long long)u * stride;
        if (v < v1) x[u] = ld_cg_v4(src + v * 16);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        long long v = base + (long long)u * stride;
        if (v < v1) st_v4(my_slot + v * 16, x[u]);
      }
    }
  }
  if (d.rank != d.P - 1 && w == 0 && tid < Ops<T>::V) {
    const long long e = d.nvec * Ops<T>::V + tid;
    if (e < d.n) {
      const volatile T* s = reinterpret_cast<const volatile T*>(d.ring[d.P - 1] + off);
      reinterpret_cast<T*>(my_slot)[e] = s[e];
    }
  }
}

// ---------------------------------------------------------------------------
// NVLS data phase (reduction_mode "fast", fp32, one rank per GPU): the NVSwitch
// reduces.  Every rank stages its offer (or zeros) into its copy of a
// multicast-bound region; the owner of each shard reads the switch-reduced
// sum with multimem.ld_reduce and broadcasts u = sum / P into every rank's
// result slot with multimem.st.  Per GPU that moves S + S/P each way instead
// of the two-shot's 2(P-1)/P * S, at the price of the switch's (unspecified)
// summation order -- never the fixed-order mode.

__device__ __forceinline__ void fence_proxy_alias() { asm volatile("fence.proxy.alias;" ::: "memory"); }

__device__ __forceinline__ float4 mm_ld_reduce_v4(const void* p) {
  float4 r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void mm_st_v4(void* p, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ float mm_ld_reduce_f32(const void* p) {
  float r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void mm_st_f32(void* p, float v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" :: "l"(p), "f"(v) : "memory");
}

template <typename T>
__device__ void round_nvls(const EcDesc& d, const char* const* sp, int w, long long g,
                           unsigned long long has, unsigned long long seen, bool& bad) {
  EcLocal* L = d.local;
  EcCtrl* C = d.ctrl[d.rank];
  const int tid = threadIdx.x, P = d.P, r = d.rank;
  const long long bt = blockDim.x, start = (long long)w * bt + tid, stride = (long long)d.W * bt;
  // 1. stage my offer (or zeros for a null snapshot) into my copy of the region
  const bool mine = (has >> r) & 1ull;
  const char* src = sp[r];
  {
    long long v = start;
    if (mine) {
      for (; v + 3 * stride < d.nvec; v += 4 * stride) {
        uint4 x[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) x[k] = ld_stream_v4(src + (v + k * stride) * 16);
#pragma unroll
        for (int k = 0; k < 4; ++k) st_v4(d.uc_stage + (v + k * stride) * 16, x[k]);
      }
    }
    for (; v < d.nvec; v += stride)
      st_v4(d.uc_stage + v * 16, mine ? ld_stream_v4(src + v * 16) : make_uint4(0, 0, 0, 0));
  }
  if (w == 0 && tid < 4) {
    const long long e = d.nvec * 4 + tid;
    if (e < d.n) reinterpret_cast<float*>(d.uc_stage)[e] = mine ? reinterpret_cast<const float*>(src)[e] : 0.0f;
  }
  __syncthreads();
  if (tid == 0) {
    fence_proxy_alias();
    __threadfence();
    if (atomicAdd(&L->stage_count, 1ull) + 1 == (unsigned long long)d.W * seen) {
      fence_acq_rel_sys();
      for (int q = 0; q < P; ++q) st_relaxed_sys(&d.ctrl[q]->staged_from[r], (unsigned long long)g + 1);
    }
    // 2. every rank staged
    const unsigned long long t0 = globaltimer_ns();
    for (int q = 0; q < P; ++q) {
      while (ld_acquire_sys(&C->staged_from[q]) < (unsigned long long)g + 1) {
        if (globaltimer_ns() - t0 > d.timeout_ns) {
          st_release_sys(&d.hctl->error_info, 0x400 + q);
          st_release_sys(&d.hctl->error, EC_DERR_TIMEOUT);
          break;
        }
      }
    }
    fence_proxy_alias();
    if (w == 0) L->t_rs4[(seen - 1) & 3] = globaltimer_ns();   // staged everywhere (timeline stamp)
  }
  __syncthreads();
  // 3. my shard: switch-reduced sum, / P, broadcast into every rank's slot
  const bool pow2 = (P & (P - 1)) == 0;
  const float inv = 1.0f / (float)P;
  const long long off = (g % d.R) * d.slot_bytes;
  const long long v0 = shard_lo(d.nvec, r, P), v1 = shard_lo(d.nvec, r + 1, P);
  // NVLS_U switch reductions in flight per thread before their broadcasts:
  // the switch round trip is long, so memory-level parallelism sets the rate
  constexpr int NVLS_U = 8;
  long long v = v0 + start;
  for (; v + (NVLS_U - 1) * stride < v1; v += NVLS_U * stride) {
    float4 s[NVLS_U];
#pragma unroll
    for (int k = 0; k < NVLS_U; ++k) s[k] = mm_ld_reduce_v4(d.mc_stage + (v + k * stride) * 16);
#pragma unroll
    for (int k = 0; k < NVLS_U; ++k) {
      float4 u;
      u.x = Ops<float>::divp(s[k].x, P, inv, pow2);
      u.y = Ops<float>::divp(s[k].y, P, inv, pow2);
      u.z = Ops<float>::divp(s[k].z, P, inv, pow2);
      u.w = Ops<float>::divp(s[k].w, P, inv, pow2);
      bad |= !(isfinite(u.x) && isfinite(u.y) && isfinite(u.z) && isfinite(u.w));
      mm_st_v4(d.mc_ring + off + (v + k * stride) * 16, u);
    }
  }
  for (; v < v1; v += stride) {
    float4 s = mm_ld_reduce_v4(d.mc_stage + v * 16);
    float4 u;
    u.x = Ops<float>::divp(s.x, P, inv, pow2);
    u.y = Ops<float>::divp(s.y, P, inv, pow2);
    u.z = Ops<float>::divp(s.z, P, inv, pow2);
    u.w = Ops<float>::divp(s.w, P, inv, pow2);
    bad |= !(isfinite(u.x) && isfinite(u.y) && isfinite(u.z) && isfinite(u.w));
    mm_st_v4(d.mc_ring + off + v * 16, u);
  }
  if (r == P - 1 && w == 0 && tid < 4) {
    const long long e = d.nvec * 4 + tid;
    if (e < d.n) {
      const float u = Ops<float>::divp(mm_ld_reduce_f32(d.mc_stage + e * 4), P, inv, pow2);
      bad |= !isfinite(u);
      mm_st_f32(d.mc_ring + off + e * 4, u);
    }
  }
  fence_proxy_alias();
}

template <typename T>
__device__ void engine_worker(const EcDesc& d, int w, unsigned long long epoch) {
  EcLocal* L = d.local;
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) unsigned long long full[8];
  __shared__ unsigned long long s_seq, s_has, s_src, s_updm;
  __shared__ int s_wact;
  __shared__ long long s_gen;
  __shared__ int s_exit;
  __shared__ const char* sp[EC_MAX_P];
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_seq = ld_acquire_gpu(&L->cmd_seq);
    for (int s = 0; s < d.stages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned long long seen = s_seq;
  unsigned long long it = 0;  // chunks this CTA has pipelined (stage / parity)
  __syncthreads();
  while (true) {
    if (tid == 0) {
      unsigned ns = 32;
      while (true) {
        // commands are taken one at a time, in order (up to `lead` may be out)
        unsigned long long s = ld_acquire_gpu(&L->cmd_seq);
        if (s > seen) {
          const EcCmd* cm = &L->cmd[seen & 3];
          EC_ASSERT(s - seen <= 2);     // at most lead (<= 2) commands out
          s_seq = seen + 1;
          s_gen = *(volatile const long long*)&cm->gen;
          s_has = *(volatile const unsigned long long*)&cm->has;
          s_updm = *(volatile const unsigned long long*)&cm->updm;
          s_src = *(volatile const unsigned long long*)&cm->src;
          s_wact = *(volatile const int*)&cm->wact;
          s_exit = 0;
          break;
        }
        if (ld_acquire_gpu(&L->exit_epoch) == epoch) {
          s_exit = 1;
          break;
        }
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
      }
    }
    __syncthreads();
    if (s_exit) return;
    seen = s_seq;
    const long long g = s_gen;
    const unsigned long long has = s_has;
    // this round's source per rank: its stash, or its registered gradient buffer
    for (int q = tid; q < d.P; q += blockDim.x) sp[q] = ((s_src >> q) & 1ull) ? d.gbuf[q] : d.send[q];
    __syncthreads();
    bool bad = false;
    if (d.mode == 0 || d.mode == 3) {
      const bool oneshot = d.mode == 3;
      round_tma<T>(d, sp, w, g, has, smem, full, it, bad, s_updm, oneshot, s_wact);
      // the scalar tail: reduced by the last owner and pushed to every slot,
      // or (one-shot) by every rank into its own slot
      if (w == 0 && (oneshot || d.rank == d.P - 1)) tail_push<T>(d, sp, has, g, oneshot);
    } else if (d.mode == 2) {
      round_nvls<T>(d, sp, w, g, has, seen, bad);
    } else {
      round_ldg<T>(d, sp, w, g, has, seen);
    }
    const int cs = (int)((seen - 1) & 3);     // this command's counter slot
    if (__syncthreads_or(bad) && tid == 0) atomicOr(&L->rpoison[cs], 1u);
    if (tid == 0) {
      fence_acq_rel_sys();
      const unsigned long long old = atomicAdd(&L->ag_cnt[cs], 1ull);
      if (old + 1 == (unsigned long long)d.W * (((seen - 1) >> 2) + 1)) {
        // every CTA of this rank is done: tell the world (TMA mode: our pushes
        // into every slot have landed) / ourselves (pull mode)
        fence_acq_rel_sys();
        unsigned long long word = (unsigned long long)g + 1;
        if (atomicExch(&L->rpoison[cs], 0u)) word |= EC_DONE_POISON;
        if (d.mode != 1) {
          if (d.mode == 0 || d.mode == 3) L->t_rs4[cs] = globaltimer_ns();
          for (int q = 0; q < d.P; ++q) st_relaxed_sys(&d.ctrl[q]->done_from[d.rank], word);
        } else {
          st_release_sys(&d.ctrl[d.rank]->done_from[d.rank], word);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// engine: controller (one thread per rank)

__device__ __forceinline__ unsigned int ld_relaxed_sys_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Peer-written control words, polled as a pre-check: relaxed loads of a group
// of eight are all in flight at once (an acquire load blocks the next one, and
// each costs an L2 round trip, 0.2-0.4 us under a data phase), folded to the
// min / max of f(word).  The words are monotone, so a passing pre-check stays
// passing; the caller re-reads with acquire where the word orders data.
template <bool kMax, typename F>
__device__ __forceinline__ unsigned long long poll_fold(const unsigned long long* w, int P, F f) {
  unsigned long long acc = kMax ? 0ull : ~0ull;
  for (int q0 = 0; q0 < P; q0 += 8) {
    unsigned long long v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = q0 + i < P ? ld_relaxed_sys(w + q0 + i) : (kMax ? 0ull : ~0ull);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const unsigned long long x = q0 + i < P ? f(v[i]) : (kMax ? 0ull : ~0ull);
      acc = kMax ? (x > acc ? x : acc) : (x < acc ? x : acc);
    }
  }
  return acc;
}

// The host poller's mirror for the controller: both threads are in one CTA, so
// the words the controller reads every iteration live in shared memory
// (device-memory copies in EcLocal persist them across relaunches).
struct EcHpShared {
  unsigned long long seq;    // EcLocal::hp_seq
  unsigned long long lo;     // EcLocal::hp_lo
  unsigned long long ps;     // EcLocal::hp_ps
  unsigned long long stop;   // 0 none, 1 explicit pause, 2 idle park (this launch)
};

// The controller runs the protocol of one "open" generation go (requests,
// activation, snapshot, command) while up to two rounds are in flight: once
// round g's command is out, the open generation is g + 1, so a rank whose next
// offer is already queued (back-to-back rounds, the nccl-tests pattern) snapshots
// g + 1 and exchanges its snapshot words DURING round g's data phase, and the
// workers find g + 1's command waiting when they finish g (EcDesc::lead == 2,
// fused TMA mode with R >= 3 result slots).  Round g is published when every
// owner's done word for g is in; rounds publish in order.
__device__ void engine_controller(const EcDesc& d, unsigned long long epoch, volatile EcHpShared* hp) {
  EcLocal* L = d.local;
  EcHostCtl* H = d.hctl;
  EcCtrl* C = d.ctrl[d.rank];
  const int r = d.rank, P = d.P;
  long long g = L->g, hold_from = L->hold_from, contributed_round = L->contributed_round;
  long long guard_tau = L->guard_tau, pend_lo = L->pend_lo, last_off = L->last_off;
  unsigned long long next_req = L->next_req;
  int snapped = L->snapped, contrib = L->contrib, internal_act = L->internal_act;
  int arrive_pending = L->arrive_pending, arrive_activate = L->arrive_activate;
  unsigned long long seq = L->cmd_seq;
  bool stopping = false, idle_stop = false;
  bool voted = false, park_now = false;
  unsigned long long stop_t0 = 0;
  unsigned long long t_snap = L->t_snap;
  unsigned long long t_req = 0;
  unsigned ns = 32;
  // rounds whose command is out (0, 1 or d.lead), oldest = g; the open
  // generation is go = g + n_issued.  Log data of an issued round, by gen & 1.
  int n_issued = 0;
  long long go = g;
  unsigned long long iss_fresh[2], iss_has[2], iss_tsnap[2], iss_tcmd[2], iss_treq[2], iss_seq[2];
  // Host-visible words (replies, the log, done_gen1) cost a PCIe drain at the
  // next sys fence, so they are written after the NVLink-facing work of the
  // iteration (the next snapshot's push) and published behind ONE fence:
  // replies of processed requests are buffered (status by seq & 15) ...
  unsigned char rep_st[16];
  unsigned long long rep_from = next_req;
  // ... and a completed round's log entry waits as the pending publication
  int pub_pending = 0;
  long long pub_gen = 0;
  unsigned long long pub_fresh = 0, pub_has = 0, pub_tsnap = 0, pub_tcmd = 0, pub_trs = 0,
                     pub_tdone = 0, pub_treq = 0, pub_poison = 0;
  auto flush_replies = [&]() {
    if (rep_from == next_req) return;
    for (unsigned long long q = rep_from; q < next_req; ++q)
      st_relaxed_sys(&H->reply[q % EC_REQ_RING], ((q + 1) << 8) | rep_st[q & 15]);
    st_relaxed_sys(&H->req_done, next_req);
    rep_from = next_req;
  };
  auto publish_host = [&]() {
    flush_replies();
    if (!pub_pending) return;
    EcLog* lg = &H->log[pub_gen % EC_LOG_RING];
    st_relaxed_sys(&lg->mask, pub_fresh);
    st_relaxed_sys(&lg->has, pub_has);
    st_relaxed_sys(&lg->nap, (unsigned long long)__popcll(pub_fresh));
    st_relaxed_sys(&lg->t_snap, pub_tsnap);
    st_relaxed_sys(&lg->t_cmd, pub_tcmd);
    st_relaxed_sys(&lg->t_rs, pub_trs);
    st_relaxed_sys(&lg->t_done, pub_tdone);
    st_relaxed_sys(&lg->t_req, pub_treq);
    st_relaxed_sys(&lg->poison, pub_poison);
    // the entry's own generation tag is record data (ring-overwrite check):
    // it must be visible before done_gen1, so it goes before the fence
    st_relaxed_sys(&lg->gen1, (unsigned long long)pub_gen + 1);
    fence_acq_rel_sys();                     // log entry (and replies) before done_gen1
    st_relaxed_sys(&H->done_gen1, (unsigned long long)pub_gen + 1);
    pub_pending = 0;
  };

  // write this rank's word into every rank's control block (peer stores over NVLink)
  // (one sys-scope fence, then relaxed stores: a fence-based release; every
  // sys fence on this serial path costs a PCIe/NVLink drain)
  auto push_all = [&](int which, unsigned long long v) {
    fence_acq_rel_sys();
    for (int q = 0; q < P; ++q) {
      unsigned long long* base;
      if (which == 0) base = &d.ctrl[q]->act_from[r];
      else if (which == 1) base = &d.ctrl[q]->snap_from[r];
      else base = &d.ctrl[q]->arrive_from[r];
      st_relaxed_sys(base, v);
    }
  };
  auto activate = [&]() {
    internal_act = 1;
    if (d.flavor != 0 && !d.replay) push_all(0, (unsigned long long)go + 1);
  };
  // majority with a quorum (EcDesc::quorum > 0, the north_star's phrasing):
  // the designated initiator activates only once at least `quorum` ranks have
  // boarded this generation (every boarding rank pushes an arrival word)
  const bool quorum_mode = d.flavor == 2 && d.quorum > 0 && !d.replay;
  auto initiator_activate = [&]() {
    if (quorum_mode) {
      arrive_pending = d.quorum;      // arrivals needed before activating
      arrive_activate = 1;
    } else {
      activate();
    }
  };
  auto forced_bit = [&](long long gen) -> int {
    if (gen >= d.n_forced) return -1;
    return (int)((d.forced[gen] >> r) & 1ull);
  };

  // host pin, mirrored into device memory by the host poller (engine thread
  // 32) and acknowledged HERE after this thread read it, so every later
  // snapshot check sees it (ec_wait's pin waits for the ack)
  unsigned long long host_pin = ld_relaxed_sys(&H->pin_lo);
  unsigned long long last_hs = hp->seq;
#ifdef EC_DEBUG
  unsigned long long it_ring[16];
  unsigned long long sec_ring[16][4];
  unsigned it_n = 0;
#define EC_SEC(k) sec_ring[(it_n - 1) & 15][k] = globaltimer_ns()
#else
#define EC_SEC(k)
#endif
  while (true) {
    bool progress = false;
#ifdef EC_DEBUG
    it_ring[it_n++ & 15] = globaltimer_ns();
#endif
    // the open generation takes protocol steps only while fewer than `lead`
    // rounds are in flight
    const bool open_ok = n_issued < d.lead;
    // Host-mapped words cost a PCIe round trip; the poller mirrors them (and
    // copies host-posted requests into the device ring), so this thread only
    // reads device memory.
    {
      const unsigned long long hs = hp->seq;
      if (hs != last_hs) {
        __threadfence_block();   // acquire (CTA scope): the poller's lo / ps before seq
        // A host reader re-checks done_gen1 after our ack (ec_wait): every
        // completed round must be host-visible before the ack, or a deferred
        // publication would let it pin a slot an early snapshot already took
        publish_host();
        host_pin = hp->lo;
        // release: orders the pin read before the ack
        st_release_sys(&H->pin_ack, hp->ps);
        last_hs = hs;
      }
      // stop requests: an explicit pause drains the open generation (a held
      // one is let go); an idle park (host watchdog, ec_host.cu) exits only
      // while nothing is in flight, and may be withdrawn
      const unsigned long long sk = hp->stop;
      const bool st_now = sk != 0;
      if (st_now && !stopping) stop_t0 = globaltimer_ns();
      stopping = st_now;
      idle_stop = sk == 2;
      if (!idle_stop && voted) {
        // withdrawn: take the vote back -- unless every controller had voted,
        // in which case the park is committed (the others may be gone)
        unsigned long long v = ld_acquire_gpu(d.park_votes);
        while (v < (unsigned long long)d.n_local) {
          const unsigned long long o = atomicCAS(d.park_votes, v, v - 1);
          if (o == v) break;
          v = o;
        }
        if (v >= (unsigned long long)d.n_local) park_now = true;
        else voted = false;
      }
    }
    EC_SEC(0);
    // ---- requests, strictly in sequence order: stream-posted ones sit in the
    // device ring (cheap), host-posted ones only in the host-mapped ring
    while (open_ok) {
      EcReq* dq = &L->dreq[next_req % EC_REQ_RING];
      unsigned type, fl;
      long long t, arg;
      bool dev_req = false;
      // stream-posted requests and (copied by the poller) host-posted ones;
      // the acquire load only once the relaxed one saw the request
      if (*(volatile unsigned long long*)&dq->seq1 != next_req + 1) break;
      if (ld_acquire_gpu(&dq->seq1) != next_req + 1) break;
      type = *(volatile unsigned*)&dq->type;
      fl = *(volatile unsigned*)&dq->flags;
      t = *(volatile long long*)&dq->t;
      arg = *(volatile long long*)&dq->arg;
      dev_req = !(fl & EC_CF_HOSTPOSTED);
      fl &= ~EC_CF_HOSTPOSTED;
      if (type == EC_REQ_CONTRIB && (fl & EC_CF_STEP) && t >= 0) {
        L->tl[t & 63][3] = globaltimer_ns();
#ifdef EC_DEBUG
        for (int i = 0; i < 16; ++i) {
          L->tl_it[t & 7][i] = it_ring[(it_n + i) & 15];
          for (int k = 0; k < 4; ++k) L->tl_sec[t & 7][i][k] = sec_ring[(it_n + i) & 15][k];
        }
#endif
      }
      unsigned long long status = 3;  // OK
      // while a round is in flight the open generation only moves on this
      // rank's own boarding (its offer for go, or an activation of go); any
      // other request waits for the round to publish, as the generation
      // ordering of the reference's engine has it (SPEC.md concurrency model)
      if (n_issued > 0 && !((type == EC_REQ_CONTRIB || type == EC_REQ_ACTIVATE) && t == go &&
                            !(fl & EC_CF_POISON)))
        break;
      // An offer for the generation after the open one while this rank has
      // already done its part for go (contributed or snapshotted): keep it at
      // the head of the queue until go's command is out, then take it at once
      // -- back-to-back rounds posted without host waits pay no post latency
      // between them.  (The application API never posts early; a buffer
      // re-offered early must not change while round go still reads it.)
      if (type == EC_REQ_CONTRIB && !(fl & EC_CF_POISON) && t == go + 1 &&
          (snapped || contributed_round == go))
        break;
      if (type == EC_REQ_CONTRIB && !(fl & EC_CF_POISON) && t <= go) {
        // guard ages: the offered stash now holds round t's gradient until a
        // fresh snapshot delivers it (eagersgd.py:117-124)
        if (t < pend_lo) pend_lo = t;
        if (t > last_off) last_off = t;
      }
      if (type == EC_REQ_CONTRIB) {
        if (fl & EC_CF_POISON) {
          status = 4;
        } else if (t < go || (t == go && snapped)) {
          status = 2;  // the round already consumed this rank's slot
          if (fl & EC_CF_SRC_GRAD) *(volatile int*)&L->late_copy = 1;  // keep the gradient
        } else if (t > go) {
          status = 5;
          st_release_sys(&H->error_info, (unsigned long long)t);   // info before the code
          st_release_sys(&H->error, EC_DERR_ORDER);
        } else if (d.replay && forced_bit(go) != 1) {
          status = 2;
          if (fl & EC_CF_SRC_GRAD) *(volatile int*)&L->late_copy = 1;
        } else {
          contrib = (int)(EC_SNAP_DATA | ((fl & 1u) ? EC_SNAP_FRESH : 0ull) |
                          ((fl & EC_CF_SRC_GRAD) ? EC_SNAP_SRC_GRAD : 0ull));
          if ((fl & EC_CF_STEP) && dev_req && d.mode == 0 && d.w_step <= EC_PROG_W) {
            // the step's update kernel (already resident behind the offer)
            // consumes round go's chunks as they land: owners publish arrival
            // words to us; pin slot go on its behalf now (it unpins when
            // done), before round go can even start
            *(volatile unsigned long long*)&L->pin_dev = (unsigned long long)go;
            L->fuse_seq = next_req + 1;
            contrib |= (int)EC_SNAP_UPD;
          }
          contributed_round = t;
          status = 1;
          t_req = globaltimer_ns();
          if ((fl & 4u) && !d.replay && ((fl & 2u) || d.flavor == 2)) {
            // all-arrive: every rank boards, so every rank's snapshot is its
            // own fresh offer whatever activates the round (solo/sync: its own
            // activation; majority: the designated initiator, which activates
            // only after everyone arrived) -- each snapshots at once and the
            // round starts when every snapshot is in (nap = P), without the
            // arrival barrier and activation exchanges
            internal_act = 1;
          } else if (fl & 4u) {  // all-arrive in replay mode: arrival barrier
            push_all(2, (unsigned long long)go + 1);
            arrive_pending = P;
            arrive_activate = (fl & 2u) ? 1 : 0;
          } else {
            if (quorum_mode) push_all(2, (unsigned long long)go + 1);   // counted by the initiator
            if (fl & 2u) initiator_activate();
          }
        }
      } else if (type == EC_REQ_ACTIVATE) {
        if (t == go) {
          if (quorum_mode && contributed_round == go) initiator_activate();
          else activate();
        }
      } else if (type == EC_REQ_HOLD) {
        hold_from = arg;
      } else if (type == EC_REQ_GUARD) {
        guard_tau = arg < 0 ? EC_INF_GEN : arg;
        if (t >= 0 && t < pend_lo) pend_lo = t;
      }
      EC_ASSERT(next_req - rep_from < 16);
      rep_st[next_req & 15] = (unsigned char)status;
      ++next_req;
      st_release_gpu(&L->req_done_dev, next_req);
      if (next_req - rep_from >= 16) flush_replies();
      progress = true;
    }
    EC_SEC(1);
    // ---- arrival barrier: `arrive_pending` ranks boarded (all of them in
    // all-arrive replay mode, the quorum in majority-quorum mode) -> activate
    if (open_ok && arrive_pending) {
      int n_arr = 0;
      for (int q = 0; q < P; ++q)
        n_arr += ld_acquire_sys(&C->arrive_from[q]) >= (unsigned long long)go + 1;
      if (n_arr >= arrive_pending) {
        arrive_pending = 0;
        if (arrive_activate) activate();
        progress = true;
      }
    }
    // ---- snapshot decision (collectives.py:146-153, schedule.py:452-455);
    // with a round in flight only once this rank boarded go itself
    if (open_ok && !snapped && (n_issued == 0 || contributed_round == go)) {
      bool sgo = false;
      if (d.replay) {
        int b = forced_bit(go);
        if (b == 0) sgo = true;
        else if (b == 1) sgo = contrib != 0;
      } else if (internal_act) {
        sgo = true;
      } else if (d.flavor != 0) {
        // an activation carries no data (the snapshot push fences what follows)
        const bool ext = poll_fold<true>(C->act_from, P, [](unsigned long long w) { return w; }) >=
                         (unsigned long long)go + 1;
        if (ext) {
          // staleness guard: an explicit threshold (ec_post_hold) or the
          // device-tracked ages (ec_post_guard), eagersgd.py:102-108
          const long long lo = pend_lo < last_off + 1 ? pend_lo : last_off + 1;
          const bool aged = guard_tau != EC_INF_GEN && go >= lo + guard_tau;
          const bool held = !(stopping && !idle_stop) && contributed_round < go &&
                            (go >= hold_from || aged);
          sgo = !held;
        }
      }
      if (sgo && go >= d.R) {
        // Result-slot reuse guard: peers write our slot go % R once the round
        // starts, so never snapshot go while a reader still needs generation
        // go - R.  Device readers pin in device memory (SC fence pairs with
        // wait_and_pin); the host pin is the acknowledged cached value; our
        // own updater CTAs finish a fused update before upd_fin_gen moves.
        fence_sc_gpu();
        const unsigned long long gr = (unsigned long long)(go - d.R);
        if (ld_acquire_gpu(&L->pin_dev) <= gr || host_pin <= gr) sgo = false;
      }
      if (sgo) {
        push_all(1, (((unsigned long long)go + 1) << EC_SNAP_SHIFT) | (unsigned long long)contrib);
        t_snap = globaltimer_ns();
        st_relaxed_sys(&H->snap_gen1, (unsigned long long)go + 1);
        if (contrib & (int)EC_SNAP_FRESH) {
          hold_from = EC_INF_GEN;  // stash delivered (eagersgd.py:117-124)
          pend_lo = EC_INF_GEN;
          *(volatile int*)&L->stash_null = 1;
        }
        snapped = 1;
        progress = true;
      }
    }
    // ---- round go: all snapshots in -> command to the workers (two-shot
    // reduction in the fused TMA pipeline)
    if (open_ok && snapped &&
        poll_fold<false>(C->snap_from, P, [](unsigned long long w) { return w >> EC_SNAP_SHIFT; }) >=
            (unsigned long long)go + 1) {
      bool all = true;
      unsigned long long fresh = 0, has = 0, srcg = 0, updm = 0;
      for (int q = 0; q < P; ++q) {
        unsigned long long w = ld_acquire_sys(&C->snap_from[q]);
        if ((w >> EC_SNAP_SHIFT) < (unsigned long long)go + 1) { all = false; break; }
        fresh |= (w & EC_SNAP_FRESH) << q;
        has |= ((w >> 1) & 1ull) << q;
        srcg |= ((w >> 2) & 1ull) << q;
        updm |= ((w >> 3) & 1ull) << q;
      }
      if (all) {
        EcCmd* cm = &L->cmd[seq & 3];   // the command of sequence number seq + 1
        EC_ASSERT(n_issued < d.lead && go == g + n_issued);
        cm->gen = go;
        cm->has = has;
        cm->src = srcg;
        cm->updm = updm;
        // rounds with progressive updates use the step's worker count (every
        // rank derives the same from the same snapshot words)
        cm->wact = (updm && d.w_step < d.W) ? d.w_step : d.W;
        ++seq;
        const int k = (int)(go & 1);
        iss_fresh[k] = fresh;
        iss_has[k] = has;
        iss_tsnap[k] = t_snap;
        iss_treq[k] = t_req;
        iss_seq[k] = seq;
        iss_tcmd[k] = globaltimer_ns();
        st_release_gpu(&L->cmd_seq, seq);
        ++n_issued;
        ++go;
        snapped = 0;
        contrib = 0;
        internal_act = 0;
        arrive_pending = 0;
        arrive_activate = 0;
        t_req = 0;
        progress = true;
        continue;   // the next generation may already be decidable
      }
    }
    EC_SEC(2);
    // host-visible words of this iteration's work (after any snapshot push)
    publish_host();
    EC_SEC(3);
    // ---- the oldest round in flight: complete at this rank once every owner's
    // data for g is in our slot (TMA mode) / our own all-gather is done (pull)
    if (n_issued > 0) {
      const int k = (int)(g & 1);
      const int q_lo = d.mode != 1 ? 0 : r, q_n = d.mode != 1 ? P : 1;
      bool all = poll_fold<false>(C->done_from + q_lo, q_n, [](unsigned long long w) {
                   return w & ~EC_DONE_POISON;
                 }) >= (unsigned long long)g + 1;
      unsigned long long poison = 0;
      for (int q = q_lo; q < q_lo + q_n && all; ++q) {
        const unsigned long long wq = ld_acquire_sys(&C->done_from[q]);
        if ((wq & ~EC_DONE_POISON) < (unsigned long long)g + 1) all = false;
        else if ((wq & ~EC_DONE_POISON) == (unsigned long long)g + 1) poison |= wq & EC_DONE_POISON;
      }
      if (!all) {
        if (globaltimer_ns() - iss_tcmd[k] > d.timeout_ns) {
          st_release_sys(&H->error_info, (unsigned long long)g);
          st_release_sys(&H->error, EC_DERR_TIMEOUT);
          break;   // watchdog: park with the round abandoned (error word set)
        }
      } else {
        const unsigned long long t_done = globaltimer_ns();
        EC_ASSERT(L->cmd[(iss_seq[k] - 1) & 3].gen == g);   // rounds complete in order
        publish_host();                          // at most one publication waits
        pub_gen = g;
        pub_fresh = iss_fresh[k];
        pub_has = iss_has[k];
        pub_tsnap = iss_tsnap[k];
        pub_tcmd = iss_tcmd[k];
        pub_trs = *(volatile unsigned long long*)&L->t_rs4[(iss_seq[k] - 1) & 3];
        pub_tdone = t_done;
        pub_treq = iss_treq[k];
        pub_poison = poison ? 1ull : 0ull;
        pub_pending = 1;
        // device waiters (the async step's update) see it at once; the host
        // after the next snapshot push (publish_host)
        st_release_gpu(&L->done_gen1_dev, (unsigned long long)g + 1);
        ++g;
        --n_issued;
        progress = true;
        continue;
      }
    }
    if (park_now) break;
    if (stopping) {
      const bool idle = n_issued == 0 && !snapped && !arrive_pending;
      if (idle_stop) {
        // every controller of the launch must agree (they exit together and the
        // host relaunches them together): vote while idle, leave when all have
        if (idle && !voted) {
          atomicAdd(d.park_votes, 1ull);
          voted = true;
        }
        if (voted && ld_acquire_gpu(d.park_votes) >= (unsigned long long)d.n_local) break;
      } else if (idle || (n_issued == 0 && globaltimer_ns() - stop_t0 > 2000000000ull)) {
        break;
      }
    }
    if (progress) {
      ns = 32;
    } else {
      __nanosleep(ns);
      // a round in flight: poll its done words at a short interval
      if (ns < (n_issued ? 128u : d.idle_sleep_ns)) ns <<= 1;
    }
  }
  publish_host();
  // park: persist the protocol state, release the workers, acknowledge.  A
  // parked engine has no round in flight (a watchdog timeout parks with the
  // round abandoned; its error word is set).
  L->g = g;
  L->hold_from = hold_from;
  L->contributed_round = contributed_round;
  L->next_req = next_req;
  L->snapped = snapped;
  L->contrib = contrib;
  L->internal_act = internal_act;
  L->arrive_pending = arrive_pending;
  L->arrive_activate = arrive_activate;
  L->t_snap = t_snap;
  L->guard_tau = guard_tau;
  L->pend_lo = pend_lo;
  L->last_off = last_off;
  __threadfence();
  st_release_gpu(&L->exit_epoch, epoch);
  st_release_sys(&H->exited, epoch);
}

// engine: host poller (thread 32 of the controller's CTA).  Mirrors the host
// pin and stop words into EcLocal and copies host-posted requests into the
// device request ring in sequence order (stream-posted sequence numbers are
// skipped once their kernel posted them), so the controller thread never
// stalls on a PCIe read.  Runs until the controller parks.
__device__ void engine_host_poller(const EcDesc& d, unsigned long long epoch, volatile EcHpShared* hp) {
  EcLocal* L = d.local;
  EcHostCtl* H = d.hctl;
  unsigned long long pn = *(volatile unsigned long long*)&L->next_req;   // parked cursor
  unsigned long long last_ps = ~0ull, last_lo = ~0ull, changes = *(volatile unsigned long long*)&L->hp_seq;
  while (ld_acquire_gpu(&L->exit_epoch) != epoch) {
    // the pin moves either through the acknowledged host handshake (pin_seq)
    // or through a stream-ordered kernel store (ec_set_pin ordered): mirror
    // both, the latter without an acknowledgement
    const unsigned long long ps = ld_acquire_sys(&H->pin_seq);
    const unsigned long long lo = ld_relaxed_sys(&H->pin_lo);
    if (ps != last_ps || lo != last_lo) {
      st_relaxed_gpu(&L->hp_lo, lo);
      st_relaxed_gpu(&L->hp_ps, ps);
      st_release_gpu(&L->hp_seq, ++changes);
      hp->lo = lo;
      hp->ps = ps;
      __threadfence_block();   // release (CTA scope): lo / ps before seq
      hp->seq = changes;
      last_ps = ps;
      last_lo = lo;
    }
    {
      const unsigned long long sk = ld_relaxed_sys(&H->stop);
      if (sk != hp->stop) {
        *(volatile unsigned long long*)&L->hp_stop_kind = sk;
        st_release_gpu(&L->hp_stop, sk ? epoch : 0ull);
        hp->stop = sk;
      }
    }
    while (true) {
      EcReq* dq = &L->dreq[pn % EC_REQ_RING];
      if (ld_acquire_gpu(&dq->seq1) == pn + 1) {   // stream-posted: nothing to copy
        ++pn;
        continue;
      }
      EcReq* q = &H->req[pn % EC_REQ_RING];
      if (ld_acquire_sys(&q->seq1) != pn + 1) break;
      volatile EcReq* v = dq;
      v->type = ld_relaxed_sys_u32(&q->type);
      v->flags = ld_relaxed_sys_u32(&q->flags) | EC_CF_HOSTPOSTED;
      v->t = (long long)ld_relaxed_sys((const unsigned long long*)&q->t);
      v->arg = (long long)ld_relaxed_sys((const unsigned long long*)&q->arg);
      __threadfence();
      st_release_gpu(&dq->seq1, pn + 1);
      ++pn;
    }
    __nanosleep(1000);
  }
}

template <typename T>
__global__ void __launch_bounds__(256, 2)
ec_engine(const EcDesc* __restrict__ descs, int blocks_per_rank, unsigned long long epoch) {
  const int lr = blockIdx.x / blocks_per_rank;
  const int role = blockIdx.x % blocks_per_rank;
  const EcDesc& d = descs[lr];
  if (role == 0) {
    __shared__ EcHpShared hp;
    if (threadIdx.x == 0) {
      // a relaunch starts from the persisted mirror (a stop request is the
      // poller's to see again: the host clears it before relaunching)
      hp.seq = *(volatile unsigned long long*)&d.local->hp_seq;
      hp.lo = *(volatile unsigned long long*)&d.local->hp_lo;
      hp.ps = *(volatile unsigned long long*)&d.local->hp_ps;
      hp.stop = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) engine_controller(d, epoch, &hp);
    else if (threadIdx.x == 32) engine_host_poller(d, epoch, &hp);
    return;
  }
  engine_worker<T>(d, role - 1, epoch);
}

template __global__ void ec_engine<float>(const EcDesc*, int, unsigned long long);
template __global__ void ec_engine<double>(const EcDesc*, int, unsigned long long);
template __global__ void ec_engine<long long>(const EcDesc*, int, unsigned long long);

// ---------------------------------------------------------------------------
// direct mode: a world of ONE rank.  With no peers there is no external
// activation, no snapshot race and nothing to pull, so the controller's request
// handling runs as a one-thread kernel in stream order and the round is an
// ordinary grid launch right behind it: no persistent kernel holds SMs and the
// whole step is profilable with ncu.  Same state words, replies and log as the
// engine (EcLocal / EcHostCtl), so the host API cannot tell the difference.

// decide one request against the device state (no host-visible stores);
// returns the reply status (EC_R_*)
__device__ unsigned long long direct_decide_core(const EcDesc& d, unsigned int type,
                                                 unsigned int flags, long long t, long long arg) {
  EcLocal* L = d.local;
  EcHostCtl* H = d.hctl;
  const long long g = L->g;
  unsigned long long status = 3;
  if (type == EC_REQ_CONTRIB) {
    if (flags & EC_CF_SRC_GRAD_AUTO) {
      if (*(volatile int*)&L->stash_null) flags |= EC_CF_SRC_GRAD;
      flags &= ~EC_CF_SRC_GRAD_AUTO;
    }
    const unsigned int poison = *(volatile unsigned int*)&L->poison;
    *(volatile unsigned int*)&L->poison = 0u;
    if (!(flags & EC_CF_SRC_GRAD)) *(volatile int*)&L->stash_null = 0;  // the stash holds an offer
    if (poison) {
      status = 4;
    } else if (t < g || (t == g && L->snapped)) {
      status = 2;
      if (flags & EC_CF_SRC_GRAD) L->late_copy = 1;
    } else if (t > g) {
      status = 5;
      st_release_sys(&H->error_info, (unsigned long long)t);
      st_release_sys(&H->error, EC_DERR_ORDER);
    } else {
      L->contrib = (int)(EC_SNAP_DATA | ((flags & 1u) ? EC_SNAP_FRESH : 0ull) |
                         ((flags & EC_CF_SRC_GRAD) ? EC_SNAP_SRC_GRAD : 0ull));
      L->contributed_round = t;
      status = 1;
      if (flags & 2u) L->snapped = 1;  // own activation: P == 1, everyone has arrived
    }
  } else if (type == EC_REQ_ACTIVATE) {
    if (t == g) L->snapped = 1;
  } else if (type == EC_REQ_HOLD) {
    L->hold_from = arg;
  }
  return status;
}

// Direct mode answers requests from kernels on more than one stream (a step's
// publication runs on its own stream, ec_host.cu): every writer of the
// monotone host words waits for its predecessor, so req_done / done_gen1 never
// move backwards.
__device__ void direct_wait_turn(const EcDesc& d, const unsigned long long* word,
                                 unsigned long long need) {
  if (ld_acquire_gpu(word) >= need) return;
  const unsigned long long t0 = globaltimer_ns();
  while (ld_acquire_gpu(word) < need) {
    if (globaltimer_ns() - t0 > d.timeout_ns) {
      st_release_sys(&d.hctl->error_info, need);
      st_release_sys(&d.hctl->error, EC_DERR_TIMEOUT);
      return;
    }
    __nanosleep(256);
  }
}

__device__ void direct_reply(const EcDesc& d, unsigned long long seq, unsigned long long status) {
  EcLocal* L = d.local;
  EcHostCtl* H = d.hctl;
  direct_wait_turn(d, &L->req_done_dev, seq);
  __threadfence();
  st_release_sys(&H->reply[seq % EC_REQ_RING], ((seq + 1) << 8) | status);
  st_release_sys(&H->req_done, seq + 1);
  st_release_gpu(&L->req_done_dev, seq + 1);
}

__global__ void ec_direct_decide(const EcDesc* __restrict__ dp, unsigned long long seq,
                                 unsigned int type, unsigned int flags, long long t, long long arg) {
  if (threadIdx.x == 0) direct_reply(*dp, seq, direct_decide_core(*dp, type, flags, t, arg));
}

struct DirectStepReport;
__device__ void direct_publish(const EcDesc& d, long long g, int contrib, unsigned long long has,
                               const DirectStepReport* step);

template <typename T>
__global__ void __launch_bounds__(256, 6)
ec_direct_round(const EcDesc* __restrict__ dp) {
  const EcDesc& d = *dp;
  EcLocal* L = d.local;
  if (!*(volatile int*)&L->snapped) return;   // nothing activated: no round
  const long long g = L->g;
  const int contrib = L->contrib;
  const unsigned long long has = (contrib & (int)EC_SNAP_DATA) ? 1ull : 0ull;
  const char* sp[1] = {(contrib & (int)EC_SNAP_SRC_GRAD) ? d.gbuf[d.rank] : d.send[d.rank]};
  char* slot = d.ring[d.rank] + (g % d.R) * d.slot_bytes;
  const long long start = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  rs_fixed<T, 1, 4>(d, sp, has, 0, d.nvec, slot, start, stride, (T)1, true);
  if (blockIdx.x == 0 && threadIdx.x < Ops<T>::V) rs_tail<T>(d, sp, has, slot, threadIdx.x);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long old = atomicAdd(&L->rs_count, 1ull);
    if (old + 1 == gridDim.x) {
      L->rs_count = 0;
      direct_publish(d, g, contrib, has, nullptr);
    }
  }
}

// the last CTA of a direct round: log, stash/hold state, next generation.
// Every host-visible word is a plain store ordered by ONE sys fence before the
// flags the host polls (a release per word would drain PCIe once per word).
// With step != nullptr it also reports the fused step (ec_direct_step_kernel):
// the request's reply and the step's generation / finiteness / time.
struct DirectStepReport {
  unsigned long long seq, status, t0;
  long long t;
  bool bad;
  unsigned long long t1;   // the step's kernel had completed (publication kernel entry)
};

__device__ void direct_publish(const EcDesc& d, long long g, int contrib, unsigned long long has,
                               const DirectStepReport* step = nullptr) {
  EcLocal* L = d.local;
  EcHostCtl* H = d.hctl;
  const unsigned long long fresh = (contrib & (int)EC_SNAP_FRESH) ? 1ull : 0ull;
  direct_wait_turn(d, &L->done_gen1_dev, (unsigned long long)g);
  if (step) direct_wait_turn(d, &L->req_done_dev, step->seq);
  EcLog* lg = &H->log[g % EC_LOG_RING];
  st_relaxed_sys(&lg->mask, fresh);
  st_relaxed_sys(&lg->has, has);
  st_relaxed_sys(&lg->nap, fresh);
  const unsigned long long tn = globaltimer_ns();
  st_relaxed_sys(&lg->t_snap, tn);
  st_relaxed_sys(&lg->t_cmd, tn);
  st_relaxed_sys(&lg->t_rs, tn);
  st_relaxed_sys(&lg->t_done, tn);
  if (!step) {   // a step's block 0 made these transitions when it decided
    if (fresh) {
      L->hold_from = EC_INF_GEN;
      L->stash_null = 1;
    }
    L->g = g + 1;
    L->snapped = 0;
    L->contrib = 0;
  }
  if (step) {
    const long long ts = step->t % EC_REQ_RING;
    st_relaxed_sys(&H->stepgen[ts], (unsigned long long)g + 1);
    st_relaxed_sys(&H->stepbad[ts], step->bad ? 1ull : 0ull);
    st_relaxed_sys(&H->stepns[ts], step->t1 - step->t0);
  }
  st_relaxed_sys(&lg->gen1, (unsigned long long)g + 1);   // record data: before the fence
  fence_acq_rel_sys();
  st_relaxed_sys(&H->snap_gen1, (unsigned long long)g + 1);
  st_relaxed_sys(&H->done_gen1, (unsigned long long)g + 1);
  st_relaxed_gpu(&L->done_gen1_dev, (unsigned long long)g + 1);
  if (step) {
    st_relaxed_sys(&H->reply[step->seq % EC_REQ_RING], ((step->seq + 1) << 8) | step->status);
    st_relaxed_sys(&H->req_done, step->seq + 1);
    st_relaxed_gpu(&L->req_done_dev, step->seq + 1);
    st_relaxed_sys(&H->steptag[step->t % EC_REQ_RING], (unsigned long long)step->t + 1);
  }
}

// ---------------------------------------------------------------------------
// standalone streaming kernels

// gate != nullptr: a preceding ec_finite_kernel's verdict; a non-finite
// gradient leaves the stash untouched (folding into a PENDING stash must not
// poison the gradients it already holds, eagersgd.py:145-147)
template <typename T, int MODE>
__global__ void __launch_bounds__(256, 6)
ec_fold_kernel(T* __restrict__ stash, const T* __restrict__ grad, long long n,
               unsigned int* nonfinite, int vec_ok, const unsigned int* gate) {
  if (gate && *(volatile const unsigned int*)gate) return;
  constexpr int V = Ops<T>::V;
  constexpr int U = 4;
  bool bad = false;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  long long done = 0;
  if (vec_ok) {
    const long long nv = n / V;
    for (long long base = tid; base < nv; base += nth * U) {
      Vec16<T> gv[U], sv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        long long v = base + u * nth;
        if (v < nv) {
          gv[u].raw = ld_stream_v4(grad + v * V);
          if (MODE == 1) sv[u].raw = ld_stream_v4(stash + v * V);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        long long v = base + u * nth;
        if (v < nv) {
          Vec16<T> o;
#pragma unroll
          for (int l = 0; l < V; ++l) {
            bad |= !Ops<T>::finite(gv[u].e[l]);
            o.e[l] = MODE == 1 ? Ops<T>::add(sv[u].e[l], gv[u].e[l]) : Ops<T>::canon(gv[u].e[l]);
          }
          st_v4(stash + v * V, o.raw);
        }
      }
    }
    done = nv * V;
  }
  for (long long e = done + tid; e < n; e += nth) {
    T gv = grad[e];
    bad |= !Ops<T>::finite(gv);
    stash[e] = MODE == 1 ? Ops<T>::add(stash[e], gv) : Ops<T>::canon(gv);
  }
  if (nonfinite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1u);
}

// flag |= any(!isfinite(grad)) -- the check pass ahead of a gated ADD fold
template <typename T>
__global__ void __launch_bounds__(256, 6)
ec_finite_kernel(const T* __restrict__ grad, long long n, unsigned int* flag, int vec_ok) {
  constexpr int V = Ops<T>::V;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  bool bad = false;
  long long done = 0;
  if (vec_ok) {
    const long long nv = n / V;
    for (long long v = tid; v < nv; v += nth) {
      Vec16<T> g;
      g.raw = ld_stream_v4(grad + v * V);
#pragma unroll
      for (int l = 0; l < V; ++l) bad |= !Ops<T>::finite(g.e[l]);
    }
    done = nv * V;
  }
  for (long long e = done + tid; e < n; e += nth) bad |= !Ops<T>::finite(grad[e]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

template <typename T>
__global__ void __launch_bounds__(256, 6)
ec_update_kernel(T* __restrict__ w, const T* __restrict__ u, T lr, long long n, int vec_ok) {
  constexpr int V = Ops<T>::V;
  constexpr int U = 4;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  long long done = 0;
  if (vec_ok) {
    const long long nv = n / V;
    for (long long base = tid; base < nv; base += nth * U) {
      Vec16<T> wv[U], uv[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        long long v = base + k * nth;
        if (v < nv) {
          wv[k].raw = ld_stream_v4(w + v * V);
          uv[k].raw = ld_stream_v4(u + v * V);
        }
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        long long v = base + k * nth;
        if (v < nv) {
#pragma unroll
          for (int l = 0; l < V; ++l) wv[k].e[l] = Ops<T>::sgd(wv[k].e[l], lr, uv[k].e[l]);
          st_v4(w + v * V, wv[k].raw);
        }
      }
    }
    done = nv * V;
  }
  for (long long e = done + tid; e < n; e += nth) w[e] = Ops<T>::sgd(w[e], lr, u[e]);
}

template <typename T>
__global__ void __launch_bounds__(256, 6)
ec_momentum_kernel(T* __restrict__ w, T* __restrict__ buf, const T* __restrict__ u, T lr, T mu,
                   long long n, int vec_ok) {
  constexpr int V = Ops<T>::V;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  long long done = 0;
  if (vec_ok) {
    const long long nv = n / V;
    for (long long v = tid; v < nv; v += nth) {
      Vec16<T> wv, bv, uv;
      wv.raw = ld_stream_v4(w + v * V);
      bv.raw = ld_stream_v4(buf + v * V);
      uv.raw = ld_stream_v4(u + v * V);
#pragma unroll
      for (int l = 0; l < V; ++l) {
        bv.e[l] = Ops<T>::mom(mu, bv.e[l], uv.e[l]);
        wv.e[l] = Ops<T>::sgd(wv.e[l], lr, bv.e[l]);
      }
      st_v4(buf + v * V, bv.raw);
      st_v4(w + v * V, wv.raw);
    }
    done = nv * V;
  }
  for (long long e = done + tid; e < n; e += nth) {
    T b = Ops<T>::mom(mu, buf[e], u[e]);
    buf[e] = b;
    w[e] = Ops<T>::sgd(w[e], lr, b);
  }
}

struct EcSrcs {
  const void* p[EC_MAX_P];
};

template <typename T, int P>
__device__ __forceinline__ void reduce_vec(const EcSrcs& s, unsigned long long has, T* dst, long long v,
                                           int div, T inv, bool pow2, int p) {
  constexpr int V = Ops<T>::V;
  Vec16<T> x[P];
#pragma unroll
  for (int q = 0; q < P; ++q)
    x[q].raw = ((has >> q) & 1ull) ? ld_stream_v4(reinterpret_cast<const T*>(s.p[q]) + v * V)
                                   : make_uint4(0, 0, 0, 0);
  Vec16<T> o;
#pragma unroll
  for (int l = 0; l < V; ++l) {
    T c[P];
#pragma unroll
    for (int q = 0; q < P; ++q) c[q] = Ops<T>::canon(x[q].e[l]);
    T sum = tree_sum<T, P>(c);
    o.e[l] = div ? Ops<T>::divp(sum, p, inv, pow2) : sum;
  }
  st_v4(dst + v * V, o.raw);
}

template <typename T>
__global__ void __launch_bounds__(256, 6)
ec_reduce_kernel(EcSrcs s, int p, unsigned long long has, T* __restrict__ dst, long long n,
                 int div, int vec_ok) {
  constexpr int V = Ops<T>::V;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  const bool pow2 = (p & (p - 1)) == 0;
  const T inv = (T)1 / (T)p;
  long long done = 0;
  if (vec_ok) {
    const long long nv = n / V;
    for (long long v = tid; v < nv; v += nth) {
      switch (p) {
        case 1: reduce_vec<T, 1>(s, has, dst, v, div, inv, pow2, p); break;
        case 2: reduce_vec<T, 2>(s, has, dst, v, div, inv, pow2, p); break;
        case 3: reduce_vec<T, 3>(s, has, dst, v, div, inv, pow2, p); break;
        case 4: reduce_vec<T, 4>(s, has, dst, v, div, inv, pow2, p); break;
        case 5: reduce_vec<T, 5>(s, has, dst, v, div, inv, pow2, p); break;
        case 6: reduce_vec<T, 6>(s, has, dst, v, div, inv, pow2, p); break;
        case 7: reduce_vec<T, 7>(s, has, dst, v, div, inv, pow2, p); break;
        case 8: reduce_vec<T, 8>(s, has, dst, v, div, inv, pow2, p); break;
        default: {
          Vec16<T> o;
#pragma unroll
          for (int l = 0; l < V; ++l) {
            auto leaf = [&](int q) -> T {
              if (!((has >> q) & 1ull)) return Ops<T>::zero();
              return Ops<T>::canon(reinterpret_cast<const T*>(s.p[q])[v * V + l]);
            };
            T sum = tree_sum_dyn<T>(p, leaf);
            o.e[l] = div ? Ops<T>::divp(sum, p, inv, pow2) : sum;
          }
          st_v4(dst + v * V, o.raw);
        }
      }
    }
    done = nv * V;
  }
  for (long long e = done + tid; e < n; e += nth) {
    auto leaf = [&](int q) -> T {
      if (!((has >> q) & 1ull)) return Ops<T>::zero();
      return Ops<T>::canon(reinterpret_cast<const T*>(s.p[q])[e]);
    };
    T sum = tree_sum_dyn<T>(p, leaf);
    dst[e] = div ? Ops<T>::divp(sum, p, inv, pow2) : sum;
  }
}

__global__ void ec_write_u64_kernel(unsigned long long* p, unsigned long long v) {
  if (threadIdx.x == 0) {
    fence_acq_rel_sys();
    st_release_sys(p, v);
  }
}

__global__ void ec_spin_kernel(unsigned long long ns) {
  if (threadIdx.x != 0) return;
  const unsigned long long t0 = globaltimer_ns();
  while (globaltimer_ns() - t0 < ns) __nanosleep(1000);
}

// ---------------------------------------------------------------------------
// asynchronous eager-SGD step: every decision the host used to wait for is
// taken on the device, in stream order, so a step is five launches and no
// host round trip: fold (mode from the device's stash state) -> post ->
// wait for a generation >= t (pin it) -> update from that slot -> unpin.

// post a request into the device ring (one thread)
__device__ __forceinline__ void post_request(EcLocal* L, unsigned long long seq1, unsigned type,
                                             unsigned flags, long long t, long long arg) {
  if (type == EC_REQ_CONTRIB) {
    if (*(volatile unsigned int*)&L->poison) flags |= EC_CF_POISON;
    *(volatile unsigned int*)&L->poison = 0u;
    // the stash / send buffer now holds an offer (unless the gradient buffer is offered)
    if (!(flags & EC_CF_SRC_GRAD)) *(volatile int*)&L->stash_null = 0;
  }
  EcReq* rec = &L->dreq[(seq1 - 1) % EC_REQ_RING];
  EC_ASSERT(seq1 - 1 - *(volatile unsigned long long*)&L->req_done_dev < EC_REQ_RING);
  volatile EcReq* v = rec;
  v->type = type;
  v->flags = flags;
  v->t = t;
  v->arg = arg;
  st_release_gpu(&rec->seq1, seq1);   // release: the fields (and stash_null) before seq1
  atomicMax(&L->posted, seq1);
}

// fold with the device-decided mode; with seq1 != 0 the last CTA also posts the
// offer (fused fold + post: one launch, the offer leaves as the stash is ready)
template <typename T>
__global__ void __launch_bounds__(256, 6)
ec_fold_auto_kernel(T* __restrict__ stash, const T* __restrict__ grad, long long n,
                    EcLocal* __restrict__ L, int vec_ok, unsigned long long seq1, unsigned flags,
                    long long t, int zero_copy) {
  asm volatile("griddepcontrol.wait;" ::: "memory");   // PDL-launched behind the previous step
  if (seq1 != 0 && blockIdx.x == 0 && threadIdx.x == 0) L->tl[t & 63][1] = globaltimer_ns();
  const int add = *(volatile int*)&L->stash_null ? 0 : 1;
  if (zero_copy && !add) {
    // null stash and the gradient sits in the registered buffer: offer it in
    // place (the reduction reads it over NVLink); nothing to fold
    if (seq1 != 0 && blockIdx.x == 0 && threadIdx.x == 0) {
      L->tl[t & 63][2] = globaltimer_ns();
      post_request(L, seq1, EC_REQ_CONTRIB, flags | EC_CF_SRC_GRAD, t, 0);
    }
    return;
  }
  constexpr int V = Ops<T>::V;
  bool bad = false;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  long long done = 0;
  if (vec_ok) {
    constexpr int U = 2;
    const long long nv = n / V;
    for (long long base = tid; base < nv; base += nth * U) {
      Vec16<T> gv[U], sv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long v = base + u * nth;
        if (v < nv) {
          gv[u].raw = ld_stream_v4(grad + v * V);
          if (add) sv[u].raw = ld_stream_v4(stash + v * V);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long v = base + u * nth;
        if (v < nv) {
          Vec16<T> o;
#pragma unroll
          for (int l = 0; l < V; ++l) {
            bad |= !Ops<T>::finite(gv[u].e[l]);
            o.e[l] = add ? Ops<T>::add(sv[u].e[l], gv[u].e[l]) : Ops<T>::canon(gv[u].e[l]);
          }
          st_v4(stash + v * V, o.raw);
        }
      }
    }
    done = nv * V;
  }
  for (long long e = done + tid; e < n; e += nth) {
    T gv = grad[e];
    bad |= !Ops<T>::finite(gv);
    stash[e] = add ? Ops<T>::add(stash[e], gv) : Ops<T>::canon(gv);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(&L->poison, 1u);
  if (seq1 == 0) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&L->fold_count, 1ull) == gridDim.x - 1) {
      __threadfence();
      L->fold_count = 0;
      L->tl[t & 63][2] = globaltimer_ns();
      post_request(L, seq1, EC_REQ_CONTRIB, flags, t, 0);
    }
  }
}

// wait for a generation >= t, pin it, publish it for the update (one thread)
// `lead`: how far the engine's snapshot frontier may run ahead of the last
// published generation (EcDesc::lead); a pin of G is safe once no snapshot of
// G + R can have happened, i.e. while done + lead < G + R
__device__ void wait_and_pin(EcLocal* L, EcHostCtl* H, long long t, int R, int lead,
                             unsigned long long timeout_ns, unsigned long long seq1) {
  const unsigned long long t0 = globaltimer_ns();
  unsigned long long d1;
  // the step's own offer must have been decided first (a refused zero-copy
  // offer asks this step to preserve the gradient in the stash)
  while (seq1 && ld_acquire_gpu(&L->req_done_dev) < seq1) {
    if (ld_relaxed_sys(&H->error) || globaltimer_ns() - t0 > timeout_ns) break;
    __nanosleep(64);
  }
  if (seq1 && *(volatile unsigned long long*)&L->fuse_seq == seq1) {
    // accepted for round t with arrival words: this kernel applies round t's
    // result chunk by chunk as it lands (the controller pinned slot t)
    L->step_fused = 1;
    L->step_late = 0;
    L->step_gen = t;
    L->upd_t0 = globaltimer_ns();
    st_relaxed_sys(&H->stepgen[t % EC_REQ_RING], (unsigned long long)t + 1);
    st_release_gpu(&L->step_tag, (unsigned long long)t + 1);
    return;
  }
  L->step_fused = 0;
  L->step_late = *(volatile int*)&L->late_copy;
  if (L->step_late) *(volatile int*)&L->late_copy = 0;
  while ((d1 = ld_acquire_gpu(&L->done_gen1_dev)) < (unsigned long long)t + 1) {
    if (ld_relaxed_sys(&H->error) || globaltimer_ns() - t0 > timeout_ns) {
      st_release_sys(&H->error_info, 0x200);
      st_release_sys(&H->error, EC_DERR_TIMEOUT);
      d1 = ld_acquire_gpu(&L->done_gen1_dev);
      break;
    }
    __nanosleep(64);
  }
  long long G = (long long)d1 - 1;
  // pin G (Dekker with the controller's check before snapshotting G + R;
  // both sides on this GPU, so gpu-scope SC fences suffice)
  while (true) {
    st_relaxed_gpu(&L->pin_dev, (unsigned long long)G);
    fence_sc_gpu();
    const long long D = (long long)ld_acquire_gpu(&L->done_gen1_dev) - 1;
    if (D < G + R - lead) break;
    G = D;
  }
  EC_ASSERT(G >= t || ld_relaxed_sys(&H->error) != 0);
  L->step_gen = G;
  L->upd_t0 = globaltimer_ns();
  st_relaxed_sys(&H->stepgen[t % EC_REQ_RING], (unsigned long long)G + 1);
  st_release_gpu(&L->step_tag, (unsigned long long)t + 1);
}

// stream-ordered wait for round t to complete at this rank (no pin): lets a
// host enqueue back-to-back rounds the way nccl-tests enqueues collectives
__global__ void ec_wait_done_kernel(EcLocal* L, EcHostCtl* H, long long t,
                                    unsigned long long timeout_ns) {
  if (threadIdx.x != 0) return;
  const unsigned long long t0 = globaltimer_ns();
  while (ld_acquire_gpu(&L->done_gen1_dev) < (unsigned long long)t + 1) {
    if (ld_relaxed_sys(&H->error) || globaltimer_ns() - t0 > timeout_ns) {
      st_release_sys(&H->error_info, 0x300);
      st_release_sys(&H->error, EC_DERR_TIMEOUT);
      break;
    }
  }
}

__global__ void ec_wait_gen_kernel(EcLocal* L, EcHostCtl* H, long long t, int R, int lead,
                                   unsigned long long timeout_ns) {
  if (threadIdx.x == 0) {
    wait_and_pin(L, H, t, R, lead, timeout_ns, 0);
    st_release_sys(&H->steptag[t % EC_REQ_RING], (unsigned long long)t + 1);
  }
}

// w = w - lr*u (or the momentum form), 16-byte vectors, U in flight per thread;
// returns whether this thread read a non-finite u
template <typename T, bool MOM, int U>
__device__ __forceinline__ bool update_body(T* __restrict__ w, T* __restrict__ mom,
                                            const T* __restrict__ u, T lr, T mu, long long n,
                                            int vec_ok) {
  constexpr int V = Ops<T>::V;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  long long done = 0;
  bool bad = false;
  if (vec_ok) {
    const long long nv = n / V;
    for (long long base = tid; base < nv; base += nth * U) {
      Vec16<T> wv[U], uv[U], bv[MOM ? U : 1];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const long long v = base + k * nth;
        if (v < nv) {
          wv[k].raw = ld_stream_v4(w + v * V);
          uv[k].raw = ld_cg_v4(u + v * V);
          if (MOM) bv[MOM ? k : 0].raw = ld_stream_v4(mom + v * V);
        }
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const long long v = base + k * nth;
        if (v < nv) {
#pragma unroll
          for (int l = 0; l < V; ++l) {
            bad |= !Ops<T>::finite(uv[k].e[l]);
            if (MOM) {
              bv[MOM ? k : 0].e[l] = Ops<T>::mom(mu, bv[MOM ? k : 0].e[l], uv[k].e[l]);
              wv[k].e[l] = Ops<T>::sgd(wv[k].e[l], lr, bv[MOM ? k : 0].e[l]);
            } else {
              wv[k].e[l] = Ops<T>::sgd(wv[k].e[l], lr, uv[k].e[l]);
            }
          }
          if (MOM) st_v4(mom + v * V, bv[MOM ? k : 0].raw);
          st_v4(w + v * V, wv[k].raw);
        }
      }
    }
    done = nv * V;
  }
  for (long long e = done + tid; e < n; e += nth) {
    T uu = u[e];
    bad |= !Ops<T>::finite(uu);
    if (MOM) {
      T b = Ops<T>::mom(mu, mom[e], uu);
      mom[e] = b;
      uu = b;
    }
    w[e] = Ops<T>::sgd(w[e], lr, uu);
  }
  return bad;
}

// update from the slot of the step's generation; with H != nullptr the kernel
// also performs the wait (block 0) and the last CTA releases the pin
// (fused wait + update + unpin: one launch)
// Progressive update (the step's offer was accepted for round g with arrival
// words): CTAs claim chunks in arrival order (k-th chunk of every owner's
// workers, then k+1 ...), wait for the owner worker's arrival word, and apply
// w - lr*u (or the momentum form) to the chunk -- the HBM-bound update runs
// while the NVLink-bound round is still moving later chunks.  Same _rn
// expressions as update_body.  Returns whether a value of u was non-finite.
template <typename T, bool MOM>
__device__ bool progressive_update(const EcDesc& d, T* __restrict__ w, T* __restrict__ mom, T lr,
                                   T mu, long long g, unsigned long long timeout_ns) {
  EcLocal* L = d.local;
  __shared__ long long s_item;
  constexpr int V = Ops<T>::V;
  constexpr int U = MOM ? 2 : 4;
  const int P = d.P, W = d.W < d.w_step ? d.W : d.w_step, chv = d.chv;   // the round's wact
  const long long nch = (d.nvec + chv - 1) / chv;
  long long kmax = 0;
  for (int q = 0; q < P; ++q) {
    const long long m = (chunk_lo(nch, q + 1, P) - chunk_lo(nch, q, P) + W - 1) / W;
    if (m > kmax) kmax = m;
  }
  const long long nitems = kmax * P * W;
  auto chunk_of = [&](long long i, int& q, int& wq, long long& k) -> long long {
    k = i / ((long long)P * W);
    const long long rem = i % ((long long)P * W);
    q = (int)(rem / W);
    wq = (int)(rem % W);
    const long long c = chunk_lo(nch, q, P) + wq + k * W;
    return c < chunk_lo(nch, q + 1, P) ? c : -1;
  };
  const T* __restrict__ u = reinterpret_cast<const T*>(d.ring[d.rank] + (g % d.R) * d.slot_bytes);
  const unsigned long long t0 = globaltimer_ns();
  bool bad = false;
  while (true) {
    if (threadIdx.x == 0) {
      long long i, c = -1;
      int q = 0, wq = 0;
      long long k = 0;
      do {
        i = (long long)atomicAdd(&L->upd_next_item, 1ull);
        if (i < nitems) c = chunk_of(i, q, wq, k);
      } while (i < nitems && c < 0);
      if (i < nitems) {
        const unsigned long long need =
            (((unsigned long long)g + 1) << EC_PROG_SHIFT) | (unsigned long long)(k + 1);
        const unsigned long long* pw = &d.ctrl[d.rank]->prog[q][wq];
        // hundreds of CTAs may wait at once: back off, or the polling starves
        // the engine's controller and its NVLink traffic
        unsigned ns = 256;
        while (ld_acquire_sys(pw) < need) {
          __nanosleep(ns);
          if (ns < 2048) ns <<= 1;
          if (globaltimer_ns() - t0 > timeout_ns) {
            st_release_sys(&d.hctl->error_info, 0x500 + q);
            st_release_sys(&d.hctl->error, EC_DERR_TIMEOUT);
            break;
          }
        }
        s_item = c;
      } else {
        s_item = -1;
      }
    }
    __syncthreads();
    const long long c = s_item;
    if (c < 0) break;
    EC_ASSERT(c < nch);
    const long long v0 = c * chv;
    const int nvv = (int)min((long long)chv, d.nvec - v0);
    for (int base = threadIdx.x; base < nvv; base += blockDim.x * U) {
      Vec16<T> uv[U], wv[U], bv[MOM ? U : 1];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int v = base + k * blockDim.x;
        if (v < nvv) {
          uv[k].raw = ld_cg_v4(u + (v0 + v) * V);
          wv[k].raw = ld_stream_v4(w + (v0 + v) * V);
          if (MOM) bv[MOM ? k : 0].raw = ld_stream_v4(mom + (v0 + v) * V);
        }
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int v = base + k * blockDim.x;
        if (v < nvv) {
#pragma unroll
          for (int l = 0; l < V; ++l) {
            bad |= !Ops<T>::finite(uv[k].e[l]);
            if (MOM) {
              bv[MOM ? k : 0].e[l] = Ops<T>::mom(mu, bv[MOM ? k : 0].e[l], uv[k].e[l]);
              wv[k].e[l] = Ops<T>::sgd(wv[k].e[l], lr, bv[MOM ? k : 0].e[l]);
            } else {
              wv[k].e[l] = Ops<T>::sgd(wv[k].e[l], lr, uv[k].e[l]);
            }
          }
          if (MOM) st_v4(mom + (v0 + v) * V, bv[MOM ? k : 0].raw);
          st_v4(w + (v0 + v) * V, wv[k].raw);
        }
      }
    }
    __syncthreads();   // s_item is reused
  }
  return bad;
}

template <typename T, bool MOM>
__device__ __forceinline__ void update_gen_body(T* __restrict__ w, T* __restrict__ mom,
                                                const char* __restrict__ ring, long long slot_bytes,
                                                int R, EcLocal* __restrict__ L, T lr, T mu,
                                                long long n, int vec_ok, EcHostCtl* H, long long t,
                                                unsigned long long timeout_ns, unsigned long long seq1,
                                                T* __restrict__ stash, const T* __restrict__ gbuf,
                                                const EcDesc* __restrict__ dp, int pub_side = 0) {
  __shared__ long long s_gen;
  __shared__ int s_late, s_fusedu;
  if (threadIdx.x == 0) {
    if (H != nullptr) {
      if (blockIdx.x == 0) wait_and_pin(L, H, t, R, dp->lead, timeout_ns, seq1);
      while (ld_acquire_gpu(&L->step_tag) != (unsigned long long)t + 1) __nanosleep(256);
    }
    s_gen = *(volatile const long long*)&L->step_gen;
    s_late = H != nullptr ? *(volatile const int*)&L->step_late : 0;
    s_fusedu = H != nullptr ? *(volatile const int*)&L->step_fused : 0;
    asm volatile("fence.proxy.alias;" ::: "memory");  // slot may be written via a multicast alias
  }
  __syncthreads();
  const long long G = s_gen;
  const T* __restrict__ u = reinterpret_cast<const T*>(ring + (G % R) * slot_bytes);
  bool bad;
  if (s_fusedu) {
    bad = progressive_update<T, MOM>(*dp, w, mom, lr, mu, G, timeout_ns);
  } else {
    if (s_late && stash && gbuf) {
      // a zero-copy offer missed its round: the gradient joins the stash (0 + g)
      // before the caller's next backward overwrites the gradient buffer
      const long long tid0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
      const long long nth0 = (long long)gridDim.x * blockDim.x;
      for (long long e = tid0; e < n; e += nth0) stash[e] = Ops<T>::canon(gbuf[e]);
    }
    bad = update_body<T, MOM, MOM ? 2 : 4>(w, mom, u, lr, mu, n, vec_ok);
  }
  // the next step's offer kernel may be scheduled now (it waits for our completion)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (H == nullptr) return;
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&L->upd_bad, 1u);
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&L->upd_count, 1ull) == gridDim.x - 1) {
      L->upd_count = 0;
      if (s_fusedu) {
        // the round's publication: the scalar tail (reduced by the last owner
        // with plain stores) and the log are in once done moves past G
        L->upd_next_item = 0;
        const unsigned long long tw = globaltimer_ns();
        while (ld_acquire_gpu(&L->done_gen1_dev) < (unsigned long long)G + 1) {
          if (ld_relaxed_sys(&H->error) || globaltimer_ns() - tw > timeout_ns) break;
          __nanosleep(64);
        }
        const volatile T* uv = u;
        bool tbad = false;
        for (long long e = dp->nvec * Ops<T>::V; e < n; ++e) {
          T uu = uv[e];
          tbad |= !Ops<T>::finite(uu);
          if (MOM) {
            const T b = Ops<T>::mom(mu, mom[e], uu);
            mom[e] = b;
            uu = b;
          }
          w[e] = Ops<T>::sgd(w[e], lr, uu);
        }
        if (tbad) atomicOr(&L->upd_bad, 1u);
      }
      if (s_late) *(volatile int*)&L->stash_null = 0;
      const unsigned int sbad = atomicExch(&L->upd_bad, 0u) ? 1u : 0u;
      const unsigned long long t1 = globaltimer_ns();
      L->tl[t & 63][0] = t1;
      st_release_gpu(&L->pin_dev, ~0ull);  // every CTA has read the slot: unpin
      const unsigned long long sns = t1 - *(volatile unsigned long long*)&L->upd_t0;
      if (pub_side) {
        // a direct step's out-of-line path: its publication kernel (own
        // stream, after the earlier steps' publications) reports it
        L->srep[t % EC_REQ_RING].ns = sns;
        L->srep[t % EC_REQ_RING].bad = sbad;
      } else {
        st_relaxed_sys(&H->stepbad[t % EC_REQ_RING], sbad);
        st_relaxed_sys(&H->stepns[t % EC_REQ_RING], sns);
        st_release_sys(&H->steptag[t % EC_REQ_RING], (unsigned long long)t + 1);
      }
    }
  }
}

template <typename T, bool MOM>
__global__ void __launch_bounds__(256, 4)
ec_update_gen_kernel(T* __restrict__ w, T* __restrict__ mom, const char* __restrict__ ring,
                     long long slot_bytes, int R, EcLocal* __restrict__ L, T lr, T mu,
                     long long n, int vec_ok, EcHostCtl* H, long long t,
                     unsigned long long timeout_ns, unsigned long long seq1,
                     T* __restrict__ stash, const T* __restrict__ gbuf,
                     const EcDesc* __restrict__ dp) {
  update_gen_body<T, MOM>(w, mom, ring, slot_bytes, R, L, lr, mu, n, vec_ok, H, t, timeout_ns, seq1,
                          stash, gbuf, dp);
}

// Direct mode (world of one) async step, ONE pass per element: decide the
// step's offer (block 0), then -- when it opened round t, the common case --
// u = (0 + x) / 1 into the slot and w -= lr*u (or the momentum form) from the
// register copy of u, so the update never re-reads the slot.  x is the
// registered gradient buffer (zero-copy offer, null stash), the stash (folded
// by ec_fold_auto), or -- FOLD, a zero-copy call that met a non-null stash --
// stash + g, folded in this same pass.  Bit-identical to fold + decide + round
// + update as separate launches (same expressions, same order).
//
// Shape (measured, profiles/): full occupancy -- one 16-byte vector of each
// stream per thread, 8 CTAs of 256 threads per SM, one CTA per 256 vectors.
// Block 0 decides and publishes the decision packed into ONE word
// (dec_tag = (seq+1) << 8 | bits), so every other CTA's prologue is a single
// acquire load; completion is the kernel boundary (ec_direct_publish_kernel,
// launched behind it on the communicator's publication stream, writes every
// host-visible word behind one sys fence), so no CTA pays a fence or a counter
// atomic, and the next step's kernel does not wait for the publication: block
// 0 makes the round's state transitions when it decides and leaves the report
// in EcLocal::drep.  The rare no-round path (refused offer) runs out of line
// with the ordinary wait + update body.
#define EC_DW_FUSED 1u
#define EC_DW_FOLD 2u
#define EC_DW_HAS 4u
#define EC_DW_SRCG 8u

template <typename T, bool MOM>
__device__ __noinline__ void direct_step_fallback(const EcDesc& d, unsigned long long seq,
                                                  unsigned long long status, int fold, T* w,
                                                  T* mom, T lr, T mu, int vec_ok, long long t,
                                                  unsigned long long timeout_ns) {
  EcLocal* L = d.local;
  T* stash = reinterpret_cast<T*>(d.send[d.rank]);
  const T* gbuf = reinterpret_cast<const T*>(d.gbuf[d.rank]);
  const long long n = d.n;
  if (fold) {
    const long long tid0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nth0 = (long long)gridDim.x * blockDim.x;
    for (long long e = tid0; e < n; e += nth0) stash[e] = Ops<T>::add(stash[e], gbuf[e]);
  }
  // the reply and the step's report come from ec_direct_publish_kernel (this
  // kernel never waits for an earlier publication: its CTAs would hold every
  // SM slot that publication needs)
  (void)status;
  update_gen_body<T, MOM>(w, mom, d.ring[d.rank], d.slot_bytes, d.R, L, lr, mu, n, vec_ok, d.hctl,
                          t, timeout_ns, 0, stash, gbuf, &d, 1);
}

template <typename T, bool MOM>
__global__ void __launch_bounds__(256, 8)
ec_direct_step_kernel(const EcDesc* __restrict__ dp, unsigned long long seq,
                           unsigned int flags, T* __restrict__ w, T* __restrict__ mom, T lr, T mu,
                           int vec_ok, long long t, unsigned long long timeout_ns) {
  const EcDesc& d = *dp;
  EcLocal* L = d.local;
  __shared__ unsigned long long s_dw;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    unsigned long long dw;
    if (blockIdx.x == 0) {
      const unsigned long long t0 = globaltimer_ns();
      int fold, contrib, fused;
      unsigned long long status;
      {
        // direct_decide_core for an offer, from ONE batch of plain loads: every
        // writer of these words is an earlier kernel in stream order, so they
        // need no acquire, and the loads overlap instead of paying an L2 round
        // trip each while every other CTA waits for the decision
        const long long g = L->g;
        const int stash_null = L->stash_null, snapped = L->snapped, contrib0 = L->contrib;
        const unsigned int poison = L->poison;
        fold = (flags & EC_CF_SRC_GRAD_AUTO) && !stash_null;
        unsigned int fl = flags;
        if (fl & EC_CF_SRC_GRAD_AUTO) {
          if (stash_null) fl |= EC_CF_SRC_GRAD;
          fl &= ~EC_CF_SRC_GRAD_AUTO;
        }
        if (poison) L->poison = 0u;
        if (!(fl & EC_CF_SRC_GRAD) && stash_null) L->stash_null = 0;   // the stash holds an offer
        contrib = contrib0;
        fused = snapped;
        if (poison) {
          status = 4;
        } else if (t < g || (t == g && snapped)) {
          status = 2;
          if (fl & EC_CF_SRC_GRAD) L->late_copy = 1;
        } else if (t > g) {
          status = 5;
          st_release_sys(&d.hctl->error_info, (unsigned long long)t);
          st_release_sys(&d.hctl->error, EC_DERR_ORDER);
        } else {
          contrib = (int)(EC_SNAP_DATA | ((fl & 1u) ? EC_SNAP_FRESH : 0ull) |
                          ((fl & EC_CF_SRC_GRAD) ? EC_SNAP_SRC_GRAD : 0ull));
          L->contrib = contrib;
          L->contributed_round = t;
          status = 1;
          if (fl & 2u) {   // own activation: P == 1, everyone has arrived
            L->snapped = 1;
            fused = 1;
          }
        }
      }
      L->dec_status = status;
      L->dec_fold = fold;
      L->upd_t0 = t0;
      auto* rp = &L->drep[seq % EC_REQ_RING];
      rp->status = status;
      rp->t0 = t0;
      rp->contrib = contrib;
      rp->fused = fused ? 1u : 0u;
      rp->bad = 0u;
      if (fused) {
        // round t completes inside this launch: the next step's decision sees
        // the state after it now, whenever the publication runs
        if (contrib & (int)EC_SNAP_FRESH) {
          L->hold_from = EC_INF_GEN;
          L->stash_null = 1;
        }
        L->g = t + 1;
        L->snapped = 0;
        L->contrib = 0;
      }
      dw = ((seq + 1) << 8) | (fused ? EC_DW_FUSED : 0u) | (fold ? EC_DW_FOLD : 0u) |
           ((contrib & (int)EC_SNAP_DATA) ? EC_DW_HAS : 0u) |
           ((contrib & (int)EC_SNAP_SRC_GRAD) ? EC_DW_SRCG : 0u);
      st_release_gpu(&L->dec_tag, dw);   // release: every state word above first
    } else {
      // spin: the first wave's CTAs wait ~1 us, a sleep would wake late
      while (((dw = ld_acquire_gpu(&L->dec_tag)) >> 8) != seq + 1) {
      }
    }
    s_dw = dw;
  } else {
    // While thread 0 waits for the decision, the other threads prefetch this
    // thread's vectors into L2 (w, the momentum, and the likely source: the
    // registered bucket for a zero-copy call, else the stash): a hint, no
    // registers, and it doubles the requests each SM has in flight --
    // 70.6 -> 63.5 us per step (r2_direct_prefetch_ab.txt)
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    constexpr int V = Ops<T>::V;
    if (vec_ok && v < d.n / V) {
      const T* src_guess = reinterpret_cast<const T*>(
          (flags & EC_CF_SRC_GRAD_AUTO) ? d.gbuf[d.rank] : d.send[d.rank]);
      prefetch_l2(w + v * V);
      prefetch_l2(src_guess + v * V);
      if (MOM) prefetch_l2(mom + v * V);
    }
  }
  __syncthreads();
  const unsigned long long dw = s_dw;
  if (!(dw & EC_DW_FUSED)) {
    direct_step_fallback<T, MOM>(d, seq, *(volatile unsigned long long*)&L->dec_status,
                                 (dw & EC_DW_FOLD) ? 1 : 0, w, mom, lr, mu, vec_ok, t, timeout_ns);
    return;
  }
  // an accepted offer with activation opened round g == t (P == 1)
  const long long g = t;
  constexpr int V = Ops<T>::V;
  const bool has = (dw & EC_DW_HAS) != 0, fold = (dw & EC_DW_FOLD) != 0;
  T* stash = reinterpret_cast<T*>(d.send[d.rank]);
  const T* gbuf = reinterpret_cast<const T*>(d.gbuf[d.rank]);
  const T* src = (dw & EC_DW_SRCG) ? gbuf : stash;
  T* slot = reinterpret_cast<T*>(d.ring[d.rank] + (g % d.R) * d.slot_bytes);
  const long long n = d.n, nv = vec_ok ? n / V : 0;
  auto reduce1 = [&](T x) -> T {   // rs_fixed<T, 1>: tree of one canonical leaf, / 1
    T c[1] = {Ops<T>::canon(x)};
    return Ops<T>::divp(tree_sum<T, 1>(c), 1, (T)1, true);
  };
  bool bad = false;
  const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (v < nv) {
    Vec16<T> xv, wv, bv, gv;
    xv.raw = has ? ld_stream_v4(src + v * V) : make_uint4(0, 0, 0, 0);
    if (fold) gv.raw = ld_stream_v4(gbuf + v * V);
    wv.raw = ld_stream_v4(w + v * V);
    if (MOM) bv.raw = ld_stream_v4(mom + v * V);
    if (fold) {
#pragma unroll
      for (int l = 0; l < V; ++l) xv.e[l] = Ops<T>::add(xv.e[l], gv.e[l]);
      st_v4(stash + v * V, xv.raw);
    }
    Vec16<T> uv;
#pragma unroll
    for (int l = 0; l < V; ++l) {
      uv.e[l] = reduce1(xv.e[l]);
      bad |= !Ops<T>::finite(uv.e[l]);
      if (MOM) {
        bv.e[l] = Ops<T>::mom(mu, bv.e[l], uv.e[l]);
        wv.e[l] = Ops<T>::sgd(wv.e[l], lr, bv.e[l]);
      } else {
        wv.e[l] = Ops<T>::sgd(wv.e[l], lr, uv.e[l]);
      }
    }
    st_v4(slot + v * V, uv.raw);
    if (MOM) st_v4(mom + v * V, bv.raw);
    st_v4(w + v * V, wv.raw);
  }
  if (blockIdx.x == gridDim.x - 1) {
    // elements past the whole vectors (or all of them when unaligned)
    for (long long e = nv * V + threadIdx.x; e < n; e += blockDim.x) {
      T x = has ? src[e] : Ops<T>::zero();
      if (fold) {
        x = Ops<T>::add(x, gbuf[e]);
        stash[e] = x;
      }
      T uu = reduce1(x);
      slot[e] = uu;
      bad |= !Ops<T>::finite(uu);
      if (MOM) {
        const T b = Ops<T>::mom(mu, mom[e], uu);
        mom[e] = b;
        uu = b;
      }
      w[e] = Ops<T>::sgd(w[e], lr, uu);
    }
  }
  // completion is the kernel boundary: ec_direct_publish_kernel (launched
  // right behind, PDL) reports once every CTA's stores are visible
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
    atomicOr(&L->drep[seq % EC_REQ_RING].bad, 1u);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__global__ void ec_direct_publish_kernel(const EcDesc* __restrict__ dp, unsigned long long seq,
                                         long long t) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x != 0) return;
  const unsigned long long t1 = globaltimer_ns();
  const EcDesc& d = *dp;
  EcLocal* L = d.local;
  const auto* rp = &L->drep[seq % EC_REQ_RING];
  if (!*(volatile unsigned*)&rp->fused) {
    // the out-of-line path (no round): the offer's reply and the step report
    // (stepgen was stored by its wait; the kernel boundary made it visible)
    EcHostCtl* H = d.hctl;
    const long long ts = t % EC_REQ_RING;
    direct_wait_turn(d, &L->req_done_dev, seq);
    st_relaxed_sys(&H->stepbad[ts], *(volatile unsigned*)&L->srep[ts].bad);
    st_relaxed_sys(&H->stepns[ts], *(volatile unsigned long long*)&L->srep[ts].ns);
    st_relaxed_sys(&H->reply[seq % EC_REQ_RING],
                   ((seq + 1) << 8) | *(volatile unsigned long long*)&rp->status);
    fence_acq_rel_sys();
    st_relaxed_sys(&H->req_done, seq + 1);
    st_relaxed_gpu(&L->req_done_dev, seq + 1);
    st_relaxed_sys(&H->steptag[ts], (unsigned long long)t + 1);
    return;
  }
  const int contrib = *(volatile int*)&rp->contrib;
  DirectStepReport rep{seq, *(volatile unsigned long long*)&rp->status,
                       *(volatile unsigned long long*)&rp->t0, t,
                       *(volatile unsigned*)&rp->bad != 0u, t1};
  direct_publish(d, t, contrib, (contrib & (int)EC_SNAP_DATA) ? 1ull : 0ull, &rep);
}

__global__ void ec_post_kernel(EcLocal* L, unsigned long long seq1, unsigned int type,
                               unsigned int flags, long long t, long long arg) {
  if (threadIdx.x == 0) post_request(L, seq1, type, flags, t, arg);
}

// ---------------------------------------------------------------------------
// host-side launch helpers (C++ linkage, used by ec_host.cu)

// Launches issued by this library (bench.py reports the count for its timed region).
unsigned long long g_ec_launches = 0;
static inline void counted(int n = 1) { __atomic_add_fetch(&g_ec_launches, (unsigned long long)n, __ATOMIC_RELAXED); }

// One full wave of the kernel: SMs x resident blocks (grid-stride loops take
// the rest), queried once per kernel; never more blocks than work.
static int g_num_sms = 0;
static int sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}
// streaming kernels are __launch_bounds__(256, 6): exactly one wave is
// SMs x 6 blocks, grid-stride loops do the rest (no second-wave tail)
static inline int grid_for(long long work, int threads) {
  long long b = (work + threads - 1) / threads;
  const long long cap = (long long)sms() * 6;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

// resume (checkpoint): re-base a parked rank at generation `gen`
__global__ void ec_set_generation_kernel(EcLocal* L, EcHostCtl* H, long long gen, int stash_pending,
                                         long long contributed_round) {
  if (threadIdx.x != 0) return;
  L->g = gen;
  L->hold_from = EC_INF_GEN;
  L->contributed_round = contributed_round;
  L->snapped = 0;
  L->contrib = 0;
  L->internal_act = 0;
  L->arrive_pending = 0;
  L->arrive_activate = 0;
  L->stash_null = stash_pending ? 0 : 1;
  // guard ages restart at the resume point; the host re-seeds the pending
  // stash's oldest round with its next ec_post_guard (staleness_guard)
  L->pend_lo = EC_INF_GEN;
  L->last_off = gen - 1;
  L->poison = 0u;
  L->late_copy = 0;
  L->pin_dev = ~0ull;
  __threadfence();
  st_release_gpu(&L->done_gen1_dev, (unsigned long long)gen);
  st_release_sys(&H->snap_gen1, (unsigned long long)gen);
  st_release_sys(&H->done_gen1, (unsigned long long)gen);
}

cudaError_t launch_set_generation(EcLocal* L, EcHostCtl* H, long long gen, int stash_pending,
                                  long long contributed_round, cudaStream_t s) {
  ec_set_generation_kernel<<<1, 32, 0, s>>>(L, H, gen, stash_pending, contributed_round);
  return cudaGetLastError();
}

// stream barrier across the ranks of a communicator: every rank's kernel adds
// one to rank 0's counter (system-scope atomic over NVLink) and spins until all
// P arrivals of this epoch are in; watchdog-bounded
__global__ void ec_stream_barrier_kernel(unsigned long long* count, unsigned long long target,
                                         EcHostCtl* H, unsigned long long timeout_ns) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  atomicAdd_system(count, 1ull);
  const unsigned long long t0 = globaltimer_ns();
  while (ld_acquire_sys(count) < target) {
    if (globaltimer_ns() - t0 > timeout_ns) {
      st_release_sys(&H->error_info, 0x700);
      st_release_sys(&H->error, EC_DERR_TIMEOUT);
      break;
    }
  }
}

// Force-load every kernel of this library.  With CUDA lazy loading a kernel's
// first launch loads its code, and that load waits for running kernels -- which
// never happens while the persistent engine is resident.  Called before the
// engine first starts.
cudaError_t preload_kernels() {
  const void* fns[] = {
      (const void*)ec_engine<float>, (const void*)ec_engine<double>, (const void*)ec_engine<long long>,
      (const void*)ec_fold_kernel<float, 0>, (const void*)ec_fold_kernel<float, 1>,
      (const void*)ec_fold_kernel<double, 0>, (const void*)ec_fold_kernel<double, 1>,
      (const void*)ec_fold_kernel<long long, 0>, (const void*)ec_fold_kernel<long long, 1>,
      (const void*)ec_update_kernel<float>, (const void*)ec_update_kernel<double>,
      (const void*)ec_finite_kernel<float>, (const void*)ec_finite_kernel<double>,
      (const void*)ec_momentum_kernel<float>, (const void*)ec_momentum_kernel<double>,
      (const void*)ec_reduce_kernel<float>, (const void*)ec_reduce_kernel<double>,
      (const void*)ec_reduce_kernel<long long>,
      (const void*)ec_direct_decide, (const void*)ec_direct_round<float>,
      (const void*)ec_direct_round<double>, (const void*)ec_direct_round<long long>,
      (const void*)ec_post_kernel, (const void*)ec_write_u64_kernel, (const void*)ec_spin_kernel,
      (const void*)ec_fold_auto_kernel<float>, (const void*)ec_fold_auto_kernel<double>,
      (const void*)ec_fold_auto_kernel<long long>, (const void*)ec_wait_gen_kernel,
      (const void*)ec_wait_done_kernel,
      (const void*)ec_update_gen_kernel<float, false>, (const void*)ec_update_gen_kernel<double, false>,
      (const void*)ec_direct_step_kernel<float, false>, (const void*)ec_direct_step_kernel<double, false>,
      (const void*)ec_direct_step_kernel<float, true>, (const void*)ec_direct_step_kernel<double, true>,
      (const void*)ec_direct_publish_kernel, (const void*)ec_stream_barrier_kernel,
      (const void*)ec_set_generation_kernel,
      (const void*)ec_update_gen_kernel<float, true>, (const void*)ec_update_gen_kernel<double, true>,
  };
  for (const void* f : fns) {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// engine CTAs of this configuration that fit on one SM (shared memory /
// registers); the host budgets every engine on a device against it
int engine_blocks_per_sm(int dtype, int smem_bytes) {
  const void* fn = dtype == 0 ? (const void*)ec_engine<float>
                  : dtype == 1 ? (const void*)ec_engine<double>
                               : (const void*)ec_engine<long long>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes) != cudaSuccess)
    return 0;
  int k = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&k, fn, 256, smem_bytes) != cudaSuccess) return 0;
  return k;
}

cudaError_t launch_engine(int dtype, const EcDesc* d_descs, int n_local, int blocks_per_rank,
                          unsigned long long epoch, int smem_bytes, cudaStream_t s) {
  void* args[] = {(void*)&d_descs, (void*)&blocks_per_rank, (void*)&epoch};
  dim3 grid(n_local * blocks_per_rank), block(256);
  const void* fn = dtype == 0 ? (const void*)ec_engine<float>
                  : dtype == 1 ? (const void*)ec_engine<double>
                               : (const void*)ec_engine<long long>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  if (e != cudaSuccess) return e;
  counted();
  if (getenv("EC_NONCOOP")) return cudaLaunchKernel(fn, grid, block, args, smem_bytes, s);
  return cudaLaunchCooperativeKernel(fn, grid, block, args, smem_bytes, s);
}

// gated != 0 (ADD into a pending stash, float types, a poison flag given):
// a check pass first, and the fold writes nothing if it found a non-finite value
cudaError_t launch_fold(int dtype, void* stash, const void* grad, long long n, int mode,
                        unsigned int* nonfinite, cudaStream_t s, int gated) {
  counted();
  const int vec_ok = ((((uintptr_t)stash) | ((uintptr_t)grad)) & 15) == 0;
  const int V = dtype == 0 ? 4 : 2;
  const int grid = grid_for((n / V + 3) / 4 + 1, 256);
  const unsigned int* gate = nullptr;
  if (gated && mode && nonfinite && dtype != 2) {
    counted();
    const int vg = (((uintptr_t)grad) & 15) == 0;
    const int cg = grid_for(n / V + 1, 256);
    if (dtype == 0) ec_finite_kernel<float><<<cg, 256, 0, s>>>((const float*)grad, n, nonfinite, vg);
    else ec_finite_kernel<double><<<cg, 256, 0, s>>>((const double*)grad, n, nonfinite, vg);
    gate = nonfinite;
  }
  if (dtype == 0) {
    if (mode) ec_fold_kernel<float, 1><<<grid, 256, 0, s>>>((float*)stash, (const float*)grad, n, nonfinite, vec_ok, gate);
    else ec_fold_kernel<float, 0><<<grid, 256, 0, s>>>((float*)stash, (const float*)grad, n, nonfinite, vec_ok, gate);
  } else if (dtype == 1) {
    if (mode) ec_fold_kernel<double, 1><<<grid, 256, 0, s>>>((double*)stash, (const double*)grad, n, nonfinite, vec_ok, gate);
    else ec_fold_kernel<double, 0><<<grid, 256, 0, s>>>((double*)stash, (const double*)grad, n, nonfinite, vec_ok, gate);
  } else {
    if (mode) ec_fold_kernel<long long, 1><<<grid, 256, 0, s>>>((long long*)stash, (const long long*)grad, n, nonfinite, vec_ok, gate);
    else ec_fold_kernel<long long, 0><<<grid, 256, 0, s>>>((long long*)stash, (const long long*)grad, n, nonfinite, vec_ok, gate);
  }
  return cudaGetLastError();
}

cudaError_t launch_update(int dtype, void* w, const void* u, double lr, long long n, cudaStream_t s) {
  counted();
  const int vec_ok = ((((uintptr_t)w) | ((uintptr_t)u)) & 15) == 0;
  const int V = dtype == 0 ? 4 : 2;
  const int grid = grid_for((n / V + 3) / 4 + 1, 256);
  if (dtype == 0) ec_update_kernel<float><<<grid, 256, 0, s>>>((float*)w, (const float*)u, (float)lr, n, vec_ok);
  else if (dtype == 1) ec_update_kernel<double><<<grid, 256, 0, s>>>((double*)w, (const double*)u, lr, n, vec_ok);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_momentum(int dtype, void* w, void* buf, const void* u, double lr, double mu,
                            long long n, cudaStream_t s) {
  counted();
  const int vec_ok = ((((uintptr_t)w) | ((uintptr_t)u) | ((uintptr_t)buf)) & 15) == 0;
  const int V = dtype == 0 ? 4 : 2;
  const int grid = grid_for(n / V + 1, 256);
  if (dtype == 0) ec_momentum_kernel<float><<<grid, 256, 0, s>>>((float*)w, (float*)buf, (const float*)u, (float)lr, (float)mu, n, vec_ok);
  else if (dtype == 1) ec_momentum_kernel<double><<<grid, 256, 0, s>>>((double*)w, (double*)buf, (const double*)u, lr, mu, n, vec_ok);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_reduce(int dtype, const void* const* srcs, int p, unsigned long long has, void* dst,
                          long long n, int div, cudaStream_t s) {
  counted();
  EcSrcs S;
  uintptr_t bits = (uintptr_t)dst;
  for (int q = 0; q < EC_MAX_P; ++q) {
    S.p[q] = q < p ? srcs[q] : nullptr;
    if (q < p) bits |= (uintptr_t)srcs[q];
  }
  const int vec_ok = (bits & 15) == 0;
  const int V = dtype == 0 ? 4 : 2;
  const int grid = grid_for(n / V + 1, 256);
  if (dtype == 0) ec_reduce_kernel<float><<<grid, 256, 0, s>>>(S, p, has, (float*)dst, n, div, vec_ok);
  else if (dtype == 1) ec_reduce_kernel<double><<<grid, 256, 0, s>>>(S, p, has, (double*)dst, n, div, vec_ok);
  else ec_reduce_kernel<long long><<<grid, 256, 0, s>>>(S, p, has, (long long*)dst, n, div, vec_ok);
  return cudaGetLastError();
}

cudaError_t launch_post(EcLocal* L, unsigned long long seq1, unsigned int type, unsigned int flags,
                        long long t, long long arg, cudaStream_t s) {
  counted();
  ec_post_kernel<<<1, 32, 0, s>>>(L, seq1, type, flags, t, arg);
  return cudaGetLastError();
}

cudaError_t launch_direct(int dtype, const EcDesc* d_desc, long long nvec, unsigned long long seq,
                          unsigned int type, unsigned int flags, long long t, long long arg,
                          cudaStream_t s) {
  const bool no_round = type == EC_REQ_HOLD || type == EC_REQ_GUARD;
  counted(no_round ? 1 : 2);
  ec_direct_decide<<<1, 32, 0, s>>>(d_desc, seq, type, flags, t, arg);
  if (no_round) return cudaGetLastError();
  const int grid = grid_for((nvec + 3) / 4 + 1, 256);
  if (dtype == 0) ec_direct_round<float><<<grid, 256, 0, s>>>(d_desc);
  else if (dtype == 1) ec_direct_round<double><<<grid, 256, 0, s>>>(d_desc);
  else ec_direct_round<long long><<<grid, 256, 0, s>>>(d_desc);
  return cudaGetLastError();
}

cudaError_t launch_fold_auto(int dtype, void* stash, const void* grad, long long n, EcLocal* L,
                             unsigned long long seq1, unsigned flags, long long t, int zero_copy,
                             cudaStream_t s) {
  counted();
  const int vec_ok = ((((uintptr_t)stash) | ((uintptr_t)grad)) & 15) == 0;
  const int V = dtype == 0 ? 4 : 2;
  const int grid = grid_for((n / V + 1) / 2 + 1, 256);
  // programmatic dependent launch: scheduled while the previous step's update
  // kernel drains (griddepcontrol.wait in the kernel orders every read)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = getenv("EC_NO_PDL") ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (dtype == 0)
    return cudaLaunchKernelEx(&cfg, ec_fold_auto_kernel<float>, (float*)stash, (const float*)grad, n, L,
                              vec_ok, seq1, flags, t, zero_copy);
  if (dtype == 1)
    return cudaLaunchKernelEx(&cfg, ec_fold_auto_kernel<double>, (double*)stash, (const double*)grad, n,
                              L, vec_ok, seq1, flags, t, zero_copy);
  return cudaLaunchKernelEx(&cfg, ec_fold_auto_kernel<long long>, (long long*)stash,
                            (const long long*)grad, n, L, vec_ok, seq1, flags, t, zero_copy);
}

cudaError_t launch_wait_done(EcLocal* L, EcHostCtl* H, long long t, unsigned long long timeout_ns,
                             cudaStream_t s) {
  counted();
  ec_wait_done_kernel<<<1, 32, 0, s>>>(L, H, t, timeout_ns);
  return cudaGetLastError();
}

cudaError_t launch_wait_gen(EcLocal* L, EcHostCtl* H, long long t, int R, int lead,
                            unsigned long long timeout_ns, cudaStream_t s) {
  counted();
  ec_wait_gen_kernel<<<1, 32, 0, s>>>(L, H, t, R, lead, timeout_ns);
  return cudaGetLastError();
}

cudaError_t launch_update_gen(int dtype, void* w, void* mom, const char* ring, long long slot_bytes,
                              int R, EcLocal* L, double lr, double mu, long long n, EcHostCtl* H,
                              long long t, unsigned long long timeout_ns, unsigned long long seq1,
                              void* stash, const void* gbuf, const EcDesc* dp, int progressive,
                              int share, cudaStream_t s) {
  counted();
  const int vec_ok = ((((uintptr_t)w) | ((uintptr_t)mom) | ((uintptr_t)ring) | slot_bytes) & 15) == 0;
  const int V = dtype == 0 ? 4 : 2;
  // __launch_bounds__(256, 4): one wave is SMs x 4 blocks
  long long gb = ((n / V + 1) / 4 + 255) / 256 + 1;
  // a progressive update shares the SMs with the running round: 2 CTAs per SM
  // (measured: 296 CTAs beat 592 by 1-1.5 % per step at P=2/4; 148 leaves too
  // much of the update after the round)
  const int per_sm = progressive ? 2 : 4;
  int grid = (int)(gb < (long long)sms() * per_sm ? gb : (long long)sms() * per_sm);
  // ranks sharing one GPU (emulated worlds): each rank's update may spin on a
  // round another local rank has yet to join, so together they must leave that
  // rank room to run -- split the wave between the local ranks
  if (share > 1) grid = grid / share > 0 ? grid / share : 1;
  if (const char* e = getenv("EC_UPD_GRID")) {
    const int g = atoi(e);
    if (g > 0 && g < grid) grid = g;
  }
  if (dtype == 0) {
    auto kern = mom ? ec_update_gen_kernel<float, true> : ec_update_gen_kernel<float, false>;
    kern<<<grid, 256, 0, s>>>((float*)w, (float*)mom, ring, slot_bytes, R, L, (float)lr, (float)mu, n,
                              vec_ok, H, t, timeout_ns, seq1, (float*)stash, (const float*)gbuf, dp);
  } else if (dtype == 1) {
    auto kern = mom ? ec_update_gen_kernel<double, true> : ec_update_gen_kernel<double, false>;
    kern<<<grid, 256, 0, s>>>((double*)w, (double*)mom, ring, slot_bytes, R, L, lr, mu, n, vec_ok, H,
                              t, timeout_ns, seq1, (double*)stash, (const double*)gbuf, dp);
  }
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_direct_step(int dtype, const EcDesc* d_desc, unsigned long long seq,
                               unsigned int flags, void* w, void* mom, const void* ring,
                               long long slot_bytes, const void* src0, const void* src1,
                               double lr, double mu, long long n, long long t,
                               unsigned long long timeout_ns, cudaStream_t s,
                               cudaStream_t ps, cudaEvent_t pev) {
  counted();
  const int vec_ok = ((((uintptr_t)w) | ((uintptr_t)mom) | ((uintptr_t)ring) | slot_bytes |
                       ((uintptr_t)src0) | ((uintptr_t)src1)) & 15) == 0;
  const int V = dtype == 0 ? 4 : 2;
  // programmatic dependent launch: the grid is scheduled while the previous
  // kernel on the stream drains (the kernel's griddepcontrol.wait orders its reads)
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = getenv("EC_NO_PDL") ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // full-occupancy shape: one CTA per 256 vectors (>= 1 CTA for the tail)
  const long long nvv = vec_ok ? n / V : 0;
  cfg.gridDim = dim3((unsigned)((nvv + 255) / 256 > 0 ? (nvv + 255) / 256 : 1));
  cudaError_t e = cudaErrorInvalidValue;
  if (dtype == 0) {
    auto kern = mom ? ec_direct_step_kernel<float, true> : ec_direct_step_kernel<float, false>;
    e = cudaLaunchKernelEx(&cfg, kern, d_desc, seq, flags, (float*)w, (float*)mom, (float)lr,
                           (float)mu, vec_ok, t, timeout_ns);
  } else if (dtype == 1) {
    auto kern = mom ? ec_direct_step_kernel<double, true> : ec_direct_step_kernel<double, false>;
    e = cudaLaunchKernelEx(&cfg, kern, d_desc, seq, flags, (double*)w, (double*)mom, lr, mu,
                           vec_ok, t, timeout_ns);
  }
  if (e != cudaSuccess) return e;
  counted();
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(32);
  if (ps) {
    // the publication (host-visible words behind a system-scope fence, ~4 us)
    // on its own stream: the next step's kernel waits for this one only
    if ((e = cudaEventRecord(pev, s)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(ps, pev, 0)) != cudaSuccess) return e;
    cfg.stream = ps;
    cfg.numAttrs = 0;
  }
  return cudaLaunchKernelEx(&cfg, ec_direct_publish_kernel, d_desc, seq, t);
}

cudaError_t launch_stream_barrier(unsigned long long* count, unsigned long long target,
                                  EcHostCtl* H, unsigned long long timeout_ns, cudaStream_t s) {
  counted();
  ec_stream_barrier_kernel<<<1, 32, 0, s>>>(count, target, H, timeout_ns);
  return cudaGetLastError();
}

cudaError_t launch_write_u64(unsigned long long* p, unsigned long long v, cudaStream_t s) {
  counted();
  ec_write_u64_kernel<<<1, 32, 0, s>>>(p, v);
  return cudaGetLastError();
}

cudaError_t launch_spin(unsigned long long ns, cudaStream_t s) {
  counted();
  ec_spin_kernel<<<1, 32, 0, s>>>(ns);
  return cudaGetLastError();
}
