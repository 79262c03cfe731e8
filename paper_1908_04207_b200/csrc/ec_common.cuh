// Shared layouts and PTX helpers of the eagercoll_b200 engine (sm_100a).
//
// Memory map per rank:
//   EcCtrl     device memory, IPC-mapped by every peer.  Peers WRITE their
//              per-source words here (activation, snapshot, shard-ready,
//              arrival), so every wait is a poll of local HBM/L2.
//   EcLocal    device memory, private to the rank's engine CTAs (round command,
//              worker counters, controller state saved across pause/resume).
//   EcHostCtl  pinned, host-mapped: request ring (host/stream -> engine),
//              replies, done generation and per-generation mask log
//              (engine -> host), pin and stop words (host -> engine).
//   send       the rank's contribution / eager-SGD stash (n elements).
//   ring       R result slots of n elements; slot g % R holds u of generation g.
#pragma once
#include <assert.h>
#include <stdint.h>

// Device-side invariant checks of the checked build (-DEC_DEBUG, build.py
// --debug): a failed check traps the kernel with file:line.  Free otherwise.
#ifdef EC_DEBUG
#define EC_ASSERT(x) assert(x)
#else
#define EC_ASSERT(x) ((void)0)
#endif

#define EC_MAX_P 64
#define EC_REQ_RING 1024
#define EC_LOG_RING 4096
#define EC_INF_GEN 0x7fffffffffffffffLL

// request types
#define EC_REQ_CONTRIB 1
#define EC_REQ_ACTIVATE 2
#define EC_REQ_HOLD 3
// staleness guard with device-tracked ages (eagersgd.py:89-110): arg = tau
// (< 0 disables), t = the lowest pending round to seed (< 0: none)
#define EC_REQ_GUARD 4
// internal contribution flag (set by the post kernel from the fold's poison word)
#define EC_CF_POISON 0x100

// snapshot word: ((gen+1) << 4) | upd << 3 | src_grad << 2 | has_data << 1 | fresh
#define EC_SNAP_FRESH 1ull
#define EC_SNAP_DATA 2ull
#define EC_SNAP_SRC_GRAD 4ull   // the offer is the registered gradient buffer, not the stash
#define EC_SNAP_UPD 8ull        // this rank updates progressively: owners publish arrival words
#define EC_SNAP_SHIFT 4
// contribution flag: the offer's step update kernel follows it on the stream and
// consumes the round's chunks as they land (owners publish arrival words)
#define EC_CF_STEP 32u
// internal: a host-posted request the engine's poller copied into the device ring
#define EC_CF_HOSTPOSTED 0x200u
// arrival words: owner worker (q, w) publishes ((gen+1) << 24) | chunks landed
#define EC_PROG_W 128
#define EC_PROG_SHIFT 24
// contribution flag: offer the registered gradient buffer (zero-copy, stash null)
#define EC_CF_SRC_GRAD 8u
// direct mode: offer the gradient buffer iff the stash is still null at decision time
#define EC_CF_SRC_GRAD_AUTO 16u
// done word: gen + 1, top bit = a reduced value of this owner's shard was non-finite
#define EC_DONE_POISON (1ull << 63)

// device error codes (EcHostCtl::error)
#define EC_DERR_ORDER 1      // contribution for a future generation
#define EC_DERR_TIMEOUT 2    // watchdog expired inside a round
#define EC_DERR_REPLAY 3     // replay table exhausted / inconsistent

struct alignas(128) EcCtrl {
  unsigned long long act_from[EC_MAX_P];     // gen+1 activated by source rank
  unsigned long long snap_from[EC_MAX_P];    // snapshot word of source rank
  unsigned long long rsdone_from[EC_MAX_P];  // gen+1: source's reduced shard ready
  unsigned long long arrive_from[EC_MAX_P];  // gen+1: source boarded (all-arrive)
  unsigned long long done_from[EC_MAX_P];    // gen+1: source's data for gen is in our slot
  unsigned long long staged_from[EC_MAX_P];  // gen+1: source staged its offer (NVLS mode)
  // fused updates: owner q's worker w has stored its first k chunks of
  // generation g into our slot when prog[q][w] >= ((g+1) << 24) | k
  unsigned long long prog[EC_MAX_P][EC_PROG_W];
  unsigned long long bar_count;   // rank 0's copy: stream-barrier arrivals (monotone)
  unsigned long long pad_bar[15];
};

struct alignas(64) EcReq {
  unsigned long long seq1;   // request sequence + 1; written last (release)
  unsigned int type;
  unsigned int flags;
  long long t;
  long long arg;
  unsigned long long pad[4];
};

// one round command (controller -> workers); command s (s = 1, 2, ...) sits in
// EcLocal::cmd[(s - 1) & 3] -- up to EcDesc::lead rounds are in flight
struct EcCmd {
  long long gen;
  unsigned long long has;          // has-data mask of the round
  unsigned long long src;          // ranks whose offer is their gradient buffer
  unsigned long long updm;         // ranks updating progressively (owners signal arrivals)
  int wact;                        // worker CTAs the round uses (<= EcDesc::W)
  int pad;
};

struct alignas(128) EcLocal {
  // round commands: controller -> workers
  unsigned long long cmd_seq;      // commands issued (monotone)
  unsigned long long exit_epoch;   // workers of launch `epoch` exit when this equals it
  unsigned long long pad0[6];
  EcCmd cmd[4];
  unsigned long long rs_count;     // worker CTAs finished reduce-scatter (monotone)
  unsigned long long pad1[7];
  // worker CTAs finished command s, counted in ag_cnt[(s - 1) & 3] (monotone)
  unsigned long long ag_cnt[4];
  unsigned long long t_rs4[4];     // globaltimer when command s's last worker finished
  unsigned int rpoison[4];         // command s's CTAs saw a non-finite reduced value
  unsigned long long pad2[2];
  unsigned long long round_done;   // last cmd_seq fully done
  unsigned long long pad3[7];
  // controller state (persisted across pause/resume)
  long long g;                     // current generation
  long long hold_from;
  long long contributed_round;
  unsigned long long next_req;
  int snapped;
  int contrib;                     // EC_SNAP_* bits of the accepted offer
  int internal_act;
  int arrive_pending;              // all-arrive: activate once everyone boarded
  int arrive_activate;
  int initialized;
  unsigned long long t_snap;       // globaltimer at this generation's snapshot
  unsigned long long t_rs;         // globaltimer when the last worker finished its shard
  unsigned int poison;             // fold's non-finite flag (device word)
  int pad4;
  unsigned long long posted;       // doorbell: highest stream-posted request seq + 1
  unsigned long long done_gen1_dev;  // device mirror of EcHostCtl::done_gen1 (async steps)
  long long step_gen;              // generation the current async step's update reads
  int stash_null;                  // 1: the stash holds no pending gradient (fold writes 0+g)
  int pad5;
  unsigned long long fold_count;   // CTAs of the fused fold+post kernel done (last one posts)
  unsigned long long upd_count;    // CTAs of the fused wait+update kernel done (last one unpins)
  unsigned long long step_tag;     // t + 1 once step_gen holds step t's generation
  unsigned long long upd_t0;       // globaltimer when the fused update's compute began
  unsigned long long req_done_dev; // requests the controller has processed (device mirror)
  int late_copy;                   // a zero-copy offer was refused: copy gbuf -> stash
  int step_late;                   // latched late_copy for the current async step's update
  unsigned int pad_rp;
  unsigned int upd_bad;            // the async step's update read a non-finite u
  unsigned long long pin_dev;      // device-side pin (async steps): lowest gen still read
  unsigned long long stage_count;  // NVLS: CTAs that staged this round (monotone)
  unsigned long long dec_tag;      // direct step: seq + 1 once block 0 decided the step's offer
  unsigned long long dec_status;   // direct step: the decision's reply status
  int dec_fold;                    // direct step: fold the gradient into the stash in-pass
  int pad7;
  unsigned long long fuse_seq;     // request seq + 1 of the last offer accepted with arrival words
  int step_fused;                  // the current async step updates progressively (arrival words)
  int pad8;
  unsigned long long upd_next_item;  // progressive update: next chunk item to claim
  // direct step seq's report, by seq % EC_REQ_RING: written by the step's
  // block 0 (and its CTAs' finiteness bits), read by the publication kernel,
  // which may run after the next step already decided (its own stream)
  struct {
    unsigned long long status, t0;
    int contrib;
    unsigned int fused, bad, pad;
  } drep[EC_REQ_RING];
  // async step t's report (P > 1), by t % EC_REQ_RING: written by the update
  // kernel's last CTA, made host-visible by ec_step_publish_kernel on the
  // rank's publication stream
  struct {
    unsigned long long ns;
    unsigned int bad, pad;
  } srep[EC_REQ_RING];
  // host poller (engine thread 32): mirrors of host-mapped words, so the
  // controller thread never stalls on a PCIe read
  unsigned long long hp_seq;       // changes of the mirrored host pin (monotone)
  unsigned long long hp_lo;        // mirrored host pin (EcHostCtl::pin_lo)
  unsigned long long hp_ps;        // the pin_seq it was read with (acknowledged)
  unsigned long long hp_stop;      // epoch whose stop request the poller saw (0: none)
  unsigned long long hp_stop_kind; // 1 = explicit pause, 2 = idle park (only when idle)
  unsigned long long park_votes;   // rank_lo's copy: local controllers agreeing to an idle park
  // staleness guard (controller-owned, persisted across pause/resume): a
  // generation g is held until this rank contributes when
  // g >= min(pend_lo, last_off + 1) + guard_tau -- the oldest gradient not yet
  // delivered (a pending stash round, or the step in progress after the last
  // offer), eagersgd.py:102-108
  // %globaltimer stamps of async step t (slot t % 64): its update kernel's
  // report, the next fold/post kernel's start and its post (step timeline)
  unsigned long long tl[64][4];    // [3]: the controller saw the step's offer
  // checked build only: the controller's last 16 iteration starts when it saw
  // step t's offer (tl_it[t % 8]), for the step-boundary study
  unsigned long long tl_it[8][16];
  unsigned long long tl_sec[8][16][4];   // section stamps of those iterations
  unsigned long long nv_rx, nv_tx; // bytes this rank's workers pulled from / pushed to other
                                   // ranks (fused TMA modes; monotone, ec_comm_traffic)
  long long guard_tau;             // EC_INF_GEN: guard off
  long long pend_lo;               // oldest offered round still in the stash (EC_INF_GEN: none)
  long long last_off;              // round of the last offer processed (-1: none yet)
  EcReq dreq[EC_REQ_RING];         // stream-posted requests (device copy of the ring)
};



struct alignas(64) EcLog {
  unsigned long long gen1;
  unsigned long long mask;
  unsigned long long has;
  unsigned long long nap;
  // %globaltimer (ns) of this rank's engine: snapshot taken, round command
  // issued (all snapshots in), own shard reduced, round published
  unsigned long long t_snap, t_cmd, t_rs, t_done;
  unsigned long long t_req;        // this rank's offer for the generation was processed
  unsigned long long poison;       // some owner reduced a non-finite value in this generation
  unsigned long long pad[2];
};

struct alignas(128) EcHostCtl {
  unsigned long long stop;          // host -> engine: 1 drain and exit, 2 exit if idle (idle park)
  unsigned long long pin_lo;        // host -> engine: lowest generation the host still reads
  unsigned long long pin_seq;       // host -> engine: bumped with every host pin
  unsigned long long pin_ack;       // engine -> host: last pin_seq the controller has seen
  unsigned long long pad0[12];
  unsigned long long done_gen1;     // engine -> host: last completed generation + 1
  unsigned long long req_done;      // engine -> host: requests consumed
  unsigned long long error;
  unsigned long long error_info;
  unsigned long long exited;        // engine -> host: controller parked (pause ack)
  unsigned long long snap_gen1;     // engine -> host: last snapshotted generation + 1
  unsigned long long pad1[10];
  EcReq req[EC_REQ_RING];
  unsigned long long reply[EC_REQ_RING];   // ((seq+1) << 8) | status
  unsigned long long stepgen[EC_REQ_RING]; // async step t: generation its update read, + 1
  unsigned long long steptag[EC_REQ_RING]; // t + 1 once stepgen[t % RING] is valid
  unsigned long long stepns[EC_REQ_RING];  // async step t: update compute duration (ns)
  unsigned long long stepbad[EC_REQ_RING]; // async step t: u had a non-finite element
  EcLog log[EC_LOG_RING];
};

struct EcDesc {
  int rank, P, flavor, dtype;
  int R, W, replay, vec;              // ring slots, worker CTAs, replay flag, elems / 16 B
  int w_step;                         // worker CTAs of a round with progressive step updates
  unsigned idle_sleep_ns;             // controller's back-off cap with nothing in flight
  int quorum;                         // majority: arrivals the initiator waits for (0: none,
                                      // the reference's rule, collectives.py:311-317)
  int lead;                           // rounds the engine may have in flight (1, or 2: the
                                      // next round's snapshot overlaps the current data phase)
  int mode;                           // data phase: 0 = fused TMA two-shot, 1 = two-phase ld.cg
                                      // pull, 2 = NVLS (multimem.ld_reduce / multimem.st, fast
                                      // mode), 3 = fused TMA one-shot (small messages)
  int chv, stages;                    // TMA chunk (16-B vectors) and pipeline depth
  int sig_every;                      // chunks per arrival word (progressive updates; 0 = ~4/round)
  int smem_bytes;
  long long n, nvec;                  // elements, whole 16-B vectors
  long long slot_bytes;
  long long n_forced;
  unsigned long long timeout_ns;      // in-round watchdog
  EcCtrl* ctrl[EC_MAX_P];
  char* send[EC_MAX_P];
  char* ring[EC_MAX_P];
  char* gbuf[EC_MAX_P];               // registered gradient buffers (zero-copy offers)
  char* mc_stage;                     // NVLS: multicast view of the staging region
  char* mc_ring;                      // NVLS: multicast view of the result ring
  char* uc_stage;                     // NVLS: this rank's unicast view of the staging region
  EcHostCtl* hctl;
  EcLocal* local;
  unsigned long long* park_votes;     // &local of rank_lo ->park_votes (shared by the launch)
  int n_local;                        // controllers in this launch
  const unsigned long long* forced;
};

// ----------------------------------------------------------------------------
// PTX helpers.  Cross-GPU and host-visible words use .sys scope; engine-internal
// counters use .gpu scope.  Data moved between rounds is read with ld.cg (L2
// only) so no SM ever serves a stale L1 line of a reused slot.

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_sc_sys() { asm volatile("fence.sc.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_sc_gpu() { asm volatile("fence.sc.gpu;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" :: "l"(p));
}
__device__ __forceinline__ uint4 ld_cg_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_v4(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ uint4 ld_stream_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
