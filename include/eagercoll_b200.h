/*
 * eagercoll_b200 -- C ABI of the B200-native partial-collective engine
 * (solo / majority / sync allreduce + the eager-SGD fold and update kernels).
 *
 * This is the drop-in boundary.  The reference (arXiv 1908.04207 artifact,
 * /root/reference/pkg/src/eagercoll) is pure Python; its path is reached through
 * `AllreduceHandle` (collectives.py:207-345) sitting on an `Engine`
 * (schedule.py:178-465) that a transport pumps (transport.py:169-320).  Each
 * entry point below replaces one reference operation, cited per function.
 * The Python host package (paper_1908_04207_b200/) binds these with ctypes;
 * INTEGRATION.md shows the binding.
 *
 * Conventions: plain pointers and sizes only; device pointers are CUDA device
 * addresses; `stream` is a cudaStream_t passed as void* (NULL = legacy default
 * stream).  Every function returns 0 on success or a negative EC_E* code, with a
 * thread-local message in ec_last_error().  Element types: EC_F32 (the product
 * path), EC_F64 and EC_I64 (the reference's "f8"/"i8", collectives.py:40).
 * One ec_comm_t serves the local ranks of one collective instance (`cid`); a
 * process normally holds one local rank per GPU, or all P ranks of an
 * emulated world on one GPU.
 */
#ifndef EAGERCOLL_B200_H
#define EAGERCOLL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* element types (collectives.py:40 _ELEMENTS, plus fp32) */
enum { EC_F32 = 0, EC_F64 = 1, EC_I64 = 2 };
/* flavors (collectives.py:37) */
enum { EC_SYNC = 0, EC_SOLO = 1, EC_MAJORITY = 2 };
/* fold modes (eagersgd.py:55-57): COPY = stash was null (0 + grad), ADD = stash + grad */
enum { EC_FOLD_COPY = 0, EC_FOLD_ADD = 1 };
/* contribution flags */
enum {
  EC_CF_FRESH = 1,      /* set this rank's flag bit (collectives.py:304-306) */
  EC_CF_ACTIVATE = 2,   /* activate after an accepted offer (eagersgd.py:162-163) */
  EC_CF_ALL_ARRIVE = 4, /* bench: activate only once every rank has boarded */
};
/* request replies */
enum {
  EC_R_PENDING = 0, EC_R_ACCEPTED = 1, EC_R_REFUSED = 2, EC_R_OK = 3,
  EC_R_POISONED = 4, EC_R_ERROR = 5
};
/* error codes */
enum {
  EC_OK = 0, EC_E_ARG = -1, EC_E_CUDA = -2, EC_E_TIMEOUT = -3, EC_E_STATE = -4,
  EC_E_ORDER = -5, EC_E_DEVICE = -6, EC_E_NOMEM = -7
};

typedef struct ec_comm ec_comm_t;

/* Library identity and the thread-local message of the last failing call
 * (no reference counterpart: the reference raises Python exceptions,
 * collectives.py:51-59, schedule.py:38-55). */
int ec_version(void);
const char* ec_last_error(void);
/* Number of kernels this library has launched in the process (instrumentation;
 * no reference counterpart). */
uint64_t ec_launch_count(void);

/* ---- communicator lifecycle ------------------------------------------------
 * Replaces AllreduceHandle.__init__ + Engine(...) + commit()
 * (collectives.py:218-235, schedule.py:186-273) for ranks
 * [rank_lo, rank_lo + n_local) of a world of `world_size`.  Allocates per local
 * rank: the peer-visible control block, the send/stash buffer (n_elems), a ring
 * of `ring_slots` result slots, host-mapped request/reply/log pages.
 * workers_per_rank = worker CTAs of the persistent engine per rank (0 = auto). */
int ec_comm_create(int world_size, int rank_lo, int n_local, int device,
                   int64_t n_elems, int dtype, int flavor, int ring_slots,
                   int workers_per_rank, ec_comm_t** out);
/* CUDA IPC handles of local rank `local_idx`'s buffers, for exchange over the
 * process group at init (replaces transport.register_engine, transport.py:205-214). */
int ec_comm_export(ec_comm_t* c, int local_idx, void* blob, size_t cap, size_t* len);
/* Map a remote rank's buffers from its exported blob (the peer side of
 * transport.register_engine, transport.py:205-214). */
int ec_comm_import(ec_comm_t* c, int peer_rank, const void* blob, size_t len);
/* Majority with a quorum (opt-in extension; the reference's rule, the default
 * 0, activates at the designated initiator's arrival without counting,
 * collectives.py:311-317): the initiator_for_round rank activates only once
 * at least `min_arrivals` ranks (ceil(P/2) for "at least half", the
 * north_star's phrasing) have boarded the generation.  Before ec_comm_start. */
int ec_comm_set_quorum(ec_comm_t* c, int min_arrivals);
/* Replay mode: force generation g's inclusion mask to masks[g] (g < n) --
 * participation recorded from a reference run, so the
 * snapshot decisions of collectives.py:146-153 are reproduced exactly. */
int ec_comm_set_replay(ec_comm_t* c, int local_idx, const uint64_t* masks, int64_t n);
/* NVLS ("fast" reduction mode, fp32, one rank per GPU; no reference
 * counterpart -- CollectiveConfig.reduction_mode is an extension): the NVSwitch reduces.
 * One rank ec_nvls_create()s the multicast object and shares the fabric-handle
 * blob; every rank ec_nvls_attach()es it (the creator passes NULL); after all
 * ranks attached, every rank ec_nvls_bind()s its memory, which also switches the
 * data phase to multimem.ld_reduce / multimem.st.  Summation order inside the
 * switch is unspecified: never bit-exact, within fp32 rounding of the sum. */
int ec_nvls_supported(int device);
int ec_nvls_create(ec_comm_t* c, void* blob, size_t cap, size_t* len);
int ec_nvls_attach(ec_comm_t* c, const void* blob, size_t len);
int ec_nvls_bind(ec_comm_t* c);
/* Start (or resume) the persistent engine kernel on the comm's own stream: the
 * device form of the engine's pump (schedule.py:346-465, driven by
 * transport.py:233-317 in the reference). */
int ec_comm_start(ec_comm_t* c);
/* Drain and stop the engine at a round boundary so device-wide syncs return;
 * ec_comm_start resumes it with all protocol state preserved. */
int ec_comm_pause(ec_comm_t* c, int timeout_ms);
/* Idle park (no reference counterpart; the simulator has no resident kernel):
 * after EC_IDLE_PARK_MS (default 100, 0 = never) with no API call and no
 * completed round, and nothing outstanding, a library thread parks the
 * engine so device-wide syncs in user code (torch.cuda.synchronize,
 * cudaFree) return; the next post relaunches it, and for remote peers the
 * thread relaunches it when a peer activates, snapshots or boards the next
 * generation.  Counters of parks / wakes and whether it is parked now. */
int ec_comm_idle_stats(ec_comm_t* c, uint64_t* parks, uint64_t* wakes, int* parked);
/* Bytes local rank `local_idx`'s workers have pulled from (rx) and pushed to
 * (tx) OTHER ranks' memory since creation, in the fused TMA data phases: the
 * NVLink traffic the engine issues (no reference counterpart; the hardware's
 * NVLink byte counters are not exposed on every platform).  Two-shot rounds
 * issue (P-1)/P * S each way per rank, 2(P-1)/P * S in all = the bus bytes. */
int ec_comm_traffic(ec_comm_t* c, int local_idx, uint64_t* rx_bytes, uint64_t* tx_bytes);
/* %globaltimer stamps of async step t (one of the last 64; instrumentation,
 * no reference counterpart): t4 = {its update kernel's report, its fold/post
 * kernel's start, that kernel's post, the controller seeing the offer} --
 * the step boundary between one round's completion and the next offer. */
int ec_step_times(ec_comm_t* c, int local_idx, int64_t t, uint64_t* t4);
/* Checked build (EC_DEBUG) diagnostics: the controller's last 16 loop-iteration
 * start stamps when it saw step t's offer (one of the last 8 steps), then
 * 16 x 4 section stamps of those iterations (t16 holds 80 words); zeros in
 * the production build.  No reference counterpart. */
int ec_step_iterations(ec_comm_t* c, int local_idx, int64_t t, uint64_t* t16);
int ec_comm_destroy(ec_comm_t* c);
/* Device error word (watchdog timeout, out-of-order round): the reference's
 * TimeoutError / AssertionError (collectives.py:298,331). */
int ec_comm_error(ec_comm_t* c, int local_idx, uint64_t* code, uint64_t* info);
/* Diagnostics snapshot of a local rank's engine (16 int64 words, see ec_host.cu;
 * no reference counterpart). */
int ec_debug_state(ec_comm_t* c, int local_idx, int64_t* out16);

/* device addresses of the local rank's send buffer (the stash / send buffer,
 * eagersgd.py:68, collectives.py:301-303), its registered gradient buffer
 * (write the gradient here and pass it to ec_step_async: while the stash is
 * null the reduction reads it in place, no fold) and result slot `gen % R`
 * (the recv buffer, schedule.py:382-390) */
void* ec_send_ptr(ec_comm_t* c, int local_idx);
void* ec_grad_ptr(ec_comm_t* c, int local_idx);
void* ec_slot_ptr(ec_comm_t* c, int local_idx, int64_t gen);
int64_t ec_n_elems(ec_comm_t* c);
/* 1 when ec_step_async updates progressively: the step's update kernel applies
 * eagersgd.py:165 to each chunk of the round's result as it lands (owners
 * publish per-chunk-group arrival words), overlapping the NVLink-bound round */
int ec_comm_progressive(ec_comm_t* c);
/* enqueue a device-side barrier across all ranks of the communicator on
 * `stream` (a one-thread kernel: system-scope arrival count in rank 0's
 * control block).  Every rank must call it the same number of times.  Used to
 * align the start of timed regions; no reference counterpart (the simulator
 * has one clock). */
int ec_stream_barrier(ec_comm_t* c, int local_idx, void* stream);
/* resume from a checkpoint (extending eagersgd.py:281-299's
 * EGW1): re-base a parked rank so its next round is `gen`, with its stash
 * holding an offer (`stash_pending`) or null, and `contributed_round` as the
 * staleness guard's last contribution.  Every rank resumes at the same gen. */
int ec_comm_set_generation(ec_comm_t* c, int local_idx, int64_t gen, int stash_pending,
                           int64_t contributed_round);

/* ---- application protocol -------------------------------------------------
 * GradientBuffer.fold (eagersgd.py:55-57) into the send buffer, stream-ordered.
 * Non-finite gradients set a poison flag that the next post turns into
 * EC_R_POISONED (train_step's DivergenceError, eagersgd.py:145-147). */
int ec_fold(ec_comm_t* c, int local_idx, const void* grad, int mode, void* stream);
/* np.copyto(send, vec) of try_contribute (collectives.py:301-303), stream-ordered. */
int ec_copy_in(ec_comm_t* c, int local_idx, const void* src, void* stream);
/* try_contribute(t, ..., fresh) [+ activate(t)] (collectives.py:291-317), posted
 * in stream order after the fold/copy; *seq identifies the reply. */
int ec_post_contribute(ec_comm_t* c, int local_idx, int64_t t, uint32_t flags,
                       void* stream, uint64_t* seq);
/* activate(t) (collectives.py:311-317), posted from the host. */
int ec_post_activate(ec_comm_t* c, int local_idx, int64_t t, uint64_t* seq);
/* staleness guard (eagersgd.py:89-110): generations >= hold_from are held
 * until this rank contributes; INT64_MAX disables. */
int ec_post_hold(ec_comm_t* c, int local_idx, int64_t hold_from, uint64_t* seq);
/* staleness_guard (eagersgd.py:89-110) with the ages tracked on the device,
 * so every step path -- including the stream-ordered ec_step_async -- is
 * guarded without a host round trip: generation g is held until this rank
 * contributes when g >= min(oldest round still pending in the stash, the
 * round after the last offer) + tau (eagersgd.py:102-108).  tau < 0 turns it
 * off; pending_lo >= 0 seeds the oldest pending round (e.g. after a resume). */
int ec_post_guard(ec_comm_t* c, int local_idx, int64_t tau, int64_t pending_lo, uint64_t* seq);
/* Reply to request `seq` (EC_R_*), waiting up to timeout_ms (0 = poll once):
 * try_contribute's bool (collectives.py:291-309). */
int ec_reply(ec_comm_t* c, int local_idx, uint64_t seq, int timeout_ms, int* status);
/* done_generation (collectives.py:278-289); -1 before the first round. */
int ec_done_gen(ec_comm_t* c, int local_idx, int64_t* gen);
/* wait_done / wait_blocking (collectives.py:319-332): block until a generation
 * >= t completed, return the latest one with its mask and nap.  pin != 0 pins
 * its result slot against reuse until ec_set_pin releases it. */
int ec_wait(ec_comm_t* c, int local_idx, int64_t t, int timeout_ms, int pin,
            int64_t* gen, uint64_t* mask, int* nap);
/* call_round in one call (collectives.py:334-345): ec_post_contribute(t, flags)
 * + ec_reply + ec_wait(t, unpinned).  *status is the offer's reply. */
int ec_round(ec_comm_t* c, int local_idx, int64_t t, uint32_t flags, void* stream,
             int timeout_ms, int* status, int64_t* gen, uint64_t* mask, int* nap);
/* call_round (collectives.py:334-345) offered in stream order with a
 * stream-ordered wait for its completion behind it: back-to-back rounds with no
 * host round trip (bandwidth sweeps). */
int ec_round_async(ec_comm_t* c, int local_idx, int64_t t, uint32_t flags, void* stream,
                   uint64_t* seq);
/* One eager-SGD step of the hot path in one call (eagersgd.py:129-167):
 * fold grad into the stash (fold_mode, skipped if grad is NULL), offer it
 * (flags), wait for the latest generation >= t (pinned), w = w - lr*u (or the
 * momentum form when mom != NULL and mu != 0), release the pin in stream order.
 * *status = the offer's reply; on EC_R_POISONED nothing else happens. */
int ec_step(ec_comm_t* c, int local_idx, int64_t t, const void* grad, int fold_mode,
            uint32_t flags, void* w, void* mom, double lr, double mu, void* stream,
            int timeout_ms, int* status, int64_t* gen, uint64_t* mask, int* nap);
/* The same step with no host round trip (stream-ordered, returns at once):
 * fold with the mode the device's stash state dictates (null stash: 0 + g),
 * post the offer, wait ON THE DEVICE for a generation >= t and pin it, update
 * from that slot, unpin.  The host reads the outcome later with
 * ec_step_result(seq, t); steps must be issued in order.  The device-side
 * wait occupies `stream`: ranks sharing one GPU need distinct streams.  Not
 * capturable: under stream capture it returns EC_E_STATE (each step's launch
 * arguments carry a fresh request sequence number). */
int ec_step_async(ec_comm_t* c, int local_idx, int64_t t, const void* grad, uint32_t flags,
                  void* w, void* mom, double lr, double mu, void* stream, uint64_t* seq);
/* The outcome of an ec_step_async step: what train_step returns
 * (eagersgd.py:166-167: the offer's reply, the generation applied, its mask
 * and nap). */
int ec_step_result(ec_comm_t* c, int local_idx, uint64_t seq, int64_t t, int timeout_ms,
                   int* status, int64_t* gen, uint64_t* mask, int* nap);
/* Instrumentation (no reference counterpart): with profiling on, ec_step brackets its fold and update
 * launches with CUDA events; ec_profile_read sums the durations
 * (ms_sum[0]/counts[0] = fold, [1] = update) and clears the record. */
int ec_profile_enable(int on);
/* %globaltimer duration of the update of the last step reconciled by
 * ec_step_result (from the device wait's release to the last CTA). */
int ec_step_update_ns(ec_comm_t* c, int local_idx, uint64_t* ns);
int ec_profile_read(double* ms_sum2, int64_t* counts2);
/* Mask / nap of an earlier generation from the device log: CollectiveResult's
 * included / nap (collectives.py:70-75, 254-274), the RoundRecord source
 * (trace.py:15-45). */
int ec_gen_info(ec_comm_t* c, int local_idx, int64_t gen, uint64_t* mask,
                uint64_t* has_data, int* nap);
/* Device timestamps (%globaltimer ns) of a completed generation at this rank
 * (the timing behind LatencyRecord, trace.py:38-45):
 * t5 = {snapshot taken, reduction issued (all snapshots in), own data phase
 * done, published, own offer processed (0 if none)}. */
int ec_gen_times(ec_comm_t* c, int local_idx, int64_t gen, uint64_t* t5);
/* Result-slot pin (no reference counterpart: the reference copies u out,
 * collectives.py:260; here slots are read in place).
 * Lowest generation the host may still read: the engine never overwrites the
 * slot of generation h unless h < pin_lo.  ordered != 0 performs the store in
 * `stream` order (release after the update kernel read the slot); ordered == 0
 * stores from the host immediately. */
int ec_set_pin(ec_comm_t* c, int local_idx, uint64_t pin_lo, int ordered, void* stream);

/* ---- standalone sm_100a kernels (no communicator) --------------------------- */
/* stash (+)= grad: mode COPY writes 0+grad, ADD writes stash+grad (eagersgd.py:56). */
int ec_fold_raw(void* stash, const void* grad, int64_t n, int dtype, int mode,
                uint32_t* nonfinite_flag, void* stream);
/* w = w - lr*u, two roundings, no FMA (eagersgd.py:165). */
int ec_sgd_update(void* w, const void* u, double lr, int64_t n, int dtype, void* stream);
/* buf = mu*buf + u ; w = w - lr*buf: the opt-in momentum form of
 * eagersgd.py:165 (the reference is plain SGD; mu == 0 is it). */
int ec_momentum_update(void* w, void* buf, const void* u, double lr, double mu,
                       int64_t n, int dtype, void* stream);
/* tree_order_sum (collectives.py:385-403) of p device vectors in the engine's
 * snapshot semantics (0+x leaves, has_mask bit clear = null), optionally / p
 * (collectives.py:254-260).  srcs is a HOST array of p device pointers. */
int ec_local_reduce(const void* const* srcs, int p, uint64_t has_mask, void* dst,
                    int64_t n, int dtype, int divide, void* stream);
/* Device-side imbalance injection (transport.py:137-149): spin for ns. */
int ec_spin(uint64_t ns, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* EAGERCOLL_B200_H */
