/*
 * lars.h — C ABI of the B200-native LARS gradient-combine-and-update library.
 *
 * The operation (arxiv 1903.12650, /root/reference/PAPER.md):
 *   * data-parallel gradients "are combined to update all the weights"         PAPER.md:29-31 (§I)
 *   * warm-up "which raises learning rate gradually"                           PAPER.md:96-98 (§III-A-1)
 *   * LARS "adjusts the learning rate of each layer according to the norms
 *     weight and gradient"
 *   * decay patterns "step, polynomial, linear"
 *   * "special GPU kernel for batched norm computations"                        PAPER.md:130-135 (§III-B-2)
 *   * gradients "gathered" into multi-megabyte allreduces                       PAPER.md:147-153 (§III-C-1)
 *   * "compute and communicate using half precision ... update own weights
 *     using single precision"; "original optimizer"; warm-up + LARS            PAPER.md:183-185 (§IV)
 *   * 1,280,000 images / 81,920 batch -> 16 updates per epoch, 1,440 in total   PAPER.md:210-211 (§IV)
 *
 * For iteration t (0-based) and every tensor l of the layout (readings in DESIGN.md §Readings):
 *   G      = s * sum_r g_r                                 (s = hp.grad_scale; sum over P ranks)
 *   lr(t)  = base*(t+1)/W  (t < W);  base*((T-t)/(T-W))^p  (W <= t < T)
 *   lambda = eta*||w_l|| / (||G_l|| + beta*||w_l|| + eps)  for weight-kind tensors when ||w_l|| > 0
 *            and the denominator exceeds eps; otherwise 1.  Skip kinds (bias, BN gamma/beta):
 *            lambda = 1, beta_l = 0.
 *   v      <- mu*v + lr(t)*lambda*(G + beta_l*w);   w <- w - v
 *   If any ||w_l|| or ||G_l|| is non-finite the whole step is skipped: w and m are left bitwise unchanged.
 *   The rank sum is a value in the gradient wire dtype (reading #29): an element whose sum
 *   overflows grad_dtype (|sum| >= 65520 for fp16) is infinite, so such a step is skipped too.
 *
 * Conventions for every entry point:
 *   * Pointers named w, g, m are CUDA DEVICE pointers on the handle's device unless the name ends in _host.
 *   * Flat buffers hold `padded_numel` elements (lars_layout); tensor l lives at elements
 *     [offsets[l], offsets[l] + numel_l). Offsets are library-assigned (64-element aligned), so
 *     segments never overlap. Padding elements are never read or written by lars_step.
 *   * w and m are float32 (master weights and momentum); g is hp.grad_dtype.
 *   * Base pointers must be 256-byte aligned, else LARS_ERR_ALIGNMENT.
 *   * The caller owns w, g, m. The library owns its scratch (work lists, LR table, partial norms,
 *     coefficients, status, NCCL communicator) and frees it in lars_destroy.
 *   * Argument errors are returned synchronously before anything is enqueued. Steps never synchronize
 *     the host: numeric overflow is reported through lars_last_step_skipped, not a return code.
 *   * `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   * One handle is driven by one host thread at a time, one in-flight step per handle.
 */
#ifndef LARS_B200_H
#define LARS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LARS_OK = 0,
  LARS_ERR_INVALID_ARG = 1, /* null pointer, bad hyper-parameter, bad rank                         */
  LARS_ERR_LAYOUT = 2,      /* numel <= 0, unknown kind, n <= 0, layout hash differs across ranks   */
  LARS_ERR_ITER_RANGE = 3,  /* iter outside [0, T)                                     */
  LARS_ERR_ALIGNMENT = 4,   /* a base pointer is not 256-byte aligned                               */
  LARS_ERR_CUDA = 5,        /* a CUDA runtime call failed                                           */
  LARS_ERR_NCCL = 6,        /* an NCCL call failed                                                  */
  LARS_ERR_OOM = 7,         /* device or host allocation failed                                     */
  LARS_ERR_NO_COMM = 8,     /* dp step before lars_comm_init (or no fused/half-weight buffers)      */
  LARS_ERR_NO_DEVICE = 9    /* a device operation on a host-only (device = -1) handle               */
} lars_status_t;

/* Per-tensor kind (SPEC.md:33-36 ParamSegment.kind; reading #4). */
typedef enum {
  LARS_KIND_WEIGHT = 0,   /* conv / fc weights: LARS trust ratio + weight decay */
  LARS_KIND_BIAS = 1,     /* skip kinds: lambda = 1, no weight decay            */
  LARS_KIND_BN_GAMMA = 2,
  LARS_KIND_BN_BETA = 3
} lars_kind_t;

/* How the flat layout is split into P rank shards (hp.shard_policy). */
typedef enum {
  LARS_SHARD_CONTIGUOUS = 0, /* default: layout order, equal shards, <= P-1 layers straddle shard
                                boundaries (their norms are completed across ranks); the flat layout
                                (offsets) is the same for every P                                      */
  LARS_SHARD_LPT = 1,        /* whole layers bin-packed (longest processing time): no layer spans ranks,
                                offsets depend on P, padding grows when one layer exceeds ~N/P          */
  LARS_SHARD_GROUPS = 2      /* static backward-order groups (§III-C-2: "we statically
                                group layers into several groups beforehand"; sized "several megabytes",
                                PAPER.md:153): walking the tensors from last to first (the order backward
                                produces them), a group closes when its gradient bytes first reach
                                hp.group_bytes; the remaining tensors form the residual group. Every
                                group's flat span is padded to a multiple of 64*P elements and cut into P
                                equal slices; rank r owns slice r of EVERY group, so each group is
                                reduce-scattered on its own as soon as backward has produced it
                                (dp_group_ready) while the rest of backward runs. NCCL path only.       */
} lars_shard_policy_t;

/* Gradient wire dtype: fp16 is the paper's; bf16 optional; fp32 allowed. */
typedef enum { LARS_F32 = 0, LARS_F16 = 1, LARS_BF16 = 2 } lars_dtype_t;

typedef struct {
  int64_t numel;  /* > 0 */
  int32_t kind;   /* lars_kind_t */
  int32_t fan_in; /* fan-in of a weight-kind layer for lars_init_weights (0: numel); else unused */
} lars_tensor_t;

typedef struct {
  double base_lr;        /* REQUIRED, > 0: the paper gives no value (reading #9)                 */
  double eta;            /* LARS trust coefficient (default 1e-3, reading #5/#10)                 */
  double momentum;       /* mu in [0, 1) (default 0.9)                                            */
  double weight_decay;   /* beta >= 0, weight-kind tensors only (default 5e-5)                    */
  double eps;            /* trust-ratio denominator guard >= 0 (default 0)                        */
  double warmup_epochs;  /* W = round-half-up(warmup_epochs * ipe) iterations (default 5)         */
  double poly_power;     /* p >= 0 (p = 1 linear, p = 0 constant; default 2)                       */
  double grad_scale;     /* s: G = s * sum_r g_r (default 1.0; e.g. 1/(P*loss_scale)); finite,
                          * nonzero, |s| <= 2^64, else lars_init returns LARS_ERR_INVALID_ARG    */
  int64_t global_batch;  /* B > 0 (default 81,920)                                    */
  int64_t dataset_size;  /* D > 0 images per epoch (default 1,280,000)               */
  int32_t total_epochs;  /* E > 0 (default 90)                                   */
  int32_t grad_dtype;    /* lars_dtype_t of g                                                     */
  int32_t nranks;        /* data-parallel world size P the layout is planned for (default 1)       */
  int32_t tile_elems;    /* minimum work-tile size in elements; 0 = library default                */
  int32_t shard_policy;  /* lars_shard_policy_t (default LARS_SHARD_CONTIGUOUS)                    */
  uint32_t flags;        /* LARS_FLAG_* (default 0)                                               */
  int32_t buckets;       /* NCCL path, P > 1: K >= 2 splits every shard into K tile-aligned buckets;
                            reduce-scatter bucket k (grouped ncclReduce, one per root) overlaps the
                            norms of bucket k-1, and the update of bucket k overlaps the weight
                            broadcast of bucket k-1 ("several megabytes"). 0/1 =
                            one ncclReduceScatter + one ncclAllGather (default)                    */
  int32_t decay;         /* lars_decay_t after the warm-up (default LARS_DECAY_POLY)              */
  int32_t n_milestones;  /* LARS_DECAY_STEP: number of milestones (0..8)                          */
  int32_t reserved;      /* must be 0                                                             */
  double step_gamma;     /* LARS_DECAY_STEP: factor applied at every milestone (default 0.1)       */
  double milestones[8];  /* LARS_DECAY_STEP: ascending milestones in epochs                        */
  int64_t group_bytes;   /* LARS_SHARD_GROUPS: gradient bytes (grad_dtype) that close a group
                            (default 4 MiB, SPEC.md scheduler default; > 0)                         */
} lars_hparams_t;

/* Learning-rate decay after the warm-up ("step, polynomial, linear"):
 *   LARS_DECAY_POLY: base * ((T - t) / (T - W))^p   (p = 1 linear, p = 0 constant)
 *   LARS_DECAY_STEP: base * step_gamma^k, k = number of milestones M_j = round(milestones[j] * ipe) <= t */
typedef enum { LARS_DECAY_POLY = 0, LARS_DECAY_STEP = 1 } lars_decay_t;

/* Carry the weight norms: K2 also produces sum(w_new^2) for every layer, so the next step's K1 reads only
 * g (8 -> 4 B/param of norm traffic with fp32 g, 6 -> 2 with fp16). Valid as long as the weights are
 * changed by this handle's steps only: passing a different w pointer invalidates automatically; call
 * lars_invalidate_carried_norms after modifying w in place any other way (e.g. loading a checkpoint). */
#define LARS_FLAG_CARRY_WNORM 1u

/* Momentum form of SPEC.md:186 ("velocity accumulates (grad + wd w) and lr multiplies at application"):
 * v <- mu v + (s g + beta_l w);  w <- w - lr(t) lambda v.   Default (flag clear) is reading #2:
 * v <- mu v + lr(t) lambda (s g + beta_l w);  w <- w - v.  Both agree on a step from v = 0. */
#define LARS_FLAG_LR_AT_APPLY 2u

/* Half-precision compute weights (ZeRO-1 style; "compute and communicate using
 * half precision ... update own weights using single precision"). grad_dtype LARS_F16 or LARS_BF16,
 * contiguous or LPT shards. Each rank keeps fp32 master weights and momentum for ITS SHARD only; the step's
 * all-gather moves the new weights rounded to grad_dtype (round to nearest even) into a library-owned
 * compute-weight buffer (lars_compute_weights), which then holds the full model on every rank, bitwise
 * identical — half the all-gather bytes of the fp32 default. Elements of w outside this rank's shard are
 * neither read nor written (they go stale); read the model from the compute-weight buffer instead. */
#define LARS_FLAG_HALF_WEIGHTS 4u

typedef struct lars_ctx* lars_handle_t;

/* Fills *hp with the defaults listed above (base_lr = 0: the caller must set it). */
void lars_hparams_default(lars_hparams_t* hp);

/* Plans the flat layout (offsets, per-rank shards for hp->nranks, work tiles), the schedule
 * (ipe = ceil(D/B), T = E*ipe, W) and the LR table lr[0..T) in double; uploads them to `device`.
 * device = -1 builds a host-only handle (plan + schedule queries only; no CUDA calls).
 * Errors: LARS_ERR_LAYOUT (n <= 0, numel <= 0, unknown kind), LARS_ERR_INVALID_ARG (bad hp),
 * LARS_ERR_CUDA / LARS_ERR_OOM. No kernel runs. */
lars_status_t lars_init(const lars_tensor_t* tensors, int32_t n, const lars_hparams_t* hp,
                        int32_t device, lars_handle_t* out);

/* offsets[n] (elements) of every tensor in the flat buffers, and the flat length (P * S). Rank r owns
 * elements [r*S, (r+1)*S) (lars_shard_range); see lars_shard_policy_t for how layers map to shards.
 * Either output may be NULL. */
lars_status_t lars_layout(lars_handle_t h, int64_t* offsets, int64_t* padded_numel);

/* Schedule: iterations per epoch, total iterations T, warm-up iterations W. Any output may be NULL. */
lars_status_t lars_schedule(lars_handle_t h, int64_t* ipe, int64_t* total_iters, int64_t* warmup_iters);

/* lr(iter) exactly as the kernels use it (double). LARS_ERR_ITER_RANGE outside [0, T). */
lars_status_t lars_lr_at(lars_handle_t h, int64_t iter, double* lr);

/* Element range [begin, end) of rank `rank`'s shard (P = 1: the whole flat buffer). Under LARS_SHARD_GROUPS
 * a rank's elements are not contiguous (slice r of every group, see lars_groups): LARS_ERR_INVALID_ARG. */
lars_status_t lars_shard_range(lars_handle_t h, int32_t rank, int64_t* begin, int64_t* end);

/* owner[n]: the rank whose shard holds each tensor's first element (a layer that straddles a shard
 * boundary under LARS_SHARD_CONTIGUOUS is updated piecewise by every rank it touches). */
lars_status_t lars_tensor_owner(lars_handle_t h, int32_t* owner);

/* Parallel deterministic initialization (§III-B-1: "every process has the same seed and
 * initializes weights in parallel ... without the broadcast operation"). Fills every layer of w (device, fp32, lars_layout offsets; padding untouched) on `stream`:
 *   weight kind: truncated normal in [-2 sigma, 2 sigma], sigma = sqrt(2 / fan_in) ("truncated_normal",
 *                PAPER.md:268), by inverse CDF: z = sqrt(2) erfinv(2p - 1), p = Phi(-2) + u (1 - 2 Phi(-2));
 *   BN gamma: 1;  BN beta, bias: 0.
 * u = (x >> 11) * 2^-53 with x word (i mod 4) of Philox4x64-10(counter = (i / 4, layer, 0, 0),
 * key = (seed, 0x4C415253)) for element i of layer l: a pure function of (seed, layer, i), so every rank and
 * every launch configuration produces bitwise the same weights with zero communication. */
lars_status_t lars_init_weights(lars_handle_t h, float* w, uint64_t seed, void* stream);

/* Static backward-order groups (LARS_SHARD_GROUPS; any other policy reports ONE group = the whole flat buffer).
 * Group k (k = 0 first: the group backward completes first, i.e. the one holding the LAST tensor) covers flat
 * elements [begin[k], begin[k] + len[k]) and tensors first_tensor[k] .. last_tensor[k] (inclusive, flat
 * order); rank r owns [begin[k] + r*len[k]/P, begin[k] + (r+1)*len[k]/P). Call with NULL arrays to get
 * *ngroups, then with arrays of that many entries (any array may be NULL). */
lars_status_t lars_groups(lars_handle_t h, int32_t* ngroups, int64_t* begin, int64_t* len, int32_t* first_tensor,
                          int32_t* last_tensor);

/* Work decomposition of the single-GPU work list (rank < 0) or of a rank's shard: tiles (= CTAs of K1/K2),
 * segments (pieces of layers inside tiles) and warp chunks. Any output may be NULL. */
lars_status_t lars_work_info(lars_handle_t h, int32_t rank, int32_t* ntiles, int32_t* nsegs, int32_t* nchunks);

/* Verifies the structural invariants of the single-GPU work list (rank < 0) or of a rank's shard that the
 * kernels rely on for in-bounds, race-free access: tiles partition the segments with no empty tile; a tile's
 * chunks fit the kernels' shared-memory partials; every tensor's segments tile exactly its elements on this
 * rank (64-element aligned starts); chunks tile their segment (<= 2,048 elements, 32-byte aligned); nothing
 * lies outside the rank's shard or the flat buffer. LARS_OK, or LARS_ERR_LAYOUT with *reason (static string,
 * may be NULL) naming the violated invariant. Host only; no CUDA calls. */
lars_status_t lars_check_work(lars_handle_t h, int32_t rank, const char** reason);

/* 64-bit FNV-1a hash of (layout, hyper-parameters, P); equal on every rank that planned alike. */
lars_status_t lars_layout_hash(lars_handle_t h, uint64_t* hash);

/* One LARS update of every tensor on one GPU: g is the already-combined gradient (P = 1 semantics,
 * G = s*g). Enqueues the segmented norm kernel (K1: all per-layer ||w||, ||g||, lambda, lr*lambda,
 * non-finite check) and the fused update kernel (K2: unscale + weight decay + momentum + update,
 * streaming w, g, m once) on `stream`; returns without synchronizing. */
lars_status_t lars_step(lars_handle_t h, float* w, const void* g, float* m, int64_t iter, void* stream);

/* lars_step with the iteration in DEVICE memory (an aligned int64): K1 reads *iter_dev and, once every layer
 * has used it, stores *iter_dev + 1 — so one captured CUDA graph replays the whole warm-up + decay schedule
 * (1,440 updates at B = 81,920). An iteration outside [0, T) is reported on the device:
 * the step is skipped and lars_last_step_skipped returns 2. */
lars_status_t lars_step_dev_iter(lars_handle_t h, float* w, const void* g, float* m, int64_t* iter_dev, void* stream);

/* Same as lars_step, but the gradient comes from HOST memory g_host (pinned for async copies,
 * padded_numel elements of grad_dtype): the library copies it into one of two device staging buffers on its
 * own copy stream (ordered before the step on `stream` by an event; the copy for the next call overlaps this
 * step's kernels), runs the step on `stream`, and copies the step status + per-layer norms back into
 * library-owned pinned memory (read them with lars_last_step_skipped / lars_last_norms). g_host must stay
 * unmodified until the step has completed on `stream`. */
lars_status_t lars_step_host_grad(lars_handle_t h, float* w, const void* g_host, float* m,
                                  int64_t iter, void* stream);

/* 128-byte NCCL unique id for lars_comm_init (rank 0 creates it; the caller broadcasts it). */
lars_status_t lars_get_unique_id(void* id128);

/* Creates the NCCL communicator for this handle (nranks must equal hp.nranks, else LARS_ERR_INVALID_ARG),
 * checks that every rank planned the same layout (hash min == max over ranks, else LARS_ERR_LAYOUT), and
 * allocates the reduced-gradient shard buffer (and, when eligible, the fused path's symmetric buffers).
 * nranks = 1 is valid: a one-rank communicator runs every data-parallel kernel and collective on one GPU.
 * Collective: every rank must call it. */
lars_status_t lars_comm_init(lars_handle_t h, int32_t nranks, int32_t rank, const void* id128);

/* Data-parallel step on rank `rank` (P = hp.nranks):
 *   C1 reduce-scatter:  gsum = sum_r g_r over the rank's shard (NCCL, wire dtype, NVLink)
 *   K1 + K2 on the rank's shard only (m is shard-owned: only [begin, end) is read and written)
 *   C2 all-gather:      every rank receives all updated fp32 weights (in place in w)
 * g (the rank's local full gradient) is NOT modified. On completion (stream-ordered) w is bitwise
 * identical on all ranks (with LARS_FLAG_HALF_WEIGHTS: the compute-weight buffers are, and w is current on
 * this rank's shard only). When w and g are the lars_dp_buffers pointers, the fused NVLink kernels replace
 * C1/K1/K2/C2 (same results, fp32 sums). Collective: every rank must call it with the same iter. */
lars_status_t dp_allreduce_lars_step(lars_handle_t h, float* w, const void* g, float* m, int64_t iter,
                                     void* stream);

/* Overlap with backward (LARS_SHARD_GROUPS, NCCL path; "We start to operate allreduce
 * operation for a part of layers without waiting all layers to be finished ... Allreduce operation is
 * scheduled as soon as each process finishes backward processing of all layers in a group").
 * The caller's backward has written every tensor of group `group` into g, ordered on `stream`: the library
 * starts that group's reduce-scatter on its own communication stream (after an event on `stream`) and
 * returns; the remaining backward work on `stream` runs concurrently. Groups must be reported in order
 * 0, 1, 2, ... (every rank then issues the same collective sequence, SPEC.md scheduler) with the same g,
 * else LARS_ERR_INVALID_ARG. The following dp_allreduce_lars_step (same g) issues the groups not reported
 * yet, waits for all of them, and finishes the step; its values do not depend on which groups were
 * reported early. Collective: every rank must report the same groups. */
lars_status_t dp_group_ready(lars_handle_t h, const void* g, int32_t group, void* stream);

/* Overlap trace (instrumentation for benchmarks and the schedule checker): lars_group_trace_enable(h, 1)
 * records timing events around every group's reduce-scatter from the next step on. lars_group_trace_read
 * synchronizes and returns, for the LAST step, milliseconds relative to `ref_event` (a cudaEvent_t created
 * with timing and recorded by the caller, passed as void*; NULL = group 0's ready event): ready[k]
 * (dp_group_ready or, for groups issued by the step itself, the step call), rs_start[k], rs_end[k]
 * (n = ngroups entries each) and *applied (the step's end on the caller's stream). Arrays may be NULL.
 * The overlapped reduce-scatters use a split communicator limited to LARS_GROUP_MAX_CTAS CTAs (env,
 * default 8; 0 = the main communicator) so they take few SMs from the backward kernels they overlap. */
lars_status_t lars_group_trace_enable(lars_handle_t h, int32_t enable);
lars_status_t lars_group_trace_read(lars_handle_t h, void* ref_event, double* ready, double* rs_start, double* rs_end,
                                    double* applied);

/* dp_allreduce_lars_step with the iteration in device memory (see lars_step_dev_iter). */
lars_status_t dp_allreduce_lars_step_dev_iter(lars_handle_t h, float* w, const void* g, float* m, int64_t* iter_dev,
                                              void* stream);

/* Same as dp_allreduce_lars_step with the rank's local gradient in HOST memory g_host (pinned for async
 * copies, padded_numel elements): H2D copy into a library staging buffer, the dp step, then a D2H copy of
 * the step status + per-layer norms into library-owned pinned memory. With w = the lars_dp_buffers weight
 * buffer (fused path) the gradient goes into one of TWO symmetric gradient buffers, alternating per call and
 * copied on the library's copy stream (ordered before the step on `stream` by an event), so the next call's
 * copy overlaps this step; every rank must make the same sequence of calls. Otherwise the copy runs on
 * `stream`. g_host must stay unmodified until the step has completed on `stream`. */
lars_status_t dp_allreduce_lars_step_host_grad(lars_handle_t h, float* w, const void* g_host, float* m,
                                               int64_t iter, void* stream);

/* Per-phase device timing with CUDA events recorded on the step's stream (instrumentation for benchmarks;
 * off by default). lars_profile_enable(h, 1) clears the accumulators and starts recording;
 * lars_profile_enable(h, 0) stops. lars_profile_read synchronizes and returns accumulated milliseconds per
 * phase since enable: ms[0] reduce-scatter (C1), ms[1] norms (K1), ms[2] skip/split allreduce (C3 +
 * finisher), ms[3] update (K2), ms[4] all-gather (C2); single-GPU steps fill ms[1] and ms[3]; the fused
 * data-parallel path fills ms[1] (F1: reduce + norms) and ms[3] (F2: update + gather; the skip/split exchange
 * lives inside F1's tail and F2's head). Profiling records events between the kernels, which suspends the
 * programmatic overlap of F1 and F2: the per-phase sum exceeds an unprofiled step.
 * *steps = steps timed. */
lars_status_t lars_profile_enable(lars_handle_t h, int32_t enable);
lars_status_t lars_profile_read(lars_handle_t h, double* ms, int64_t* steps);

/* The library-owned weight (fp32) and gradient (grad_dtype) buffers of the FUSED data-parallel path:
 * padded_numel elements each, in NCCL symmetric memory (ncclMemAlloc + window registration) so every rank
 * reaches every other rank's buffers over NVLink. When dp_allreduce_lars_step is given exactly these two
 * pointers it runs two kernels instead of NCCL collectives + three kernels: F1 sums this rank's shard of the
 * gradient over all ranks (fp32, rank order, peer loads over NVLink) while computing the layer norms, and its
 * last CTA publishes the skip flag and split-layer sums into every rank's exchange slot; F2 collects them,
 * updates the shard and stores every new weight into every rank's buffer (the all-gather). One LSA barrier
 * at F1's entry (every rank's gradient is complete) and one at F2's exit (every rank's weights are). F1 is a
 * cooperative launch (its CTAs wait for CTA 0's barrier, so the grid is guaranteed co-resident). Available after lars_comm_init when all ranks share one NVLink domain (NCCL LSA team = world)
 * and LARS_DP_FUSED is not "0"; otherwise LARS_ERR_NO_COMM. Other pointers keep the NCCL path. */
lars_status_t lars_dp_buffers(lars_handle_t h, float** w, void** g);

/* LARS_FLAG_HALF_WEIGHTS: the library-owned compute-weight buffer (padded_numel elements of grad_dtype, the
 * lars_layout offsets; owned by the library). It holds RNE(w) once seeded by lars_init_weights or
 * lars_publish_compute_weights (after lars_comm_init), and after every dp step, applied or skipped (a skipped
 * step publishes the unchanged master weights). LARS_ERR_NO_COMM before lars_comm_init, LARS_ERR_INVALID_ARG
 * without the flag. */
lars_status_t lars_compute_weights(lars_handle_t h, void** w_half);

/* LARS_FLAG_HALF_WEIGHTS: writes RNE(w) of the WHOLE layout (w: device fp32, padded_numel elements, a full
 * replica such as every rank holds after loading a checkpoint) into this rank's compute-weight buffer on
 * `stream`. LARS_ERR_NO_COMM before lars_comm_init, LARS_ERR_INVALID_ARG without the flag. */
lars_status_t lars_publish_compute_weights(lars_handle_t h, const float* w, void* stream);

/* Device pointer to the reduced gradient shard of the last dp step (S elements of *dtype: the wire dtype on
 * the NCCL path, LARS_F32 on the fused path; first element = global element `begin`). Owned by the library.
 * Under LARS_SHARD_GROUPS the buffer is flat (begin = 0, end = padded_numel) and only this rank's slices of
 * every group hold reduced values. */
lars_status_t lars_reduced_grad(lars_handle_t h, const void** dev_ptr, int32_t* dtype, int64_t* begin, int64_t* end);

/* Synchronizing readbacks of the last step (per tensor; entries of tensors this rank does not own are
 * left untouched). w_norm = ||w_l||, g_norm = ||G_l|| (grad_scale applied), lambda = trust ratio,
 * coef = lr*lambda as the update kernel used it. Any output may be NULL. */
lars_status_t lars_last_norms(lars_handle_t h, double* w_norm, double* g_norm, double* lambda, double* coef);
/* Forget the carried weight norms (LARS_FLAG_CARRY_WNORM): the next step recomputes ||w|| from w. */
lars_status_t lars_invalidate_carried_norms(lars_handle_t h);

/* *skipped: 0 = applied, 1 = skipped (non-finite norm), 2 = skipped (device iteration out of range). */
lars_status_t lars_last_step_skipped(lars_handle_t h, int32_t* skipped);

/* Frees everything the handle owns (device buffers, NCCL communicator, symmetric windows). Destroy (or reset)
 * any CUDA graph that captured this handle's steps first: an NCCL communicator referenced by a live graph
 * cannot be torn down. */
lars_status_t lars_destroy(lars_handle_t h);
const char* lars_strerror(lars_status_t s);
const char* lars_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LARS_B200_H */
