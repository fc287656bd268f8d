// Internal types shared by the planner (plan.cpp), the API (lars_api.cpp) and the kernels
// (kernels.cu). Nothing here crosses the C ABI.
#pragma once

#include <cstdint>
#include <vector>

#include <cuda_runtime_api.h>
#include <nccl.h>
#include <nccl_device/core.h>
#include <nccl_device/impl/comm__types.h>

#include "lars.h"

namespace lars {

constexpr int64_t kAlign = 64;          // element alignment of every tensor (256 B of fp32)
constexpr int kThreads = 256;           // threads per CTA of K1 / K2
#ifndef LARS_NORM_CTAS_PER_SM
#define LARS_NORM_CTAS_PER_SM 4
#endif
#ifndef LARS_NORM_UNROLL
#define LARS_NORM_UNROLL 2
#endif
#ifndef LARS_K1_PREFETCH_LINES  // 128-byte lines of each warp's first fp32 g chunk K1 prefetches before its wait
#define LARS_K1_PREFETCH_LINES 32
#endif
#ifndef LARS_K2_PREFETCH_LINES  // 128-byte lines of w and m of each warp's first fp32-g K2 chunk prefetched before its wait
#define LARS_K2_PREFETCH_LINES 16
#endif
#ifndef LARS_F2_PREFETCH_LINES  // the same for the fused data-parallel F2 (measured at P = 2)
#define LARS_F2_PREFETCH_LINES 0
#endif
#ifndef LARS_K1_KEEP_PCT  // share of each tile's fp32 K1 chunk loads (from its end) with L2::evict_last
#define LARS_K1_KEEP_PCT 100
#endif
#ifndef LARS_NORM_UNROLL_G
#define LARS_NORM_UNROLL_G 4
#endif
constexpr int kCtasPerSm = LARS_NORM_CTAS_PER_SM;      // K1 resident CTAs per SM (one static tile each)
// fused F1 CTAs per SM: 2 ranks fit 64 registers (4 CTAs/SM); 3-8 ranks' loads per vector need 128 (2/SM)
#ifndef LARS_DP_UNROLL_G2  // F1 at P <= 2, carried norms: gradient groups per lane per iteration
#define LARS_DP_UNROLL_G2 2
#endif
#ifndef LARS_DP_CTAS2  // F1 CTAs per SM at P <= 2
#define LARS_DP_CTAS2 4
#endif
constexpr int dp_norm_ctas_per_sm(int nranks) { return nranks <= 2 ? LARS_DP_CTAS2 : 2; }
constexpr int32_t kMaxTileChunks = 256; // chunk partials of one tile live in shared memory
#ifndef LARS_UPDATE_SPLIT
#define LARS_UPDATE_SPLIT 4
#endif
constexpr int32_t kUpdateSplit = LARS_UPDATE_SPLIT;  // K2 walks each tile in parts, last part first
constexpr int kNormUnroll = LARS_NORM_UNROLL;  // K1 vector groups per lane per iteration
constexpr int32_t kDefaultMinTile = 4096;
constexpr bool kK1BulkDefault = false;  // K1 bulk-copy streaming (Hyper::k1_bulk) unless LARS_K1_BULK says
constexpr bool kDeferDefault = true;  // lars_step: layer finish in K2's prologue unless LARS_DEFER_FINISH=0
constexpr int32_t kChunk = 2048;        // elements per warp work item (multiple of 256)

// One contiguous piece of one tensor inside one work tile. begin is a flat element offset,
// 64-element aligned; len may end on a ragged tensor tail.
struct Seg {
  int64_t begin;
  int32_t len;
  int32_t tensor;  // local tensor index within the work list
};
static_assert(sizeof(Seg) == 16, "Seg is uploaded as-is");

// Everything the per-segment finish of K1 needs, packed so one 32-byte load (prefetched during the chunk
// stream) replaces a chain of dependent metadata loads.
struct SegInfo {
  int32_t a, b;        // chunk range [a, b) of the segment (absolute chunk ids)
  int32_t tensor;      // local tensor id
  int32_t nseg;        // segments of that tensor
  int32_t split;       // global split slot or -1
  int32_t lars;        // 1: weight kind (trust ratio + decay)
  int32_t tseg_begin;  // first segment of the tensor
  int32_t pad;
};
static_assert(sizeof(SegInfo) == 32, "SegInfo is uploaded as-is");

// A work list: the tensors one launch of K1/K2 covers (all tensors for lars_step, the rank's
// shard for the DP step), cut into ntiles tiles of (nearly) equal element count. Tile t covers
// segs [tile_seg[t], tile_seg[t+1]); each CTA of K1/K2 owns exactly one tile (static balance).
// Segments are further cut into warp chunks of <= kChunk elements (Seg records with the same
// tensor field): tile t's chunks are [tile_chunk[t], tile_chunk[t+1]), segment s's chunks are
// [seg_chunk[s], seg_chunk[s+1]). The warps of a CTA stream chunks independently, so a tile of
// fifty 64-element BN vectors costs one memory round trip, not fifty.
struct WorkList {
  std::vector<Seg> segs;            // flat order
  std::vector<int32_t> tile_seg;    // ntiles + 1
  std::vector<Seg> chunks;          // flat order
  std::vector<int32_t> tile_chunk;  // ntiles + 1
  std::vector<int32_t> seg_chunk;   // nsegs + 1
  std::vector<int32_t> tensors;     // local -> global tensor id
  std::vector<int32_t> tseg_begin;  // local tensor -> first segment (segments are contiguous)
  std::vector<int32_t> tseg_count;  // local tensor -> number of segments
  std::vector<int32_t> tlars;       // local tensor -> 1 if weight kind (LARS + decay)
  std::vector<int32_t> tsplit;      // local tensor -> global split slot (-1: the layer is whole here)
  int64_t elems = 0;
  int32_t ntiles() const { return (int32_t)tile_seg.size() - 1; }
};

struct Plan {
  int32_t L = 0, P = 1;
  std::vector<int64_t> numel;
  std::vector<int32_t> kind;
  std::vector<int32_t> fan_in;  // 0 = numel (parallel initialization only)
  std::vector<int32_t> owner;   // rank holding the tensor's first element
  std::vector<int32_t> split;   // split slot of a tensor straddling shards (-1: whole on its owner)
  int32_t nsplit = 0;
  std::vector<int64_t> offset;  // flat offset per tensor
  int64_t S = 0;                // shard length (P = 1: == padded)
  int64_t padded = 0;           // P * S
  int64_t ipe = 0, T = 0, W = 0;
  std::vector<double> lr;       // lr[t], t in [0, T)
  uint64_t hash = 0;
  // static backward-order groups (LARS_SHARD_GROUPS; otherwise one group = the whole flat buffer)
  int32_t policy = LARS_SHARD_CONTIGUOUS;
  struct Group {
    int64_t begin = 0, len = 0;  // flat span, len a multiple of 64*P
    int32_t first = 0, last = 0; // tensors first..last (flat order)
  };
  std::vector<Group> groups;     // k = 0: the group backward completes first (holds the last tensor)
  std::vector<int32_t> group_of; // tensor -> group
};

lars_status_t validate_hparams(const lars_hparams_t& hp);
lars_status_t make_plan(const lars_tensor_t* t, int32_t n, const lars_hparams_t& hp, Plan& plan);
// Work list over the tensors owned by `rank` (rank < 0: every tensor), ~ntiles_target tiles.
WorkList make_worklist(const Plan& plan, int32_t rank, int32_t ntiles_target, int32_t min_tile);
// nullptr when the work list satisfies every invariant the kernels rely on, else the violated one.
const char* check_worklist(const Plan& plan, const WorkList& wl, int32_t rank);

// ---- kernel launchers (kernels.cu) ----
struct DevWork {
  const SegInfo* seginfo;
  const Seg* segs;
  const int32_t* tile_seg;
  const Seg* chunks;
  const int32_t* tile_chunk;
  const int32_t* seg_chunk;
  const int32_t* tseg_begin;
  const int32_t* tseg_count;
  const int32_t* tlars;
  const int32_t* tsplit;        // local tensor -> global split slot or -1
  const int32_t* split_locals;  // local ids of this rank's split layers
  int32_t nsplit_local;
  int32_t nsplit_total;         // split layers in the whole plan (C3 payload: 1 + 2 * nsplit_total doubles)
  int32_t ntiles;
  int32_t ntensors;
  int32_t grid;      // K1 and K2 CTAs (same grid: CTA b runs on the same SM in both kernels)
  int32_t nchunks;   // chunks of the work list (device bounds checks)
  int64_t elem_end;  // flat buffer length (device bounds checks: every chunk lies in [0, elem_end))
};

struct DevScratch {
  double* cpart_w;       // per chunk: sum w^2 of the chunk
  double* cpart_wnext;   // per chunk: sum w_new^2 written by K2 in carry mode (LARS_FLAG_CARRY_WNORM)
  int32_t* wnext_valid;  // 1 when cpart_wnext describes the current w (set by K2, cleared by the host)
  double* cpart_g;       // per chunk: sum g^2
  double* part_w;        // per segment: sum w^2 of the segment
  double* part_g;        // per segment: sum g^2
  unsigned* seg_done;    // per local tensor: segments finished this step (reset by the finisher)
  unsigned* tensors_done;
  unsigned* nonfinite;
  int32_t* skip;         // 1 if this step was skipped (written by K1's last finisher)
  // Data-parallel only (nullptr for the whole-layout step): the C3 allreduce payload
  // [non-finite count, (sum w^2, sum g^2) of each split layer]; K1 fills this rank's share, the finisher
  // kernel consumes the global sums and zeroes it for the next step.
  double* c3;
  double* w_norm;        // per local tensor ||w||
  double* g_norm;        // per local tensor ||G|| (grad_scale applied)
  double* lambda;        // trust ratio
  float* coef;           // lr(t) * lambda, as K2 uses it
  float* beta;           // per-tensor weight decay (0 for skip kinds)
  // Deferred finish (single GPU, Hyper::defer): K1 leaves only segment partials, a non-finite flag per K1
  // CTA and (device iteration) the step's iteration; K2 finishes the layers of its own tile.
  int32_t* nf_cta;       // per K1 CTA: 1 if one of its segment partials is non-finite
  int64_t* step_iter;    // the iteration K1 saw in *iter_dev
};

struct Hyper {
  const double* lr_table;
  int64_t iter;              // host-given iteration (iter_dev == nullptr)
  int64_t* iter_dev;         // device iteration: read by K1, advanced by one after the step's last use
  int64_t total_iters;       // T (device-side range check for iter_dev)
  double eta, weight_decay, eps, grad_scale;
  float mu, grad_scale_f;
  bool carry;                // LARS_FLAG_CARRY_WNORM
  bool lr_at_apply;          // LARS_FLAG_LR_AT_APPLY (SPEC.md:186 momentum form)
  void* w_half = nullptr;    // LARS_FLAG_HALF_WEIGHTS: compute weights (grad dtype) the update also writes
  bool k1_bulk = false;      // K1 streams its chunks through the bulk-copy engine (stream_tile_bulk)
  bool defer = false;        // single GPU: the layer finish moves from K1's tail into K2's prologue
  double lr_host = 0.0;      // lr(iter) from the host's table (host-given iteration; saves K2 a load)
};

// g_shift: the gradient of flat element e is g[e - g_shift] (the DP step reads its reduced shard).
cudaError_t launch_norms(int32_t grad_dtype, const DevWork& wk, const DevScratch& sc, const Hyper& hy,
                         const float* w, const void* g, int64_t g_shift, cudaStream_t stream);
cudaError_t launch_update(int32_t grad_dtype, const DevWork& wk, const DevScratch& sc, const Hyper& hy,
                          float* w, const void* g, int64_t g_shift, float* m, cudaStream_t stream);
// Device handles of the fused data-parallel path (symmetric NCCL windows + device communicator).
struct DpFused {
  ncclDevComm dc;
  ncclWindow_t gwin, wwin, xwin;  // gradients (wire dtype), weights (fp32), C3 exchange slots (fp64)
  int rank, nranks;
  int64_t begin;                  // first element of this rank's shard
  float* gred;                    // fp32 reduced shard (S elements)
  unsigned long long* epoch;      // local step counter (advanced by F1's final CTA)
  int64_t* step_iter;             // the iteration of the current step, recorded by F1
  unsigned long long* go;         // F1 entry: CTA 0's "all ranks are in" flag (= epoch + 1)
  unsigned* done;                 // F2 exit: CTAs counted out (the last one syncs with the other ranks)
  bool mcast;                     // NVLS multicast all-gather (multimem.st) instead of per-peer stores
  int np_template;                // F1 peer-count template bound (>= nranks; 2, 4 or 8)
  ncclWindow_t hwin = nullptr;    // LARS_FLAG_HALF_WEIGHTS: compute-weight window (grad dtype), else null
  bool bulk = false;              // F1 streams the rank sum through bulk-copy stages (TMA peer reads)
};
// F1 (reduce + norms + share publication, grid_norm CTAs), then F2 (share collection + update + gather,
// grid_update CTAs, programmatic dependent launch). Events (optional, profiling) are recorded after F1.
// Resident CTAs per SM of the F1 instance (grad dtype, carry, peer-count template) that will be launched.
int dp_reduce_norms_blocks_per_sm(int32_t grad_dtype, bool carry, int np_template, bool bulk);
// Resident K1 CTAs per SM when K1 streams through bulk-copy stages (Hyper::k1_bulk).
int norms_bulk_blocks_per_sm(int32_t grad_dtype, bool carry);
// Compute weights (grad dtype) of every element of the work list = RNE(w) (LARS_FLAG_HALF_WEIGHTS).
cudaError_t launch_publish_half(int32_t grad_dtype, const DevWork& wk, const float* w, void* w_half, cudaStream_t stream);
cudaError_t launch_dp_fused(int32_t grad_dtype, const DevWork& wk, const DevScratch& sc, const Hyper& hy, float* w,
                            float* m, const DpFused& f, int grid_norm, int grid_update, cudaStream_t stream,
                            cudaEvent_t ev1, cudaEvent_t ev2);

// Per-layer table of the parallel initialization (indexed by the work list's local layer id).
struct InitTable {
  const int64_t* offset;  // flat offset of the layer
  const int32_t* layer;   // global layer index (the Philox counter's second word)
  const int32_t* kind;
  const double* sigma;    // sqrt(2 / fan_in) for weight-kind layers
};
cudaError_t launch_init_weights(const DevWork& wk, const InitTable& it, float* w, uint64_t seed, cudaStream_t stream);

// After the C3 allreduce: finish split layers, decide the global skip, advance a device iteration.
cudaError_t launch_split_finish(const DevWork& wk, const DevScratch& sc, const Hyper& hy, cudaStream_t stream);
cudaError_t launch_step(int32_t grad_dtype, const DevWork& wk, const DevScratch& sc, const Hyper& hy,
                        float* w, const void* g, int64_t g_shift, float* m, cudaStream_t stream);

}  // namespace lars
