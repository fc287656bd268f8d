// Internal types shared by the planner (plan.cpp), the API (lars_api.cpp) and the kernels
// (kernels.cu). Nothing here crosses the C ABI.
#pragma once

#include <cstdint>
#include <vector>

#include <cuda_runtime_api.h>

#include "lars.h"

namespace lars {

constexpr int64_t kAlign = 64;          // element alignment of every tensor (256 B of fp32)
constexpr int kThreads = 256;           // threads per CTA of K1 / K2
constexpr int kCtasPerSm = 2;           // resident CTAs per SM the tile plan targets
constexpr int32_t kDefaultMinTile = 4096;

// One contiguous piece of one tensor inside one work tile. begin is a flat element offset,
// 64-element aligned; len may end on a ragged tensor tail.
struct Seg {
  int64_t begin;
  int32_t len;
  int32_t tensor;  // local tensor index within the work list
};
static_assert(sizeof(Seg) == 16, "Seg is uploaded as-is");

// A work list: the tensors one launch of K1/K2 covers (all tensors for lars_step, the rank's
// shard for the DP step), cut into ntiles tiles of (nearly) equal element count. Tile t covers
// segs [tile_seg[t], tile_seg[t+1]); each CTA of K1/K2 owns exactly one tile (static balance).
struct WorkList {
  std::vector<Seg> segs;            // flat order
  std::vector<int32_t> tile_seg;    // ntiles + 1
  std::vector<int32_t> tensors;     // local -> global tensor id
  std::vector<int32_t> tseg_begin;  // local tensor -> first segment (segments are contiguous)
  std::vector<int32_t> tseg_count;  // local tensor -> number of segments
  std::vector<int32_t> tlars;       // local tensor -> 1 if weight kind (LARS + decay)
  int64_t elems = 0;
  int32_t ntiles() const { return (int32_t)tile_seg.size() - 1; }
};

struct Plan {
  int32_t L = 0, P = 1;
  std::vector<int64_t> numel;
  std::vector<int32_t> kind;
  std::vector<int32_t> owner;   // rank per tensor
  std::vector<int64_t> offset;  // flat offset per tensor
  int64_t S = 0;                // shard length (P = 1: == padded)
  int64_t padded = 0;           // P * S
  int64_t ipe = 0, T = 0, W = 0;
  std::vector<double> lr;       // lr[t], t in [0, T)
  uint64_t hash = 0;
};

lars_status_t validate_hparams(const lars_hparams_t& hp);
lars_status_t make_plan(const lars_tensor_t* t, int32_t n, const lars_hparams_t& hp, Plan& plan);
// Work list over the tensors owned by `rank` (rank < 0: every tensor), ~ntiles_target tiles.
WorkList make_worklist(const Plan& plan, int32_t rank, int32_t ntiles_target, int32_t min_tile);

// ---- kernel launchers (kernels.cu) ----
struct DevWork {
  const Seg* segs;
  const int32_t* tile_seg;
  const int32_t* tseg_begin;
  const int32_t* tseg_count;
  const int32_t* tlars;
  int32_t ntiles;
  int32_t ntensors;
};

struct DevScratch {
  double* part_w;        // per segment: sum w^2 of the segment
  double* part_g;        // per segment: sum g^2
  unsigned* seg_done;    // per local tensor: segments finished this step (reset by the finisher)
  unsigned* tensors_done;
  unsigned* nonfinite;
  int32_t* skip;         // 1 if this step was skipped (written by K1's last finisher)
  double* w_norm;        // per local tensor ||w||
  double* g_norm;        // per local tensor ||G|| (grad_scale applied)
  double* lambda;        // trust ratio
  float* coef;           // lr(t) * lambda, as K2 uses it
  float* beta;           // per-tensor weight decay (0 for skip kinds)
};

struct Hyper {
  const double* lr_table;
  int64_t iter;
  double eta, weight_decay, eps, grad_scale;
  float mu, grad_scale_f;
};

// g_shift: the gradient of flat element e is g[e - g_shift] (the DP step reads its reduced shard).
cudaError_t launch_norms(int32_t grad_dtype, const DevWork& wk, const DevScratch& sc, const Hyper& hy,
                         const float* w, const void* g, int64_t g_shift, cudaStream_t stream);
cudaError_t launch_update(int32_t grad_dtype, const DevWork& wk, const DevScratch& sc, const Hyper& hy,
                          float* w, const void* g, int64_t g_shift, float* m, cudaStream_t stream);
cudaError_t launch_step(int32_t grad_dtype, const DevWork& wk, const DevScratch& sc, const Hyper& hy,
                        float* w, const void* g, int64_t g_shift, float* m, cudaStream_t stream);

}  // namespace lars
