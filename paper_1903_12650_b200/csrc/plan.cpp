// Host-side planner: flat layout, per-rank shards, work tiles, learning-rate schedule, layout hash.
// Runs once in lars_init. Pure C++: works on a host-only (device = -1) handle.
//
//  * Static planning "beforehand" (§III-C-2): every rank computes the same plan
//    from the same inputs with no communication; lars_comm_init only verifies the hash.
//  * Schedule (PAPER.md:96-103 warm-up + decay; PAPER.md:210-211 16 updates/epoch, 1,440 total).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "internal.h"

namespace lars {

static int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

lars_status_t validate_hparams(const lars_hparams_t& hp) {
  auto fin = [](double x) { return std::isfinite(x); };
  if (!(fin(hp.base_lr) && hp.base_lr > 0)) return LARS_ERR_INVALID_ARG;
  if (!(fin(hp.eta) && hp.eta >= 0)) return LARS_ERR_INVALID_ARG;
  if (!(fin(hp.momentum) && hp.momentum >= 0 && hp.momentum < 1)) return LARS_ERR_INVALID_ARG;
  if (!(fin(hp.weight_decay) && hp.weight_decay >= 0)) return LARS_ERR_INVALID_ARG;
  if (!(fin(hp.eps) && hp.eps >= 0)) return LARS_ERR_INVALID_ARG;
  if (!(fin(hp.warmup_epochs) && hp.warmup_epochs >= 0)) return LARS_ERR_INVALID_ARG;
  if (!(fin(hp.poly_power) && hp.poly_power >= 0)) return LARS_ERR_INVALID_ARG;
  // |s| <= 2^64 keeps ||G|| = |s| sqrt(sum g^2) finite whenever the sum is (a sum of squares of <= 2^31 fp32
  // values is < 2.5e86): a non-finite norm then means a non-finite partial sum (the deferred finish relies on it)
  if (!(fin(hp.grad_scale) && hp.grad_scale != 0 && std::fabs(hp.grad_scale) <= 0x1p64)) return LARS_ERR_INVALID_ARG;
  if (hp.global_batch <= 0 || hp.dataset_size <= 0 || hp.total_epochs <= 0) return LARS_ERR_INVALID_ARG;
  if (hp.grad_dtype < LARS_F32 || hp.grad_dtype > LARS_BF16) return LARS_ERR_INVALID_ARG;
  if (hp.nranks < 1 || hp.nranks > 4096) return LARS_ERR_INVALID_ARG;
  if (hp.tile_elems < 0) return LARS_ERR_INVALID_ARG;
  if (hp.buckets < 0 || hp.buckets > 1024 || hp.reserved != 0) return LARS_ERR_INVALID_ARG;
  if (hp.shard_policy == LARS_SHARD_GROUPS && (hp.group_bytes <= 0 || hp.buckets > 1)) return LARS_ERR_INVALID_ARG;
  if (hp.decay != LARS_DECAY_POLY && hp.decay != LARS_DECAY_STEP) return LARS_ERR_INVALID_ARG;
  if (hp.flags & ~(LARS_FLAG_CARRY_WNORM | LARS_FLAG_LR_AT_APPLY | LARS_FLAG_HALF_WEIGHTS)) return LARS_ERR_INVALID_ARG;
  if ((hp.flags & LARS_FLAG_HALF_WEIGHTS) &&
      (hp.grad_dtype == LARS_F32 || hp.shard_policy == LARS_SHARD_GROUPS || hp.buckets > 1))
    return LARS_ERR_INVALID_ARG;
  if (hp.decay == LARS_DECAY_STEP) {
    if (hp.n_milestones < 0 || hp.n_milestones > 8 || !fin(hp.step_gamma) || hp.step_gamma < 0)
      return LARS_ERR_INVALID_ARG;
    for (int i = 0; i < hp.n_milestones; ++i)
      if (!fin(hp.milestones[i]) || hp.milestones[i] < 0 || (i && hp.milestones[i] < hp.milestones[i - 1]))
        return LARS_ERR_INVALID_ARG;
  }
  return LARS_OK;
}

// ---- schedule -------------------------------------------------------------------------------
// ipe = ceil(D/B) (1,280,000/81,920 -> 16); T = E*ipe (1,440);
// W = round-half-up(warmup_epochs*ipe) (reading #7).
// lr(t) = base*(t+1)/W for t < W (linear warm-up, reading #6);
// lr(t) = base*((T-t)/(T-W))^p for W <= t < T (polynomial decay, reading #8;
//         (T-t)/(T-W) == 1-(t-W)/(T-W) without the cancellation near t = T-1).
static lars_status_t make_schedule(const lars_hparams_t& hp, Plan& p) {
  p.ipe = (hp.dataset_size + hp.global_batch - 1) / hp.global_batch;
  p.T = (int64_t)hp.total_epochs * p.ipe;
  p.W = (int64_t)std::floor(hp.warmup_epochs * (double)p.ipe + 0.5);
  if (p.W > p.T || p.T > (int64_t)1 << 26) return LARS_ERR_INVALID_ARG;
  p.lr.resize(p.T);
  std::vector<int64_t> M;  // step-decay milestones in iterations (round half up, like W)
  if (hp.decay == LARS_DECAY_STEP)
    for (int i = 0; i < hp.n_milestones; ++i) M.push_back((int64_t)std::floor(hp.milestones[i] * (double)p.ipe + 0.5));
  for (int64_t t = 0; t < p.T; ++t) {
    if (t < p.W) {
      p.lr[t] = hp.base_lr * (double)(t + 1) / (double)p.W;
    } else if (hp.decay == LARS_DECAY_STEP) {
      double lr = hp.base_lr;
      for (int64_t m : M)
        if (t >= m) lr *= hp.step_gamma;
      p.lr[t] = lr;
    } else {
      p.lr[t] = hp.base_lr * std::pow((double)(p.T - t) / (double)(p.T - p.W), hp.poly_power);
    }
  }
  return LARS_OK;
}

// ---- layout ---------------------------------------------------------------------------------
// P = 1, and P > 1 with LARS_SHARD_CONTIGUOUS (default): tensors in the given order, each at a
//   64-element aligned offset — the SAME flat layout for every P. Rank r owns [r*S, (r+1)*S) with
//   S = ceil(total/P) (64-aligned): perfectly balanced; at most P-1 tensors straddle a shard boundary
//   ("split" layers, whose norms are completed across ranks by the C3 allreduce).
// P > 1 with LARS_SHARD_LPT: whole-tensor longest-processing-time bin packing (ties: larger tensor
//   first, then lower index; equal loads -> lower rank), rank-major, tensors inside a shard in index
//   order; no layer spans ranks (SURVEY.md §8(e) "D1"), padding grows when a layer exceeds ~N/P.
// P >= 1 with LARS_SHARD_GROUPS (SPEC.md make_buckets): greedy in backward order (last
//   tensor first), a group closes when its gradient bytes first reach group_bytes, the tail is the
//   residual group. Tensors keep flat order inside and across groups; each group's span is padded to a
//   multiple of 64*P and rank r owns slice r of every group. A tensor crossing a slice boundary is split.
static void make_groups_layout(Plan& p, const std::vector<int64_t>& asz, int64_t group_bytes, int32_t esz) {
  const int32_t L = p.L, P = p.P;
  std::vector<std::pair<int32_t, int32_t>> ranges;  // (first, last) in backward order
  int64_t acc = 0;
  int32_t last = L - 1;
  for (int32_t l = L - 1; l >= 0; --l) {
    acc += p.numel[l] * esz;
    if (acc >= group_bytes || l == 0) {
      ranges.push_back({l, last});
      last = l - 1;
      acc = 0;
    }
  }
  const int32_t G = (int32_t)ranges.size();
  p.groups.assign(G, Plan::Group{});
  p.group_of.assign(L, 0);
  int64_t off = 0;
  for (int32_t k = G - 1; k >= 0; --k) {  // flat order = reverse backward order
    Plan::Group& g = p.groups[k];
    g.first = ranges[k].first;
    g.last = ranges[k].second;
    g.begin = off;
    for (int32_t l = g.first; l <= g.last; ++l) {
      p.offset[l] = off;
      p.group_of[l] = k;
      off += asz[l];
    }
    g.len = round_up(off - g.begin, kAlign * P);
    off = g.begin + g.len;
  }
  p.padded = off;
  p.S = off / P;  // elements per rank (sum of its slices)
  for (int32_t l = 0; l < L; ++l) {
    const Plan::Group& g = p.groups[p.group_of[l]];
    const int64_t c = g.len / P;
    p.owner[l] = (int32_t)((p.offset[l] - g.begin) / c);
    if ((p.offset[l] + p.numel[l] - 1 - g.begin) / c != (p.offset[l] - g.begin) / c) p.split[l] = p.nsplit++;
  }
}

static void make_layout(Plan& p, int32_t policy, int64_t group_bytes, int32_t esz) {
  const int32_t L = p.L, P = p.P;
  std::vector<int64_t> asz(L);
  for (int32_t l = 0; l < L; ++l) asz[l] = round_up(p.numel[l], kAlign);
  p.owner.assign(L, 0);
  p.offset.assign(L, 0);
  p.split.assign(L, -1);
  p.nsplit = 0;
  p.policy = policy;
  if (policy == LARS_SHARD_GROUPS) {
    make_groups_layout(p, asz, group_bytes, esz);
    return;
  }
  if (P == 1 || policy == LARS_SHARD_CONTIGUOUS) {
    int64_t off = 0;
    for (int32_t l = 0; l < L; ++l) { p.offset[l] = off; off += asz[l]; }
    const int64_t total = std::max<int64_t>(off, kAlign);
    p.S = round_up((total + P - 1) / P, kAlign);
    p.padded = p.S * P;
    for (int32_t l = 0; l < L; ++l) {
      p.owner[l] = (int32_t)(p.offset[l] / p.S);
      if ((p.offset[l] + p.numel[l] - 1) / p.S != p.offset[l] / p.S) p.split[l] = p.nsplit++;
    }
    return;
  }
  std::vector<int32_t> order(L);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return asz[a] > asz[b]; });
  std::vector<int64_t> load(P, 0);
  for (int32_t l : order) {
    int32_t best = 0;
    for (int32_t r = 1; r < P; ++r)
      if (load[r] < load[best]) best = r;
    p.owner[l] = best;
    load[best] += asz[l];
  }
  int64_t S = std::max<int64_t>(*std::max_element(load.begin(), load.end()), kAlign);
  p.S = round_up(S, kAlign);
  p.padded = p.S * P;
  std::vector<int64_t> fill(P, 0);
  for (int32_t l = 0; l < L; ++l) {
    int32_t r = p.owner[l];
    p.offset[l] = (int64_t)r * p.S + fill[r];
    fill[r] += asz[l];
  }
}

static uint64_t fnv1a(uint64_t h, const void* data, size_t n) {
  const unsigned char* c = (const unsigned char*)data;
  for (size_t i = 0; i < n; ++i) { h ^= c[i]; h *= 1099511628211ull; }
  return h;
}

lars_status_t make_plan(const lars_tensor_t* t, int32_t n, const lars_hparams_t& hp, Plan& p) {
  if (hp.shard_policy != LARS_SHARD_CONTIGUOUS && hp.shard_policy != LARS_SHARD_LPT &&
      hp.shard_policy != LARS_SHARD_GROUPS)
    return LARS_ERR_INVALID_ARG;
  if (n <= 0 || t == nullptr) return LARS_ERR_LAYOUT;
  lars_status_t st = validate_hparams(hp);
  if (st != LARS_OK) return st;
  p.L = n;
  p.P = hp.nranks;
  p.numel.resize(n);
  p.kind.resize(n);
  p.fan_in.resize(n);
  for (int32_t l = 0; l < n; ++l) {
    if (t[l].numel <= 0 || t[l].numel > ((int64_t)1 << 40)) return LARS_ERR_LAYOUT;
    if (t[l].kind < LARS_KIND_WEIGHT || t[l].kind > LARS_KIND_BN_BETA) return LARS_ERR_LAYOUT;
    if (t[l].fan_in < 0) return LARS_ERR_LAYOUT;
    p.numel[l] = t[l].numel;
    p.kind[l] = t[l].kind;
    p.fan_in[l] = t[l].fan_in;
  }
  st = make_schedule(hp, p);
  if (st != LARS_OK) return st;
  const int32_t esz = hp.grad_dtype == LARS_F32 ? 4 : 2;
  make_layout(p, hp.shard_policy, hp.group_bytes, esz);
  if (p.groups.empty()) {  // every other policy: one group, the whole flat buffer
    p.groups.assign(1, Plan::Group{0, p.padded, 0, p.L - 1});
    p.group_of.assign(p.L, 0);
  }
  uint64_t h = 1469598103934665603ull;
  h = fnv1a(h, &p.L, sizeof p.L);
  h = fnv1a(h, &p.P, sizeof p.P);
  h = fnv1a(h, p.numel.data(), p.numel.size() * sizeof(int64_t));
  h = fnv1a(h, p.kind.data(), p.kind.size() * sizeof(int32_t));
  h = fnv1a(h, p.fan_in.data(), p.fan_in.size() * sizeof(int32_t));
  h = fnv1a(h, p.offset.data(), p.offset.size() * sizeof(int64_t));
  const double hd[] = {hp.base_lr, hp.eta, hp.momentum, hp.weight_decay, hp.eps, hp.warmup_epochs,
                       hp.poly_power, hp.grad_scale, hp.step_gamma, (double)hp.decay, (double)hp.flags};
  h = fnv1a(h, hd, sizeof hd);
  const int64_t hi[] = {hp.global_batch, hp.dataset_size, hp.total_epochs, hp.grad_dtype, hp.shard_policy,
                        hp.shard_policy == LARS_SHARD_GROUPS ? hp.group_bytes : 0};
  h = fnv1a(h, hi, sizeof hi);
  h = fnv1a(h, p.lr.data(), p.lr.size() * sizeof(double));  // the whole schedule, milestones included
  p.hash = h;
  return LARS_OK;
}

// ---- work tiles -----------------------------------------------------------------------------
// The tensors of the work set are walked in flat order and cut into tiles of ~E/ntiles elements
// (E = elements of the work set, at least min_tile, a multiple of 64). Cuts inside a tensor fall on
// 64-element boundaries, so every segment starts 256-byte aligned for fp32. Every CTA then streams
// the same number of bytes whatever the tensor-size mix (most ResNet-50 layers are
// too small to occupy a GPU on their own).
// The part of tensor l inside rank `rank`'s shard, as tensor-relative [lo, hi) (rank < 0: all of it).
static void piece(const Plan& p, int32_t l, int32_t rank, int64_t& lo, int64_t& hi) {
  lo = 0;
  hi = p.numel[l];
  if (rank < 0) return;
  int64_t b = (int64_t)rank * p.S, e = b + p.S;
  if (p.policy == LARS_SHARD_GROUPS) {  // slice `rank` of the tensor's group
    const Plan::Group& g = p.groups[p.group_of[l]];
    b = g.begin + rank * (g.len / p.P);
    e = b + g.len / p.P;
  }
  lo = std::max<int64_t>(0, b - p.offset[l]);
  hi = std::min<int64_t>(p.numel[l], e - p.offset[l]);
}

static WorkList make_worklist_once(const Plan& p, int32_t rank, int32_t ntiles_target, int64_t target);

// One CTA per tile in a single wave: if tensor boundaries or the chunk cap produce more tiles than
// ntiles_target, the tile size grows until they fit.
// Tiles are balanced by COST, not elements: a piece of a layer costs its elements plus a fixed
// latency-equivalent per warp chunk and per segment (a 64-element BN vector still costs a memory round
// trip and a per-layer finish), so tiles full of small layers hold fewer elements.
#ifndef LARS_CHUNK_COST
#define LARS_CHUNK_COST 384
#endif
#ifndef LARS_SEG_COST
#define LARS_SEG_COST 512
#endif
constexpr int64_t kChunkCost = LARS_CHUNK_COST, kSegCost = LARS_SEG_COST;

WorkList make_worklist(const Plan& p, int32_t rank, int32_t ntiles_target, int32_t min_tile) {
  int64_t cost = 0;
  for (int32_t l = 0; l < p.L; ++l) {
    int64_t lo, hi;
    piece(p, l, rank, lo, hi);
    if (hi > lo) cost += (hi - lo) + kSegCost + kChunkCost * ((hi - lo + kChunk - 1) / kChunk);
  }
  ntiles_target = std::max(1, ntiles_target);
  // Smallest tile size whose plan fits the tile budget (binary search): one tile per resident CTA keeps
  // every SM equally loaded (a 512-tile plan on 592 CTA slots leaves 80 SMs a CTA short). When the chunk
  // cap forces more tiles than CTAs (very large layouts), the budget becomes the next multiple of the CTA
  // count, so the static round robin still gives every CTA the same number of tiles.
  const int64_t top = cost + kSegCost + kChunkCost + kAlign;
  int32_t budget = ntiles_target;
  while (make_worklist_once(p, rank, budget, top).ntiles() > budget) budget += ntiles_target;
  int64_t lo = std::max<int64_t>(min_tile, 1) - 1, hi = top;  // plan(hi) fits, plan(lo) is below the search
  while (hi - lo > kAlign) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (make_worklist_once(p, rank, budget, mid).ntiles() <= budget) hi = mid;
    else lo = mid;
  }
  return make_worklist_once(p, rank, budget, hi);
}

static WorkList make_worklist_once(const Plan& p, int32_t rank, int32_t ntiles_target, int64_t target) {
  WorkList wl;
  std::vector<int32_t> ids;
  for (int32_t l = 0; l < p.L; ++l) {
    int64_t lo, hi;
    piece(p, l, rank, lo, hi);
    if (hi > lo) ids.push_back(l);
  }
  std::stable_sort(ids.begin(), ids.end(), [&](int32_t a, int32_t b) { return p.offset[a] < p.offset[b]; });
  for (int32_t l : ids) {
    int64_t lo, hi;
    piece(p, l, rank, lo, hi);
    wl.elems += hi - lo;
  }
  (void)ntiles_target;
  target = std::min<int64_t>(round_up(std::max<int64_t>(target, kSegCost + kChunkCost + kAlign), kAlign),
                             (int64_t)1 << 30);
  wl.tile_seg.push_back(0);
  int64_t fill = 0, tchunks = 0;  // cost / warp chunks in the open tile
  auto close_tile = [&]() {
    wl.tile_seg.push_back((int32_t)wl.segs.size());
    fill = 0;
    tchunks = 0;
  };
  for (size_t li = 0; li < ids.size(); ++li) {
    const int32_t l = ids[li];
    wl.tensors.push_back(l);
    wl.tlars.push_back(p.kind[l] == LARS_KIND_WEIGHT ? 1 : 0);
    wl.tsplit.push_back(rank < 0 ? -1 : p.split[l]);  // a whole-layout step sees every layer whole
    wl.tseg_begin.push_back((int32_t)wl.segs.size());
    int64_t pos, end;
    piece(p, l, rank, pos, end);
    while (pos < end) {
      int64_t room = target - fill - kSegCost - kChunkCost;
      int64_t take = std::min<int64_t>(end - pos, room);
      // a tile's chunk partials live in shared memory: at most kMaxTileChunks chunks per tile
      take = std::min<int64_t>(take, (kMaxTileChunks - tchunks) * (int64_t)kChunk);
      if (take < end - pos) take = take / kAlign * kAlign;  // interior cut: 64-aligned
      if (take <= 0) {  // tile full
        close_tile();
        continue;
      }
      wl.segs.push_back(Seg{p.offset[l] + pos, (int32_t)take, (int32_t)li});
      pos += take;
      tchunks += (take + kChunk - 1) / kChunk;
      fill += take + kSegCost + kChunkCost * ((take + kChunk - 1) / kChunk);
      if (fill >= target || tchunks >= kMaxTileChunks) close_tile();
    }
    wl.tseg_count.push_back((int32_t)wl.segs.size() - wl.tseg_begin.back());
  }
  if (fill > 0 || wl.tile_seg.size() == 1) wl.tile_seg.push_back((int32_t)wl.segs.size());
  // warp chunks: every segment cut into <= kChunk-element pieces (64-aligned interior cuts)
  wl.seg_chunk.push_back(0);
  for (const Seg& sg : wl.segs) {
    for (int64_t pos = 0; pos < sg.len; pos += kChunk)
      wl.chunks.push_back(Seg{sg.begin + pos, (int32_t)std::min<int64_t>(kChunk, sg.len - pos), sg.tensor});
    wl.seg_chunk.push_back((int32_t)wl.chunks.size());
  }
  for (int32_t t : wl.tile_seg) wl.tile_chunk.push_back(wl.seg_chunk[t]);
  return wl;
}

// Structural invariants every kernel relies on for in-bounds, race-free access (the kernels index w, g, m
// only through chunks): returns a short reason, or nullptr when the work list is sound.
//  * tiles partition the segments and every tile holds at least one segment (every CTA that owns a tile
//    contributes to the step's layer count before the fused path's epoch can advance);
//  * a tile's chunks fit the shared-memory partial arrays (kMaxTileChunks);
//  * each local tensor's segments are contiguous, in flat order, and cover exactly the tensor's piece on
//    this rank; segment starts are 64-element aligned;
//  * chunks tile their segment, are <= kChunk elements, start 8-element (32 B) aligned and carry the
//    segment's tensor id;
//  * every element lies inside the rank's elements (its shard / group slices) and inside the flat buffer.
const char* check_worklist(const Plan& p, const WorkList& wl, int32_t rank) {
  const int32_t nt = wl.ntiles(), ns = (int32_t)wl.segs.size(), nc = (int32_t)wl.chunks.size();
  const int32_t nl = (int32_t)wl.tensors.size();
  if (nt < 1 || wl.tile_seg.front() != 0 || wl.tile_seg.back() != ns) return "tile_seg does not span the segments";
  for (int32_t t = 0; t < nt; ++t) {
    if (ns > 0 && wl.tile_seg[t + 1] <= wl.tile_seg[t]) return "a tile without segments";
    if (wl.tile_chunk[t] != wl.seg_chunk[wl.tile_seg[t]]) return "tile_chunk inconsistent with seg_chunk";
    if (wl.tile_chunk[t + 1] - wl.tile_chunk[t] > kMaxTileChunks) return "tile exceeds kMaxTileChunks chunks";
    // K2's deferred finish: a tile's segments are consecutive local tensors, and only its first and last
    // segment may belong to a tensor spread over several tiles
    for (int32_t s = wl.tile_seg[t]; s < wl.tile_seg[t + 1]; ++s) {
      const int32_t li = wl.segs[s].tensor;
      if (s > wl.tile_seg[t] && li != wl.segs[s - 1].tensor + 1) return "a tile's tensors are not consecutive";
      if (li >= 0 && li < (int32_t)wl.tseg_count.size() && wl.tseg_count[li] > 1 && s != wl.tile_seg[t] &&
          s != wl.tile_seg[t + 1] - 1)
        return "a multi-tile tensor inside a tile";
    }
  }
  if ((int32_t)wl.seg_chunk.size() != ns + 1 || wl.seg_chunk.front() != 0 || wl.seg_chunk.back() != nc)
    return "seg_chunk does not span the chunks";
  if ((int32_t)wl.tseg_begin.size() != nl || (int32_t)wl.tseg_count.size() != nl || (int32_t)wl.tlars.size() != nl ||
      (int32_t)wl.tsplit.size() != nl)
    return "per-tensor tables have the wrong length";
  int64_t elems = 0;
  int32_t next_seg = 0;
  for (int32_t li = 0; li < nl; ++li) {
    const int32_t l = wl.tensors[li];
    if (l < 0 || l >= p.L) return "tensor id out of range";
    if (li && p.offset[wl.tensors[li - 1]] >= p.offset[l]) return "tensors not in flat order";
    if (wl.tlars[li] != (p.kind[l] == LARS_KIND_WEIGHT ? 1 : 0)) return "tlars differs from the tensor kind";
    int64_t lo, hi;
    piece(p, l, rank, lo, hi);
    if (hi <= lo) return "a listed tensor has no elements here";
    if (rank >= 0 && (wl.tsplit[li] >= 0) != (p.split[l] >= 0)) return "tsplit differs from the plan";
    if (wl.tseg_begin[li] != next_seg || wl.tseg_count[li] < 1) return "tensor segments not contiguous";
    int64_t pos = p.offset[l] + lo;
    for (int32_t s = wl.tseg_begin[li]; s < wl.tseg_begin[li] + wl.tseg_count[li]; ++s) {
      const Seg& sg = wl.segs[s];
      if (sg.tensor != li || sg.begin != pos || sg.len <= 0) return "segments do not tile the tensor piece";
      if (sg.begin % kAlign) return "segment start not 64-element aligned";
      int64_t cpos = sg.begin;
      for (int32_t c = wl.seg_chunk[s]; c < wl.seg_chunk[s + 1]; ++c) {
        const Seg& ck = wl.chunks[c];
        if (ck.tensor != li || ck.begin != cpos || ck.len <= 0 || ck.len > kChunk) return "chunks do not tile the segment";
        if (ck.begin % 8) return "chunk start not 32-byte aligned";
        cpos += ck.len;
      }
      if (cpos != sg.begin + sg.len) return "chunks do not cover the segment";
      pos += sg.len;
    }
    if (pos != p.offset[l] + hi) return "segments do not cover the tensor piece";
    if (p.offset[l] + hi > p.padded) return "elements beyond the flat buffer";
    if (rank >= 0) {  // inside the rank's elements
      int64_t b = (int64_t)rank * p.S, e = b + p.S;
      if (p.policy == LARS_SHARD_GROUPS) {
        const Plan::Group& g = p.groups[p.group_of[l]];
        b = g.begin + rank * (g.len / p.P);
        e = b + g.len / p.P;
      }
      if (p.offset[l] + lo < b || p.offset[l] + hi > e) return "elements outside the rank's shard";
    }
    elems += hi - lo;
    next_seg += wl.tseg_count[li];
  }
  if (next_seg != ns) return "segments not owned by any tensor";
  if (elems != wl.elems) return "element count differs";
  return nullptr;
}

}  // namespace lars
