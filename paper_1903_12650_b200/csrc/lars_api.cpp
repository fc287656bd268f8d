// C ABI implementation (include/lars.h): handle, device scratch, step issue, NCCL data-parallel path.
//
// Data-parallel step:
//   C1  ncclReduceScatter(g -> gred, S, wire dtype, sum)       "gradients ... combined" PAPER.md:31;
//                                                             fp16 on the wire PAPER.md:183;
//                                                             one multi-MB message PAPER.md:147-153
//   K1  per-layer norms + trust ratio on the rank's shard
//   C3  ncclAllReduce([non-finite count, split-layer sums], sum) + finisher kernel: the skip decision is
//       global (reading #13) and layers straddling shards get their norms from every rank
//   K2  fused update of the shard
//   C2  ncclAllGather(w shard -> w)                             every replica holds the owner's fp32 weights
// Everything is stream-ordered: no host synchronization inside a step (CUDA-graph capturable).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "internal.h"

using namespace lars;

namespace {

struct DevBufs {
  WorkList wl;
  DevWork dw{};
  DevScratch sc{};
  void* mem = nullptr;
  const float* carry_w = nullptr;  // weights the carried norms describe (carry mode)
};

size_t dtype_size(int32_t dt) { return dt == LARS_F32 ? 4 : 2; }

struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

template <typename T>
T* carve(char*& p, size_t n) {
  T* r = reinterpret_cast<T*>(p);
  p += (n * sizeof(T) + 255) / 256 * 256;
  return r;
}

lars_status_t upload(DevBufs& b, int sms, int32_t nsplit_total, bool dp, int64_t elem_end) {
  const WorkList& wl = b.wl;
  const size_t ns = std::max<size_t>(wl.segs.size(), 1), nt = std::max<size_t>(wl.tensors.size(), 1),
               ntl = wl.tile_seg.size(), nc = std::max<size_t>(wl.chunks.size(), 1);
  size_t bytes = 0;
  auto add = [&](size_t n, size_t sz) { bytes += (n * sz + 255) / 256 * 256; };
  add(ns, sizeof(SegInfo));                                                             // segment finish info
  add(ns, sizeof(Seg)); add(ntl, 4); add(nt, 4); add(nt, 4); add(nt, 4);                // work list
  add(nc, sizeof(Seg)); add(ntl, 4); add(ns + 1, 4); add(nc, 8); add(nc, 8);            // chunks
  add(nc, 8); add(1, 4);                                                                // carried norms
  add(nt, 4); add(nt, 4); add(dp ? 1 + 2 * (size_t)nsplit_total : 1, 8);                // split layers, C3
  add(ns, 8); add(ns, 8); add(nt, 4); add(1, 4); add(1, 4); add(1, 4);                  // partials, counters
  add(nt, 8); add(nt, 8); add(nt, 8); add(nt, 4); add(nt, 4);                           // outputs
  const size_t ngrid = std::max<size_t>((size_t)std::min<int32_t>(wl.ntiles(), sms * kCtasPerSm), 1);
  add(ngrid, 4); add(1, 8);                                                             // deferred finish
  if (cudaMalloc(&b.mem, bytes) != cudaSuccess) return LARS_ERR_OOM;
  if (cudaMemset(b.mem, 0, bytes) != cudaSuccess) return LARS_ERR_CUDA;
  char* p = (char*)b.mem;
  SegInfo* seginfo = carve<SegInfo>(p, ns);
  Seg* segs = carve<Seg>(p, ns);
  int32_t* tile_seg = carve<int32_t>(p, ntl);
  int32_t* tsb = carve<int32_t>(p, nt);
  int32_t* tsc = carve<int32_t>(p, nt);
  int32_t* tl = carve<int32_t>(p, nt);
  Seg* chunks = carve<Seg>(p, nc);
  int32_t* tile_chunk = carve<int32_t>(p, ntl);
  int32_t* seg_chunk = carve<int32_t>(p, ns + 1);
  int32_t* tsplit = carve<int32_t>(p, nt);
  int32_t* split_locals = carve<int32_t>(p, nt);
  double* c3 = carve<double>(p, dp ? 1 + 2 * (size_t)nsplit_total : 1);
  b.sc.c3 = dp ? c3 : nullptr;
  std::vector<int32_t> locals;
  for (size_t i = 0; i < wl.tsplit.size(); ++i)
    if (wl.tsplit[i] >= 0) locals.push_back((int32_t)i);
  b.sc.cpart_w = carve<double>(p, nc);
  b.sc.cpart_wnext = carve<double>(p, nc);
  b.sc.wnext_valid = carve<int32_t>(p, 1);
  b.sc.cpart_g = carve<double>(p, nc);
  b.sc.part_w = carve<double>(p, ns);
  b.sc.part_g = carve<double>(p, ns);
  b.sc.seg_done = carve<unsigned>(p, nt);
  b.sc.tensors_done = carve<unsigned>(p, 1);
  b.sc.nonfinite = carve<unsigned>(p, 1);
  b.sc.skip = carve<int32_t>(p, 1);
  b.sc.w_norm = carve<double>(p, nt);
  b.sc.g_norm = carve<double>(p, nt);
  b.sc.lambda = carve<double>(p, nt);
  b.sc.coef = carve<float>(p, nt);
  b.sc.beta = carve<float>(p, nt);
  b.sc.nf_cta = carve<int32_t>(p, ngrid);
  b.sc.step_iter = carve<int64_t>(p, 1);
  auto cp = [](void* d, const void* s, size_t n) { return n == 0 || cudaMemcpy(d, s, n, cudaMemcpyHostToDevice) == cudaSuccess; };
  std::vector<SegInfo> si(wl.segs.size());
  for (size_t k = 0; k < wl.segs.size(); ++k) {
    const int32_t l = wl.segs[k].tensor;
    si[k] = SegInfo{wl.seg_chunk[k], wl.seg_chunk[k + 1], l, wl.tseg_count[l], wl.tsplit[l], wl.tlars[l],
                    wl.tseg_begin[l], 0};
  }
  if (!cp(seginfo, si.data(), si.size() * sizeof(SegInfo))) return LARS_ERR_CUDA;
  if (!(cp(segs, wl.segs.data(), wl.segs.size() * sizeof(Seg)) && cp(tile_seg, wl.tile_seg.data(), ntl * 4) &&
        cp(tsb, wl.tseg_begin.data(), wl.tseg_begin.size() * 4) &&
        cp(tsc, wl.tseg_count.data(), wl.tseg_count.size() * 4) && cp(tl, wl.tlars.data(), wl.tlars.size() * 4) &&
        cp(chunks, wl.chunks.data(), wl.chunks.size() * sizeof(Seg)) && cp(tile_chunk, wl.tile_chunk.data(), ntl * 4) &&
        cp(seg_chunk, wl.seg_chunk.data(), wl.seg_chunk.size() * 4) &&
        cp(tsplit, wl.tsplit.data(), wl.tsplit.size() * 4) && cp(split_locals, locals.data(), locals.size() * 4)))
    return LARS_ERR_CUDA;
  b.dw = DevWork{seginfo, segs, tile_seg, chunks, tile_chunk, seg_chunk, tsb, tsc, tl, tsplit, split_locals,
                 (int32_t)locals.size(), dp ? nsplit_total : 0, wl.ntiles(), (int32_t)wl.tensors.size(),
                 std::min<int32_t>(wl.ntiles(), sms * kCtasPerSm), (int32_t)wl.chunks.size(), elem_end};
  (void)sms;
  return LARS_OK;
}

}  // namespace

// Optional per-phase event timing (lars_profile_*): one set of 6 events per profiled step.
struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<std::array<cudaEvent_t, 6>> pending;
  std::vector<int> pending_kind;  // 1 = single GPU, 2 = data parallel
  double acc[5] = {0, 0, 0, 0, 0};
  int64_t steps = 0;
  cudaEvent_t get() {
    cudaEvent_t e = nullptr;
    if (!pool.empty()) { e = pool.back(); pool.pop_back(); return e; }
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    return e;
  }
  std::array<cudaEvent_t, 6>* begin(int kind) {
    if (!on) return nullptr;
    std::array<cudaEvent_t, 6> s;
    for (auto& e : s) e = get();
    pending.push_back(s);
    pending_kind.push_back(kind);
    return &pending.back();
  }
};

static void prof_rec(std::array<cudaEvent_t, 6>* p, int i, cudaStream_t s) {
  if (p && (*p)[i]) cudaEventRecord((*p)[i], s);
}

struct lars_ctx {
  Plan plan;
  lars_hparams_t hp{};
  int device = -1;
  int sms = 148;
  double* lr_d = nullptr;
  DevBufs full, shard;
  bool shard_ready = false;
  ncclComm_t comm = nullptr;
  int rank = 0;
  void* gred = nullptr;
  void* gstage = nullptr;
  void* pinned = nullptr;  // host mirror of skip + norms for lars_step_host_grad
  // lars_step_host_grad: two staging buffers filled on a copy stream, so the copy of step t+1's gradient
  // overlaps step t's kernels (consumed[b]: the step that read buffer b is done; copied[b]: its copy is)
  void* hstage[2] = {nullptr, nullptr};
  cudaStream_t hcs = nullptr;
  cudaEvent_t hcopied[2] = {nullptr, nullptr}, hconsumed[2] = {nullptr, nullptr};
  int hnext = 0;
  cudaStream_t last_stream = nullptr;
  const DevBufs* last = nullptr;
  Profiler prof;
  // fused data-parallel path (symmetric windows); set up by lars_comm_init when every rank is
  // reachable over NVLink (NCCL LSA team == world) and LARS_DP_FUSED != 0
  struct {
    bool ok = false;
    void *w = nullptr, *g = nullptr, *x = nullptr;
    ncclWindow_t wwin = nullptr, gwin = nullptr, xwin = nullptr;
    // second symmetric gradient buffer: dp_allreduce_lars_step_host_grad alternates g / g2 so the copy of
    // step t+1's gradient overlaps step t (peers read the buffer of the step they are in)
    void* g2 = nullptr;
    ncclWindow_t gwin2 = nullptr;
    ncclDevComm dc{};
    bool dc_ok = false;
    float* gred32 = nullptr;
    void* state = nullptr;  // epoch + step iteration
    int grid_norm = 0, grid_update = 0;
    bool mcast = false;
    int np_template = 0;
    bool bulk = false;
  } fused;
  bool k1_bulk = false;     // Hyper::k1_bulk (LARS_K1_BULK)
  bool defer = kDeferDefault;  // Hyper::defer for lars_step (LARS_DEFER_FINISH)
  int32_t last_red_dtype = LARS_F16;
  const void* last_red = nullptr;
  // bucketed NCCL schedule (hp.buckets = K >= 2): bucket k of rank r covers shard-relative elements
  // [bucket_elem[r*(K+1)+k], bucket_elem[r*(K+1)+k+1]) = this rank's tiles [bucket_tile[k], bucket_tile[k+1])
  int32_t K = 1;
  std::vector<int64_t> bucket_elem;
  std::vector<int32_t> bucket_tile;
  cudaStream_t cs = nullptr;  // communication stream of the bucketed schedule
  std::vector<cudaEvent_t> ev;
  void* init_mem = nullptr;  // InitTable of the whole-layout work list (lars_init_weights)
  InitTable init{};
  // static backward-order groups (LARS_SHARD_GROUPS): reduce-scatter of group k on cs as soon as the
  // caller reports it (dp_group_ready); the step issues the rest. Events: ready/rs_start/rs_end per group.
  int32_t next_group = 0;
  const void* group_g = nullptr;
  ncclComm_t gcomm = nullptr;    // communicator of the overlapped group reduce-scatters (fewer CTAs)
  std::vector<cudaEvent_t> gev;  // [3*G + 2]: ready[k], rs0[k], rs1[k], then rs_all_done, applied
  bool gtrace = false, gtrace_valid = false;
  // LARS_FLAG_HALF_WEIGHTS: compute weights (grad dtype, full layout); symmetric when the fused path exists
  void* whalf = nullptr;
  bool whalf_nccl_mem = false;
  ncclWindow_t hwin = nullptr;
};

// Tile-aligned buckets of ~equal element counts for every rank (the plan is static: every rank derives
// every other rank's boundaries without communication).
static void make_buckets(lars_ctx* h, int32_t ntiles_target, int32_t min_tile) {
  const int32_t K = h->K, P = h->plan.P;
  h->bucket_elem.assign((size_t)P * (K + 1), 0);
  for (int32_t r = 0; r < P; ++r) {
    const WorkList wl = r == h->rank ? h->shard.wl : make_worklist(h->plan, r, ntiles_target, min_tile);
    const int32_t nt = wl.ntiles();
    std::vector<int64_t> tile_elems(nt, 0);
    int64_t total = 0;
    for (int32_t t = 0; t < nt; ++t) {
      for (int32_t sgi = wl.tile_seg[t]; sgi < wl.tile_seg[t + 1]; ++sgi) tile_elems[t] += wl.segs[sgi].len;
      total += tile_elems[t];
    }
    std::vector<int32_t> tb(K + 1, nt);
    tb[0] = 0;
    int64_t acc = 0;
    int32_t k = 1;
    for (int32_t t = 0; t < nt && k < K; ++t) {
      acc += tile_elems[t];
      while (k < K && acc * K >= total * k) tb[k++] = t + 1;
    }
    int64_t* eb = &h->bucket_elem[(size_t)r * (K + 1)];
    for (int32_t kk = 0; kk <= K; ++kk) {
      if (kk == 0) eb[kk] = 0;
      else if (kk == K || tb[kk] >= nt) eb[kk] = h->plan.S;
      else eb[kk] = wl.segs[wl.tile_seg[tb[kk]]].begin - (int64_t)r * h->plan.S;
    }
    for (int32_t kk = 1; kk <= K; ++kk) eb[kk] = std::max(eb[kk], eb[kk - 1]);
    if (r == h->rank) h->bucket_tile = tb;
  }
}

// A contiguous tile range of a work list as its own launchable work list (device pointers offset).
static DevWork sub_work(const DevWork& w, int32_t t0, int32_t t1) {
  DevWork s = w;
  s.tile_seg = w.tile_seg + t0;
  s.tile_chunk = w.tile_chunk + t0;
  s.ntiles = t1 - t0;
  s.grid = t1 - t0;
  return s;
}

#define CUDA_OR(expr)                                      \
  do {                                                     \
    if ((expr) != cudaSuccess) return LARS_ERR_CUDA;       \
  } while (0)
#define NCCL_OR(expr)                                      \
  do {                                                     \
    if ((expr) != ncclSuccess) return LARS_ERR_NCCL;       \
  } while (0)

static size_t round4k(size_t b) { return (b + 4095) / 4096 * 4096; }

// Symmetric buffers + windows + device communicator for the fused path. Collective over the comm.
static bool fused_eligible(lars_ctx* h) {
  const char* env = getenv("LARS_DP_FUSED");
  if (env && env[0] == '0') return false;
  if (h->plan.P > 8) return false;  // kMaxRanks
  if (h->plan.policy == LARS_SHARD_GROUPS) return false;  // per-group slices: NCCL path
  return ncclTeamLsa(h->comm).nRanks == h->plan.P;  // every rank on one NVLink domain
}

static lars_status_t setup_fused(lars_ctx* h) {
  auto& f = h->fused;
  const size_t wb = round4k((size_t)h->plan.padded * 4), gb = round4k((size_t)h->plan.padded * dtype_size(h->hp.grad_dtype));
  // exchange slot per rank: [non-finite flag, split-layer sums], each value as two epoch-tagged 64-bit words
  const size_t xb = round4k((size_t)h->plan.P * 2 * (1 + 2 * (size_t)h->plan.nsplit) * sizeof(uint64_t));
  NCCL_OR(ncclMemAlloc(&f.w, wb));
  NCCL_OR(ncclMemAlloc(&f.g, gb));
  NCCL_OR(ncclMemAlloc(&f.x, xb));
  CUDA_OR(cudaMemset(f.w, 0, wb));
  CUDA_OR(cudaMemset(f.g, 0, gb));
  CUDA_OR(cudaMemset(f.x, 0, xb));
  NCCL_OR(ncclCommWindowRegister(h->comm, f.w, wb, &f.wwin, NCCL_WIN_COLL_SYMMETRIC));
  NCCL_OR(ncclCommWindowRegister(h->comm, f.g, gb, &f.gwin, NCCL_WIN_COLL_SYMMETRIC));
  NCCL_OR(ncclMemAlloc(&f.g2, gb));
  CUDA_OR(cudaMemset(f.g2, 0, gb));
  NCCL_OR(ncclCommWindowRegister(h->comm, f.g2, gb, &f.gwin2, NCCL_WIN_COLL_SYMMETRIC));
  NCCL_OR(ncclCommWindowRegister(h->comm, f.x, xb, &f.xwin, NCCL_WIN_COLL_SYMMETRIC));
  // one resident wave each (one tile per CTA). F1 is a cooperative launch sized by the occupancy of the
  // exact instance launched (lars_comm_init computed it); launch_dp_fused caps it at one CTA per tile.
  f.grid_update = h->sms * kCtasPerSm;
  ncclDevCommRequirements reqs;
  std::memset(&reqs, 0, sizeof reqs);
  reqs.lsaBarrierCount = 1;  // one barrier: F1's entry and F2's exit, each taken by a single CTA
  // NVLS multicast all-gather (multimem.st) is opt-in: measured 2x slower than per-peer stores for fp32
  // weights on B200 (profiles/README.md), so per-peer NVLink stores are the default.
  const char* mc_env = getenv("LARS_DP_MCAST");
  reqs.lsaMultimem = mc_env && mc_env[0] == '1';
  if (ncclDevCommCreate(h->comm, &reqs, &f.dc) != ncclSuccess) {
    reqs.lsaMultimem = false;
    NCCL_OR(ncclDevCommCreate(h->comm, &reqs, &f.dc));
  }
  f.mcast = reqs.lsaMultimem;
  f.dc_ok = true;
  if (cudaMalloc(&f.gred32, (size_t)h->plan.S * sizeof(float)) != cudaSuccess) return LARS_ERR_OOM;
  if (cudaMalloc(&f.state, 64) != cudaSuccess) return LARS_ERR_OOM;
  CUDA_OR(cudaMemset(f.state, 0, 64));
  CUDA_OR(cudaMemset(f.gred32, 0, (size_t)h->plan.S * sizeof(float)));
  CUDA_OR(cudaDeviceSynchronize());
  f.ok = true;
  return LARS_OK;
}

static bool aligned256(const void* p) { return ((uintptr_t)p & 255u) == 0; }
static ncclDataType_t nccl_type(int32_t dt) {
  return dt == LARS_F32 ? ncclFloat32 : dt == LARS_F16 ? ncclFloat16 : ncclBfloat16;
}

extern "C" {

void lars_hparams_default(lars_hparams_t* hp) {
  if (!hp) return;
  std::memset(hp, 0, sizeof *hp);
  hp->base_lr = 0.0;
  hp->eta = 1e-3;
  hp->momentum = 0.9;
  hp->weight_decay = 5e-5;
  hp->eps = 0.0;
  hp->warmup_epochs = 5.0;
  hp->poly_power = 2.0;
  hp->grad_scale = 1.0;
  hp->global_batch = 81920;
  hp->dataset_size = 1280000;
  hp->total_epochs = 90;
  hp->grad_dtype = LARS_F16;
  hp->nranks = 1;
  hp->tile_elems = 0;
  hp->step_gamma = 0.1;
  hp->group_bytes = (int64_t)4 << 20;
}

const char* lars_version(void) { return "lars-b200 0.1 (sm_100a)"; }

const char* lars_strerror(lars_status_t s) {
  switch (s) {
    case LARS_OK: return "ok";
    case LARS_ERR_INVALID_ARG: return "invalid argument";
    case LARS_ERR_LAYOUT: return "invalid layout (or layout differs across ranks)";
    case LARS_ERR_ITER_RANGE: return "iteration outside [0, T)";
    case LARS_ERR_ALIGNMENT: return "buffer not 256-byte aligned";
    case LARS_ERR_CUDA: return "CUDA error";
    case LARS_ERR_NCCL: return "NCCL error";
    case LARS_ERR_OOM: return "out of memory";
    case LARS_ERR_NO_COMM: return "no communicator (call lars_comm_init on a handle planned for nranks > 1)";
    case LARS_ERR_NO_DEVICE: return "host-only handle (device = -1)";
  }
  return "unknown status";
}

lars_status_t lars_init(const lars_tensor_t* tensors, int32_t n, const lars_hparams_t* hp, int32_t device,
                        lars_handle_t* out) {
  if (!out || !hp) return LARS_ERR_INVALID_ARG;
  *out = nullptr;
  lars_ctx* h = new (std::nothrow) lars_ctx();
  if (!h) return LARS_ERR_OOM;
  lars_status_t st = make_plan(tensors, n, *hp, h->plan);
  if (st != LARS_OK) { delete h; return st; }
  h->hp = *hp;
  h->device = device;
  const int32_t min_tile = hp->tile_elems > 0 ? hp->tile_elems : kDefaultMinTile;
  if (device >= 0) {
    DeviceGuard g(device);
    if (!g.ok) { delete h; return LARS_ERR_CUDA; }
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && sms > 0) h->sms = sms;
    // K1 through bulk-copy stages when its shared memory still leaves kCtasPerSm CTAs resident per SM
    // (the work list has one tile per resident CTA); LARS_K1_BULK=0/1 overrides (A/B measurement)
    if (const char* df = getenv("LARS_DEFER_FINISH")) h->defer = df[0] == '1';
    const char* kb = getenv("LARS_K1_BULK");
    h->k1_bulk = kb ? kb[0] == '1' : kK1BulkDefault;
    if (h->k1_bulk) {
      const int occ = norms_bulk_blocks_per_sm(hp->grad_dtype, (hp->flags & LARS_FLAG_CARRY_WNORM) != 0);
      if (getenv("LARS_VERBOSE")) fprintf(stderr, "[lars] K1 bulk: %d CTAs/SM resident (need %d)\n", occ, kCtasPerSm);
      if (occ < kCtasPerSm) h->k1_bulk = false;
    }
  }
  h->full.wl = make_worklist(h->plan, -1, h->sms * kCtasPerSm, min_tile);
  if (device >= 0) {
    DeviceGuard g(device);
    if (cudaMalloc(&h->lr_d, h->plan.lr.size() * sizeof(double)) != cudaSuccess) { lars_destroy(h); return LARS_ERR_OOM; }
    if (cudaMemcpy(h->lr_d, h->plan.lr.data(), h->plan.lr.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) {
      lars_destroy(h);
      return LARS_ERR_CUDA;
    }
    st = upload(h->full, h->sms, 0, false, h->plan.padded);
    if (st != LARS_OK) { lars_destroy(h); return st; }
  }
  *out = h;
  return LARS_OK;
}

lars_status_t lars_layout(lars_handle_t h, int64_t* offsets, int64_t* padded_numel) {
  if (!h) return LARS_ERR_INVALID_ARG;
  if (offsets) std::copy(h->plan.offset.begin(), h->plan.offset.end(), offsets);
  if (padded_numel) *padded_numel = h->plan.padded;
  return LARS_OK;
}

lars_status_t lars_schedule(lars_handle_t h, int64_t* ipe, int64_t* total_iters, int64_t* warmup_iters) {
  if (!h) return LARS_ERR_INVALID_ARG;
  if (ipe) *ipe = h->plan.ipe;
  if (total_iters) *total_iters = h->plan.T;
  if (warmup_iters) *warmup_iters = h->plan.W;
  return LARS_OK;
}

lars_status_t lars_lr_at(lars_handle_t h, int64_t iter, double* lr) {
  if (!h || !lr) return LARS_ERR_INVALID_ARG;
  if (iter < 0 || iter >= h->plan.T) return LARS_ERR_ITER_RANGE;
  *lr = h->plan.lr[iter];
  return LARS_OK;
}

lars_status_t lars_shard_range(lars_handle_t h, int32_t rank, int64_t* begin, int64_t* end) {
  if (!h || rank < 0 || rank >= h->plan.P) return LARS_ERR_INVALID_ARG;
  if (h->plan.policy == LARS_SHARD_GROUPS && h->plan.P > 1) return LARS_ERR_INVALID_ARG;  // not contiguous
  if (begin) *begin = (int64_t)rank * h->plan.S;
  if (end) *end = (int64_t)(rank + 1) * h->plan.S;
  return LARS_OK;
}

lars_status_t lars_groups(lars_handle_t h, int32_t* ngroups, int64_t* begin, int64_t* len, int32_t* first_tensor,
                          int32_t* last_tensor) {
  if (!h || !ngroups) return LARS_ERR_INVALID_ARG;
  const auto& G = h->plan.groups;
  *ngroups = (int32_t)G.size();
  for (size_t k = 0; k < G.size(); ++k) {
    if (begin) begin[k] = G[k].begin;
    if (len) len[k] = G[k].len;
    if (first_tensor) first_tensor[k] = G[k].first;
    if (last_tensor) last_tensor[k] = G[k].last;
  }
  return LARS_OK;
}

lars_status_t lars_tensor_owner(lars_handle_t h, int32_t* owner) {
  if (!h || !owner) return LARS_ERR_INVALID_ARG;
  std::copy(h->plan.owner.begin(), h->plan.owner.end(), owner);
  return LARS_OK;
}

lars_status_t lars_init_weights(lars_handle_t h, float* w, uint64_t seed, void* stream) {
  if (!h || !w) return LARS_ERR_INVALID_ARG;
  if (h->device < 0) return LARS_ERR_NO_DEVICE;
  if (!aligned256(w)) return LARS_ERR_ALIGNMENT;
  DeviceGuard dg(h->device);
  if (!h->init_mem) {  // per-layer table of the whole-layout work list, uploaded once
    const WorkList& wl = h->full.wl;
    const size_t n = std::max<size_t>(wl.tensors.size(), 1);
    std::vector<int64_t> off(n, 0);
    std::vector<int32_t> layer(n, 0), kind(n, 0);
    std::vector<double> sigma(n, 0.0);
    for (size_t i = 0; i < wl.tensors.size(); ++i) {
      const int32_t l = wl.tensors[i];
      off[i] = h->plan.offset[l];
      layer[i] = l;
      kind[i] = h->plan.kind[l];
      const int64_t fi = h->plan.fan_in[l] > 0 ? h->plan.fan_in[l] : h->plan.numel[l];
      sigma[i] = std::sqrt(2.0 / (double)fi);
    }
    const size_t bytes = n * (8 + 4 + 4 + 8) + 256;
    if (cudaMalloc(&h->init_mem, bytes) != cudaSuccess) { h->init_mem = nullptr; return LARS_ERR_OOM; }
    char* p = (char*)h->init_mem;
    CUDA_OR(cudaMemcpy(p, off.data(), n * 8, cudaMemcpyHostToDevice));
    CUDA_OR(cudaMemcpy(p + n * 8, sigma.data(), n * 8, cudaMemcpyHostToDevice));
    CUDA_OR(cudaMemcpy(p + n * 16, layer.data(), n * 4, cudaMemcpyHostToDevice));
    CUDA_OR(cudaMemcpy(p + n * 20, kind.data(), n * 4, cudaMemcpyHostToDevice));
    h->init = InitTable{(const int64_t*)p, (const int32_t*)(p + n * 16), (const int32_t*)(p + n * 20),
                        (const double*)(p + n * 8)};
  }
  CUDA_OR(launch_init_weights(h->full.dw, h->init, w, seed, (cudaStream_t)stream));
  h->full.carry_w = nullptr;  // new weights: any carried norms are stale
  h->shard.carry_w = nullptr;
  // every rank initializes the whole replica, so it can also write its whole compute-weight copy
  if (h->whalf) CUDA_OR(launch_publish_half(h->hp.grad_dtype, h->full.dw, w, h->whalf, (cudaStream_t)stream));
  return LARS_OK;
}

lars_status_t lars_publish_compute_weights(lars_handle_t h, const float* w, void* stream) {
  if (!h || !w) return LARS_ERR_INVALID_ARG;
  if (h->device < 0) return LARS_ERR_NO_DEVICE;
  if (!(h->hp.flags & LARS_FLAG_HALF_WEIGHTS)) return LARS_ERR_INVALID_ARG;
  if (!h->whalf) return LARS_ERR_NO_COMM;
  if (!aligned256(w)) return LARS_ERR_ALIGNMENT;
  DeviceGuard dg(h->device);
  CUDA_OR(launch_publish_half(h->hp.grad_dtype, h->full.dw, w, h->whalf, (cudaStream_t)stream));
  return LARS_OK;
}

lars_status_t lars_work_info(lars_handle_t h, int32_t rank, int32_t* ntiles, int32_t* nsegs, int32_t* nchunks) {
  if (!h || rank >= h->plan.P) return LARS_ERR_INVALID_ARG;
  WorkList tmp;
  const WorkList* wl = &h->full.wl;
  if (rank >= 0) {
    if (h->shard_ready && rank == h->rank) {
      wl = &h->shard.wl;
    } else {
      const int32_t min_tile = h->hp.tile_elems > 0 ? h->hp.tile_elems : kDefaultMinTile;
      tmp = make_worklist(h->plan, rank, h->sms * kCtasPerSm, min_tile);
      wl = &tmp;
    }
  }
  if (ntiles) *ntiles = wl->ntiles();
  if (nsegs) *nsegs = (int32_t)wl->segs.size();
  if (nchunks) *nchunks = (int32_t)wl->chunks.size();
  return LARS_OK;
}

lars_status_t lars_check_work(lars_handle_t h, int32_t rank, const char** reason) {
  if (!h || rank >= h->plan.P) return LARS_ERR_INVALID_ARG;
  WorkList tmp;
  const WorkList* wl = &h->full.wl;
  if (rank >= 0) {
    if (h->shard_ready && rank == h->rank) {
      wl = &h->shard.wl;
    } else {
      const int32_t min_tile = h->hp.tile_elems > 0 ? h->hp.tile_elems : kDefaultMinTile;
      tmp = make_worklist(h->plan, rank, h->sms * kCtasPerSm, min_tile);
      wl = &tmp;
    }
  }
  const char* why = check_worklist(h->plan, *wl, rank);
  if (reason) *reason = why ? why : "ok";
  return why ? LARS_ERR_LAYOUT : LARS_OK;
}

lars_status_t lars_layout_hash(lars_handle_t h, uint64_t* hash) {
  if (!h || !hash) return LARS_ERR_INVALID_ARG;
  *hash = h->plan.hash;
  return LARS_OK;
}

static lars_status_t check_step_args(lars_handle_t h, const void* w, const void* g, const void* m, int64_t iter) {
  if (!h || !w || !g || !m) return LARS_ERR_INVALID_ARG;
  if (h->device < 0) return LARS_ERR_NO_DEVICE;
  if (iter < 0 || iter >= h->plan.T) return LARS_ERR_ITER_RANGE;
  if (!aligned256(w) || !aligned256(g) || !aligned256(m)) return LARS_ERR_ALIGNMENT;
  return LARS_OK;
}

static Hyper hyper(lars_handle_t h, int64_t iter, int64_t* iter_dev = nullptr) {
  Hyper hy{h->lr_d, iter, iter_dev, h->plan.T, h->hp.eta, h->hp.weight_decay, h->hp.eps, h->hp.grad_scale,
           (float)h->hp.momentum, (float)h->hp.grad_scale, (h->hp.flags & LARS_FLAG_CARRY_WNORM) != 0,
           (h->hp.flags & LARS_FLAG_LR_AT_APPLY) != 0};
  hy.k1_bulk = h->k1_bulk;
  if (!iter_dev && iter >= 0 && iter < (int64_t)h->plan.lr.size()) hy.lr_host = h->plan.lr[iter];
  return hy;
}

// Carry mode: the norms K2 left are only valid for the weights it wrote. A different weight buffer (or
// an explicit lars_invalidate_carried_norms) makes the next K1 recompute ||w|| from w.
static lars_status_t carry_guard(lars_handle_t h, DevBufs& b, const float* w, cudaStream_t s) {
  if (!(h->hp.flags & LARS_FLAG_CARRY_WNORM)) return LARS_OK;
  if (b.carry_w != w) {
    CUDA_OR(cudaMemsetAsync(b.sc.wnext_valid, 0, sizeof(int32_t), s));
    b.carry_w = w;
  }
  return LARS_OK;
}

static lars_status_t step_impl(lars_handle_t h, float* w, const void* g, float* m, const Hyper& hy_in, void* stream) {
  DeviceGuard dg(h->device);
  Hyper hy = hy_in;
  hy.defer = h->defer;  // the whole-layout step (no split layers): K2 finishes the layers
  cudaStream_t s = (cudaStream_t)stream;
  lars_status_t cg = carry_guard(h, h->full, w, s);
  if (cg != LARS_OK) return cg;
  auto* pe = h->prof.begin(1);
  prof_rec(pe, 0, s);
  CUDA_OR(launch_norms(h->hp.grad_dtype, h->full.dw, h->full.sc, hy, w, g, 0, s));       // K1
  prof_rec(pe, 1, s);
  CUDA_OR(launch_update(h->hp.grad_dtype, h->full.dw, h->full.sc, hy, w, g, 0, m, s));   // K2
  prof_rec(pe, 2, s);
  h->last_stream = s;
  h->last = &h->full;
  return LARS_OK;
}

lars_status_t lars_step(lars_handle_t h, float* w, const void* g, float* m, int64_t iter, void* stream) {
  lars_status_t st = check_step_args(h, w, g, m, iter);
  if (st != LARS_OK) return st;
  return step_impl(h, w, g, m, hyper(h, iter), stream);
}

lars_status_t lars_step_dev_iter(lars_handle_t h, float* w, const void* g, float* m, int64_t* iter_dev, void* stream) {
  if (!iter_dev || ((uintptr_t)iter_dev & 7u)) return LARS_ERR_INVALID_ARG;
  lars_status_t st = check_step_args(h, w, g, m, 0);
  if (st != LARS_OK) return st;
  return step_impl(h, w, g, m, hyper(h, 0, iter_dev), stream);
}

static lars_status_t stage_host_grad(lars_handle_t h, const void* g_host, cudaStream_t s);
static lars_status_t readback_status(lars_handle_t h, const DevBufs& b, cudaStream_t s);

// The copy stream, the per-buffer events and the pinned status mirror of the host-gradient entry points.
static lars_status_t host_stage_events(lars_handle_t h, cudaStream_t s) {
  if (h->hcs) return LARS_OK;
  for (int b = 0; b < 2; ++b) {
    CUDA_OR(cudaEventCreateWithFlags(&h->hcopied[b], cudaEventDisableTiming));
    CUDA_OR(cudaEventCreateWithFlags(&h->hconsumed[b], cudaEventDisableTiming));
    CUDA_OR(cudaEventRecord(h->hconsumed[b], s));
  }
  if (!h->pinned && cudaMallocHost(&h->pinned, 256 + 2 * (size_t)h->plan.L * sizeof(double)) != cudaSuccess) {
    h->pinned = nullptr;
    return LARS_ERR_OOM;
  }
  CUDA_OR(cudaStreamCreateWithFlags(&h->hcs, cudaStreamNonBlocking));
  return LARS_OK;
}

lars_status_t lars_step_host_grad(lars_handle_t h, float* w, const void* g_host, float* m, int64_t iter,
                                  void* stream) {
  if (!h || !g_host) return LARS_ERR_INVALID_ARG;
  if (h->device < 0) return LARS_ERR_NO_DEVICE;
  DeviceGuard dg(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  lars_status_t st = check_step_args(h, w, w, m, iter);  // (g is staged: validated below)
  if (st != LARS_OK) return st;
  const size_t gbytes = (size_t)h->plan.padded * dtype_size(h->hp.grad_dtype);
  st = host_stage_events(h, s);
  if (st != LARS_OK) return st;
  for (int b = 0; b < 2; ++b)
    if (!h->hstage[b] && cudaMalloc(&h->hstage[b], gbytes) != cudaSuccess) {
      h->hstage[b] = nullptr;
      return LARS_ERR_OOM;
    }
  const int b = h->hnext;
  h->hnext ^= 1;
  // the copy waits only for the step that last read this buffer (two steps ago), not for step t-1
  CUDA_OR(cudaStreamWaitEvent(h->hcs, h->hconsumed[b], 0));
  CUDA_OR(cudaMemcpyAsync(h->hstage[b], g_host, gbytes, cudaMemcpyHostToDevice, h->hcs));
  CUDA_OR(cudaEventRecord(h->hcopied[b], h->hcs));
  CUDA_OR(cudaStreamWaitEvent(s, h->hcopied[b], 0));
  st = lars_step(h, w, h->hstage[b], m, iter, stream);
  if (st != LARS_OK) return st;
  CUDA_OR(cudaEventRecord(h->hconsumed[b], s));
  return readback_status(h, h->full, s);
}

lars_status_t lars_get_unique_id(void* id128) {
  if (!id128) return LARS_ERR_INVALID_ARG;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  NCCL_OR(ncclGetUniqueId(reinterpret_cast<ncclUniqueId*>(id128)));
  return LARS_OK;
}

lars_status_t lars_comm_init(lars_handle_t h, int32_t nranks, int32_t rank, const void* id128) {
  if (!h || !id128) return LARS_ERR_INVALID_ARG;
  if (h->device < 0) return LARS_ERR_NO_DEVICE;
  // P = 1 is allowed: a one-rank communicator runs every data-parallel kernel (fused F1/F2, the NCCL
  // path, groups, buckets, half-precision compute weights) on a single GPU.
  if (nranks != h->plan.P || rank < 0 || rank >= nranks) return LARS_ERR_INVALID_ARG;
  if (h->comm) return LARS_ERR_INVALID_ARG;
  DeviceGuard dg(h->device);
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  NCCL_OR(ncclCommInitRank(&h->comm, nranks, id, rank));
  h->rank = rank;
  // Layout agreement (static plan): min and max of the hash over ranks must match.
  uint64_t* d = nullptr;
  CUDA_OR(cudaMalloc(&d, 2 * sizeof(uint64_t)));
  const uint64_t hv[2] = {h->plan.hash, h->plan.hash};
  cudaStream_t s;
  CUDA_OR(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CUDA_OR(cudaMemcpyAsync(d, hv, sizeof hv, cudaMemcpyHostToDevice, s));
  NCCL_OR(ncclGroupStart());
  NCCL_OR(ncclAllReduce(d, d, 1, ncclUint64, ncclMin, h->comm, s));
  NCCL_OR(ncclAllReduce(d + 1, d + 1, 1, ncclUint64, ncclMax, h->comm, s));
  NCCL_OR(ncclGroupEnd());
  uint64_t r[2] = {0, 0};
  CUDA_OR(cudaMemcpyAsync(r, d, sizeof r, cudaMemcpyDeviceToHost, s));
  CUDA_OR(cudaStreamSynchronize(s));
  cudaStreamDestroy(s);
  cudaFree(d);
  if (r[0] != h->plan.hash || r[1] != h->plan.hash) return LARS_ERR_LAYOUT;
  const int32_t min_tile = h->hp.tile_elems > 0 ? h->hp.tile_elems : kDefaultMinTile;
  const bool fused = fused_eligible(h);
  int32_t ntiles_target = h->sms * kCtasPerSm;
  if (fused) {
    // F1 is instantiated for up to 2, 4 or 8 peers; LARS_DP_NP (test knob) forces a wider instance so the
    // P = 8 kernel can be exercised on a box with fewer GPUs (absent peers are predicated off). One tile
    // per resident CTA of the instance that will run.
    const char* np_env = getenv("LARS_DP_NP");
    h->fused.np_template = std::min(8, std::max(h->plan.P, np_env ? atoi(np_env) : 0));
    const bool carry = (h->hp.flags & LARS_FLAG_CARRY_WNORM) != 0;
    // F1 through bulk-copy stages (LARS_DP_BULK=0/1 overrides the default) when 4 CTAs per SM stay resident
    const char* db = getenv("LARS_DP_BULK");
    // default: bulk-copy F1 for the 2- and 8-peer instances. 8 peers (P = 5..8), emulated at P = 4 with
    // LARS_DP_NP=8: 0.231 ms/step against 0.302 for the register instance at 2 CTAs/SM
    // (profiles/r02_dp4/np8_probe); P = 2: 0.162 vs 0.166 ms (F1 4-7 us shorter, profiles/r02_dp2). The
    // 4-peer instance keeps the register loop (0.221 vs 0.227 ms, profiles/r02_dp4).
    h->fused.bulk = db ? db[0] == '1' : h->fused.np_template != 4;
    if (h->fused.bulk && dp_reduce_norms_blocks_per_sm(h->hp.grad_dtype, carry, h->fused.np_template, true) < 2)
      h->fused.bulk = false;  // (F1's work list is cut for whatever residency the instance gets)
    const int bpsm = dp_reduce_norms_blocks_per_sm(h->hp.grad_dtype, carry, h->fused.np_template, h->fused.bulk);
    if (getenv("LARS_VERBOSE"))
      fprintf(stderr, "[lars] rank %d: F1 instance for %d peers, bulk %d (bulk occupancy %d), %d CTAs/SM\n", rank,
              h->fused.np_template, (int)h->fused.bulk,
              dp_reduce_norms_blocks_per_sm(h->hp.grad_dtype, carry, h->fused.np_template, true), bpsm);
    if (bpsm <= 0) return LARS_ERR_CUDA;
    h->fused.grid_norm = h->sms * bpsm;
    ntiles_target = h->fused.grid_norm;
  }
  h->shard.wl = make_worklist(h->plan, rank, ntiles_target, min_tile);
  h->K = std::max(1, h->hp.buckets);
  if (h->K > 1) {
    make_buckets(h, ntiles_target, min_tile);
    CUDA_OR(cudaStreamCreateWithFlags(&h->cs, cudaStreamNonBlocking));
    h->ev.resize(2 * (size_t)h->K + 2, nullptr);
    for (auto& e : h->ev) CUDA_OR(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  lars_status_t st = upload(h->shard, h->sms, h->plan.nsplit, true, h->plan.padded);
  if (st != LARS_OK) return st;
  // reduced gradient: the rank's shard, or (groups) a flat buffer whose slices of every group are this rank's
  const size_t red_elems = (size_t)(h->plan.policy == LARS_SHARD_GROUPS ? h->plan.padded : h->plan.S);
  if (cudaMalloc(&h->gred, red_elems * dtype_size(h->hp.grad_dtype)) != cudaSuccess) return LARS_ERR_OOM;
  CUDA_OR(cudaMemset(h->gred, 0, red_elems * dtype_size(h->hp.grad_dtype)));
  if (h->plan.policy == LARS_SHARD_GROUPS) {
    // The group reduce-scatters run while the caller's backward kernels occupy the SMs: a split
    // communicator with at most LARS_GROUP_MAX_CTAS CTAs per collective (default 8) keeps their footprint
    // small (a collective waiting for a late peer spins on the SMs it holds). 0 = the main communicator.
    const char* mc = getenv("LARS_GROUP_MAX_CTAS");
    const int max_ctas = mc ? atoi(mc) : 8;
    if (max_ctas > 0) {
      ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
      cfg.minCTAs = 1;
      cfg.maxCTAs = max_ctas;
      NCCL_OR(ncclCommSplit(h->comm, 0, rank, &h->gcomm, &cfg));
    }
    CUDA_OR(cudaStreamCreateWithFlags(&h->cs, cudaStreamNonBlocking));
    h->gev.assign(3 * h->plan.groups.size() + 2, nullptr);
    for (auto& e : h->gev) CUDA_OR(cudaEventCreate(&e));  // timing events (also used for ordering)
  }
  h->shard_ready = true;
  if (fused) {
    st = setup_fused(h);
    if (st != LARS_OK) return st;
  }
  if (h->hp.flags & LARS_FLAG_HALF_WEIGHTS) {
    const size_t hb = round4k((size_t)h->plan.padded * dtype_size(h->hp.grad_dtype));
    if (h->fused.ok) {  // peers store into it over NVLink
      NCCL_OR(ncclMemAlloc(&h->whalf, hb));
      h->whalf_nccl_mem = true;
      NCCL_OR(ncclCommWindowRegister(h->comm, h->whalf, hb, &h->hwin, NCCL_WIN_COLL_SYMMETRIC));
    } else if (cudaMalloc(&h->whalf, hb) != cudaSuccess) {
      h->whalf = nullptr;
      return LARS_ERR_OOM;
    }
    CUDA_OR(cudaMemset(h->whalf, 0, hb));
    CUDA_OR(cudaDeviceSynchronize());
  }
  return LARS_OK;
}

// Bucketed NCCL schedule. Communication stream cs: RS(0..K-1) as grouped ncclReduce (one per root rank,
// each rank receiving its own bucket k), then the weight broadcasts. Compute stream s: K1(bucket k) after
// RS(k); C3 + finisher; K2(bucket k) -> broadcast(bucket k) on cs. The per-layer finishing of K1 spans the
// K launches (its counters persist), so results are identical to K = 1 up to NCCL's reduction order.
static lars_status_t dp_bucketed(lars_handle_t h, float* w, const void* g, float* m, const Hyper& hy, cudaStream_t s,
                                 std::array<cudaEvent_t, 6>* pe) {
  const int32_t K = h->K, P = h->plan.P, dt = h->hp.grad_dtype, me = h->rank;
  const int64_t S = h->plan.S, begin = (int64_t)me * S;
  const size_t esz = dtype_size(dt);
  cudaEvent_t* ev_rs = &h->ev[0];
  cudaEvent_t* ev_k2 = &h->ev[K];
  cudaEvent_t ev_go = h->ev[2 * K], ev_done = h->ev[2 * K + 1];
  const DevWork& wk = h->shard.dw;
  const int32_t* tb = h->bucket_tile.data();
  prof_rec(pe, 0, s);
  CUDA_OR(cudaEventRecord(ev_go, s));  // the caller's gradient is ready
  CUDA_OR(cudaStreamWaitEvent(h->cs, ev_go, 0));
  for (int32_t k = 0; k < K; ++k) {  // C1 in K buckets
    NCCL_OR(ncclGroupStart());
    for (int32_t r = 0; r < P; ++r) {
      const int64_t* eb = &h->bucket_elem[(size_t)r * (K + 1)];
      const size_t cnt = (size_t)(eb[k + 1] - eb[k]);
      if (!cnt) continue;
      NCCL_OR(ncclReduce((const char*)g + ((int64_t)r * S + eb[k]) * esz, (char*)h->gred + eb[k] * esz, cnt,
                         nccl_type(dt), ncclSum, r, h->comm, h->cs));
    }
    NCCL_OR(ncclGroupEnd());
    CUDA_OR(cudaEventRecord(ev_rs[k], h->cs));
  }
  for (int32_t k = 0; k < K; ++k) {  // K1 of bucket k as soon as its sums have landed
    CUDA_OR(cudaStreamWaitEvent(s, ev_rs[k], 0));
    if (tb[k + 1] > tb[k]) CUDA_OR(launch_norms(dt, sub_work(wk, tb[k], tb[k + 1]), h->shard.sc, hy, w, h->gred, begin, s));
  }
  prof_rec(pe, 1, s);
  prof_rec(pe, 2, s);
  NCCL_OR(ncclAllReduce(h->shard.sc.c3, h->shard.sc.c3, 1 + 2 * (size_t)h->plan.nsplit, ncclFloat64, ncclSum,
                        h->comm, s));                                                             // C3
  CUDA_OR(launch_split_finish(wk, h->shard.sc, hy, s));
  prof_rec(pe, 3, s);
  for (int32_t k = 0; k < K; ++k) {  // K2 of bucket k, then its weights go out while K2 of k+1 runs
    if (tb[k + 1] > tb[k]) CUDA_OR(launch_update(dt, sub_work(wk, tb[k], tb[k + 1]), h->shard.sc, hy, w, h->gred, begin, m, s));
    CUDA_OR(cudaEventRecord(ev_k2[k], s));
    CUDA_OR(cudaStreamWaitEvent(h->cs, ev_k2[k], 0));
    NCCL_OR(ncclGroupStart());
    for (int32_t r = 0; r < P; ++r) {  // C2: rank r broadcasts its bucket k to everyone (in place)
      const int64_t* eb = &h->bucket_elem[(size_t)r * (K + 1)];
      const size_t cnt = (size_t)(eb[k + 1] - eb[k]);
      if (!cnt) continue;
      float* p = w + (int64_t)r * S + eb[k];
      NCCL_OR(ncclBroadcast(p, p, cnt, ncclFloat32, r, h->comm, h->cs));
    }
    NCCL_OR(ncclGroupEnd());
  }
  CUDA_OR(cudaEventRecord(ev_done, h->cs));
  CUDA_OR(cudaStreamWaitEvent(s, ev_done, 0));  // the step ends on the caller's stream
  prof_rec(pe, 4, s);
  prof_rec(pe, 5, s);
  h->last_stream = s;
  h->last = &h->shard;
  h->last_red = h->gred;
  h->last_red_dtype = dt;
  return LARS_OK;
}

// Static-group schedule (LARS_SHARD_GROUPS). Communication stream cs: reduce-scatter of group k into this
// rank's slice of the flat gred buffer, in group order, each after the caller's ready event for k
// (dp_group_ready) or the step's own. Caller's stream s: K1 over every slice, C3 + finisher, K2, then one
// grouped all-gather (in place, per group) — the values are those of K = 1 up to NCCL's reduction order.
static lars_status_t issue_group(lars_handle_t h, const void* g, int32_t k, cudaStream_t s) {
  const auto& G = h->plan.groups[k];
  const int32_t P = h->plan.P, dt = h->hp.grad_dtype;
  const size_t esz = dtype_size(dt);
  const int64_t c = G.len / P;
  const int32_t ng = (int32_t)h->plan.groups.size();
  CUDA_OR(cudaEventRecord(h->gev[k], s));  // ready[k]: the caller's backward wrote every member of group k
  CUDA_OR(cudaStreamWaitEvent(h->cs, h->gev[k], 0));
  if (h->gtrace) CUDA_OR(cudaEventRecord(h->gev[ng + k], h->cs));
  NCCL_OR(ncclReduceScatter((const char*)g + G.begin * esz, (char*)h->gred + (G.begin + h->rank * c) * esz,
                            (size_t)c, nccl_type(dt), ncclSum, h->gcomm ? h->gcomm : h->comm, h->cs));
  if (h->gtrace) CUDA_OR(cudaEventRecord(h->gev[2 * ng + k], h->cs));
  return LARS_OK;
}

static lars_status_t dp_groups(lars_handle_t h, float* w, const void* g, float* m, const Hyper& hy, cudaStream_t s,
                               std::array<cudaEvent_t, 6>* pe) {
  const int32_t ng = (int32_t)h->plan.groups.size(), P = h->plan.P, dt = h->hp.grad_dtype;
  if (h->next_group > 0 && g != h->group_g) return LARS_ERR_INVALID_ARG;  // early groups used another g
  prof_rec(pe, 0, s);
  for (int32_t k = h->next_group; k < ng; ++k) {
    lars_status_t st = issue_group(h, g, k, s);
    if (st != LARS_OK) return st;
  }
  h->next_group = 0;
  h->group_g = nullptr;
  CUDA_OR(cudaEventRecord(h->gev[3 * ng], h->cs));
  CUDA_OR(cudaStreamWaitEvent(s, h->gev[3 * ng], 0));
  prof_rec(pe, 1, s);
  CUDA_OR(launch_norms(dt, h->shard.dw, h->shard.sc, hy, w, h->gred, 0, s));                       // K1
  prof_rec(pe, 2, s);
  NCCL_OR(ncclAllReduce(h->shard.sc.c3, h->shard.sc.c3, 1 + 2 * (size_t)h->plan.nsplit, ncclFloat64, ncclSum,
                        h->comm, s));                                                             // C3
  CUDA_OR(launch_split_finish(h->shard.dw, h->shard.sc, hy, s));
  prof_rec(pe, 3, s);
  CUDA_OR(launch_update(dt, h->shard.dw, h->shard.sc, hy, w, h->gred, 0, m, s));                   // K2
  prof_rec(pe, 4, s);
  NCCL_OR(ncclGroupStart());
  for (const auto& G : h->plan.groups) {                                                           // C2
    const int64_t c = G.len / P;
    NCCL_OR(ncclAllGather(w + G.begin + h->rank * c, w + G.begin, (size_t)c, ncclFloat32, h->comm, s));
  }
  NCCL_OR(ncclGroupEnd());
  prof_rec(pe, 5, s);
  CUDA_OR(cudaEventRecord(h->gev[3 * ng + 1], s));  // applied
  h->gtrace_valid = h->gtrace;
  h->last_stream = s;
  h->last = &h->shard;
  h->last_red = h->gred;
  h->last_red_dtype = dt;
  return LARS_OK;
}

lars_status_t dp_group_ready(lars_handle_t h, const void* g, int32_t group, void* stream) {
  if (!h || !g) return LARS_ERR_INVALID_ARG;
  if (h->device < 0) return LARS_ERR_NO_DEVICE;
  if (!h->comm || !h->shard_ready) return LARS_ERR_NO_COMM;
  if (h->plan.policy != LARS_SHARD_GROUPS) return LARS_ERR_INVALID_ARG;
  if (group != h->next_group || group >= (int32_t)h->plan.groups.size()) return LARS_ERR_INVALID_ARG;
  if (group > 0 && g != h->group_g) return LARS_ERR_INVALID_ARG;
  if ((uintptr_t)g & 255u) return LARS_ERR_ALIGNMENT;
  DeviceGuard dg(h->device);
  lars_status_t st = issue_group(h, g, group, (cudaStream_t)stream);
  if (st != LARS_OK) return st;
  h->group_g = g;
  h->next_group = group + 1;
  return LARS_OK;
}

lars_status_t lars_group_trace_enable(lars_handle_t h, int32_t enable) {
  if (!h) return LARS_ERR_INVALID_ARG;
  if (h->plan.policy != LARS_SHARD_GROUPS || h->gev.empty()) return LARS_ERR_NO_COMM;
  h->gtrace = enable != 0;
  h->gtrace_valid = false;
  return LARS_OK;
}

lars_status_t lars_group_trace_read(lars_handle_t h, void* ref_event, double* ready, double* rs_start, double* rs_end,
                                    double* applied) {
  if (!h) return LARS_ERR_INVALID_ARG;
  if (!h->gtrace_valid) return LARS_ERR_NO_COMM;
  DeviceGuard dg(h->device);
  const int32_t ng = (int32_t)h->plan.groups.size();
  CUDA_OR(cudaEventSynchronize(h->gev[3 * ng + 1]));
  auto rel = [&](cudaEvent_t e, double* out) -> lars_status_t {
    float ms = 0.f;
    CUDA_OR(cudaEventElapsedTime(&ms, ref_event ? (cudaEvent_t)ref_event : h->gev[0], e));
    *out = ms;
    return LARS_OK;
  };
  for (int32_t k = 0; k < ng; ++k) {
    lars_status_t st = LARS_OK;
    if (ready && (st = rel(h->gev[k], ready + k)) != LARS_OK) return st;
    if (rs_start && (st = rel(h->gev[ng + k], rs_start + k)) != LARS_OK) return st;
    if (rs_end && (st = rel(h->gev[2 * ng + k], rs_end + k)) != LARS_OK) return st;
  }
  if (applied) return rel(h->gev[3 * ng + 1], applied);
  return LARS_OK;
}

// Device-side view of the fused path's state for one launch. The 64-byte state block holds, in order: the
// step epoch, the step's iteration, F1's entry "go" flag and F2's exit counter.
static DpFused fused_view(lars_handle_t h, int64_t begin, ncclWindow_t gwin) {
  DpFused f{};
  f.dc = h->fused.dc;
  f.gwin = gwin;
  f.wwin = h->fused.wwin;
  f.xwin = h->fused.xwin;
  f.rank = h->rank;
  f.nranks = h->plan.P;
  f.begin = begin;
  f.gred = h->fused.gred32;
  char* st = (char*)h->fused.state;
  f.epoch = (unsigned long long*)st;
  f.step_iter = (int64_t*)(st + 8);
  f.go = (unsigned long long*)(st + 16);
  f.done = (unsigned*)(st + 24);
  f.mcast = h->fused.mcast;
  f.np_template = h->fused.np_template;
  f.bulk = h->fused.bulk;
  f.hwin = h->hwin;
  return f;
}

static lars_status_t dp_impl(lars_handle_t h, float* w, const void* g, float* m, const Hyper& hy, void* stream) {
  if (!h->comm || !h->shard_ready) return LARS_ERR_NO_COMM;
  DeviceGuard dg(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t S = h->plan.S, begin = (int64_t)h->rank * S;
  const int32_t dt = h->hp.grad_dtype;
  lars_status_t cg = carry_guard(h, h->shard, w, s);
  if (cg != LARS_OK) return cg;
  Hyper hy_half = hy;
  hy_half.w_half = h->whalf;  // nullptr unless LARS_FLAG_HALF_WEIGHTS
  const Hyper& hy2 = hy_half;
  auto* pe = h->prof.begin(2);
  if (h->fused.ok && (void*)w == h->fused.w && (g == h->fused.g || g == h->fused.g2)) {  // fused NVLink path
    const DpFused f = fused_view(h, begin, g == h->fused.g ? h->fused.gwin : h->fused.gwin2);
    prof_rec(pe, 0, s);
    prof_rec(pe, 1, s);
    CUDA_OR(launch_dp_fused(dt, h->shard.dw, h->shard.sc, hy2, w, m, f, h->fused.grid_norm, h->fused.grid_update, s,
                            pe ? (*pe)[2] : nullptr,
                            pe ? (*pe)[3] : nullptr));
    if (pe) {
      cudaEventRecord((*pe)[4], s);
      cudaEventRecord((*pe)[5], s);
    }
    h->last_stream = s;
    h->last = &h->shard;
    h->last_red = h->fused.gred32;
    h->last_red_dtype = LARS_F32;
    return LARS_OK;
  }
  if (h->K > 1) return dp_bucketed(h, w, g, m, hy, s, pe);
  if (h->plan.policy == LARS_SHARD_GROUPS) return dp_groups(h, w, g, m, hy, s, pe);
  prof_rec(pe, 0, s);
  NCCL_OR(ncclReduceScatter(g, h->gred, (size_t)S, nccl_type(dt), ncclSum, h->comm, s));          // C1
  prof_rec(pe, 1, s);
  CUDA_OR(launch_norms(dt, h->shard.dw, h->shard.sc, hy, w, h->gred, begin, s));                   // K1
  prof_rec(pe, 2, s);
  NCCL_OR(ncclAllReduce(h->shard.sc.c3, h->shard.sc.c3, 1 + 2 * (size_t)h->plan.nsplit, ncclFloat64, ncclSum,
                        h->comm, s));                                                             // C3
  CUDA_OR(launch_split_finish(h->shard.dw, h->shard.sc, hy, s));
  prof_rec(pe, 3, s);
  CUDA_OR(launch_update(dt, h->shard.dw, h->shard.sc, hy2, w, h->gred, begin, m, s));              // K2
  prof_rec(pe, 4, s);
  if (h->whalf) {  // compute weights in the wire dtype: half the all-gather bytes
    const size_t esz = dtype_size(dt);
    NCCL_OR(ncclAllGather((const char*)h->whalf + begin * esz, h->whalf, (size_t)S, nccl_type(dt), h->comm, s));
  } else {
    NCCL_OR(ncclAllGather(w + begin, w, (size_t)S, ncclFloat32, h->comm, s));                     // C2
  }
  prof_rec(pe, 5, s);
  h->last_stream = s;
  h->last = &h->shard;
  h->last_red = h->gred;
  h->last_red_dtype = dt;
  return LARS_OK;
}

lars_status_t dp_allreduce_lars_step(lars_handle_t h, float* w, const void* g, float* m, int64_t iter,
                                     void* stream) {
  lars_status_t st = check_step_args(h, w, g, m, iter);
  if (st != LARS_OK) return st;
  return dp_impl(h, w, g, m, hyper(h, iter), stream);
}

lars_status_t dp_allreduce_lars_step_dev_iter(lars_handle_t h, float* w, const void* g, float* m, int64_t* iter_dev,
                                              void* stream) {
  if (!iter_dev || ((uintptr_t)iter_dev & 7u)) return LARS_ERR_INVALID_ARG;
  lars_status_t st = check_step_args(h, w, g, m, 0);
  if (st != LARS_OK) return st;
  return dp_impl(h, w, g, m, hyper(h, 0, iter_dev), stream);
}

static lars_status_t stage_host_grad(lars_handle_t h, const void* g_host, cudaStream_t s) {
  const size_t gbytes = (size_t)h->plan.padded * dtype_size(h->hp.grad_dtype);
  const size_t L = (size_t)h->plan.L;
  if (!h->gstage) {
    if (cudaMalloc(&h->gstage, gbytes) != cudaSuccess) { h->gstage = nullptr; return LARS_ERR_OOM; }
    if (cudaMallocHost(&h->pinned, 256 + 2 * L * sizeof(double)) != cudaSuccess) { h->pinned = nullptr; return LARS_ERR_OOM; }
  }
  CUDA_OR(cudaMemcpyAsync(h->gstage, g_host, gbytes, cudaMemcpyHostToDevice, s));
  return LARS_OK;
}

static lars_status_t readback_status(lars_handle_t h, const DevBufs& b, cudaStream_t s) {
  char* pin = (char*)h->pinned;
  const size_t nt = b.wl.tensors.size();
  CUDA_OR(cudaMemcpyAsync(pin, b.sc.skip, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  if (nt) {
    CUDA_OR(cudaMemcpyAsync(pin + 256, b.sc.w_norm, nt * sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_OR(cudaMemcpyAsync(pin + 256 + nt * sizeof(double), b.sc.g_norm, nt * sizeof(double), cudaMemcpyDeviceToHost, s));
  }
  return LARS_OK;
}

lars_status_t dp_allreduce_lars_step_host_grad(lars_handle_t h, float* w, const void* g_host, float* m, int64_t iter,
                                               void* stream) {
  if (!h || !g_host) return LARS_ERR_INVALID_ARG;
  if (h->device < 0) return LARS_ERR_NO_DEVICE;
  if (!h->comm || !h->shard_ready) return LARS_ERR_NO_COMM;
  DeviceGuard dg(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  lars_status_t st;
  const void* gdev;
  if (h->fused.ok && (void*)w == h->fused.w) {
    // fused path: the gradient lands in one of the two symmetric buffers, copied on the library's copy stream
    // so the copy of the next step's gradient overlaps this step (the buffer is reused two steps later, after
    // this rank's step that read it — and with it every peer's F1, ordered by F2's exit barrier — completed)
    const size_t gbytes = (size_t)h->plan.padded * dtype_size(h->hp.grad_dtype);
    st = host_stage_events(h, s);
    if (st != LARS_OK) return st;
    const int b = h->hnext;
    h->hnext ^= 1;
    void* gb = b == 0 ? h->fused.g : h->fused.g2;
    CUDA_OR(cudaStreamWaitEvent(h->hcs, h->hconsumed[b], 0));
    CUDA_OR(cudaMemcpyAsync(gb, g_host, gbytes, cudaMemcpyHostToDevice, h->hcs));
    CUDA_OR(cudaEventRecord(h->hcopied[b], h->hcs));
    CUDA_OR(cudaStreamWaitEvent(s, h->hcopied[b], 0));
    st = dp_allreduce_lars_step(h, w, gb, m, iter, stream);
    if (st != LARS_OK) return st;
    CUDA_OR(cudaEventRecord(h->hconsumed[b], s));
    return readback_status(h, h->shard, s);
  } else {
    st = stage_host_grad(h, g_host, s);
    if (st != LARS_OK) return st;
    gdev = h->gstage;
  }
  st = dp_allreduce_lars_step(h, w, gdev, m, iter, stream);
  if (st != LARS_OK) return st;
  return readback_status(h, h->shard, s);
}

lars_status_t lars_profile_enable(lars_handle_t h, int32_t enable) {
  if (!h) return LARS_ERR_INVALID_ARG;
  if (h->device < 0) return LARS_ERR_NO_DEVICE;
  DeviceGuard dg(h->device);
  for (auto& s : h->prof.pending)
    for (auto e : s)
      if (e) h->prof.pool.push_back(e);
  h->prof.pending.clear();
  h->prof.pending_kind.clear();
  for (double& a : h->prof.acc) a = 0;
  h->prof.steps = 0;
  h->prof.on = enable != 0;
  return LARS_OK;
}

lars_status_t lars_profile_read(lars_handle_t h, double* ms, int64_t* steps) {
  if (!h) return LARS_ERR_INVALID_ARG;
  if (h->device < 0) return LARS_ERR_NO_DEVICE;
  DeviceGuard dg(h->device);
  Profiler& p = h->prof;
  for (size_t i = 0; i < p.pending.size(); ++i) {
    auto& ev = p.pending[i];
    const int last = p.pending_kind[i] == 1 ? 2 : 5;
    CUDA_OR(cudaEventSynchronize(ev[last]));
    float t = 0;
    if (p.pending_kind[i] == 1) {
      CUDA_OR(cudaEventElapsedTime(&t, ev[0], ev[1])); p.acc[1] += t;
      CUDA_OR(cudaEventElapsedTime(&t, ev[1], ev[2])); p.acc[3] += t;
    } else {
      for (int k = 0; k < 5; ++k) { CUDA_OR(cudaEventElapsedTime(&t, ev[k], ev[k + 1])); p.acc[k] += t; }
    }
    for (auto e : ev) p.pool.push_back(e);
    ++p.steps;
  }
  p.pending.clear();
  p.pending_kind.clear();
  if (ms) std::copy(p.acc, p.acc + 5, ms);
  if (steps) *steps = p.steps;
  return LARS_OK;
}

lars_status_t lars_dp_buffers(lars_handle_t h, float** w, void** g) {
  if (!h) return LARS_ERR_INVALID_ARG;
  if (!h->fused.ok) return LARS_ERR_NO_COMM;
  if (w) *w = (float*)h->fused.w;
  if (g) *g = h->fused.g;
  return LARS_OK;
}

lars_status_t lars_compute_weights(lars_handle_t h, void** w_half) {
  if (!h || !w_half) return LARS_ERR_INVALID_ARG;
  if (!(h->hp.flags & LARS_FLAG_HALF_WEIGHTS)) return LARS_ERR_INVALID_ARG;
  if (!h->whalf) return LARS_ERR_NO_COMM;
  *w_half = h->whalf;
  return LARS_OK;
}

lars_status_t lars_reduced_grad(lars_handle_t h, const void** dev_ptr, int32_t* dtype, int64_t* begin, int64_t* end) {
  if (!h || !dev_ptr) return LARS_ERR_INVALID_ARG;
  if (!h->gred) return LARS_ERR_NO_COMM;
  *dev_ptr = h->last_red ? h->last_red : h->gred;
  if (dtype) *dtype = h->last_red ? h->last_red_dtype : h->hp.grad_dtype;
  const bool flat = h->plan.policy == LARS_SHARD_GROUPS && h->last_red == h->gred;
  if (begin) *begin = flat ? 0 : (int64_t)h->rank * h->plan.S;
  if (end) *end = flat ? h->plan.padded : (int64_t)(h->rank + 1) * h->plan.S;
  return LARS_OK;
}

lars_status_t lars_last_norms(lars_handle_t h, double* w_norm, double* g_norm, double* lambda, double* coef) {
  if (!h) return LARS_ERR_INVALID_ARG;
  if (h->device < 0) return LARS_ERR_NO_DEVICE;
  const DevBufs* b = h->last ? h->last : &h->full;
  DeviceGuard dg(h->device);
  CUDA_OR(cudaStreamSynchronize(h->last_stream));
  const size_t nt = b->wl.tensors.size();
  std::vector<double> wn(nt), gn(nt), la(nt);
  std::vector<float> cf(nt);
  if (nt) {
    CUDA_OR(cudaMemcpy(wn.data(), b->sc.w_norm, nt * 8, cudaMemcpyDeviceToHost));
    CUDA_OR(cudaMemcpy(gn.data(), b->sc.g_norm, nt * 8, cudaMemcpyDeviceToHost));
    CUDA_OR(cudaMemcpy(la.data(), b->sc.lambda, nt * 8, cudaMemcpyDeviceToHost));
    CUDA_OR(cudaMemcpy(cf.data(), b->sc.coef, nt * 4, cudaMemcpyDeviceToHost));
  }
  for (size_t i = 0; i < nt; ++i) {
    const int32_t l = b->wl.tensors[i];
    if (w_norm) w_norm[l] = wn[i];
    if (g_norm) g_norm[l] = gn[i];
    if (lambda) lambda[l] = la[i];
    if (coef) coef[l] = (double)cf[i];
  }
  return LARS_OK;
}

lars_status_t lars_invalidate_carried_norms(lars_handle_t h) {
  if (!h) return LARS_ERR_INVALID_ARG;
  h->full.carry_w = nullptr;
  h->shard.carry_w = nullptr;
  return LARS_OK;
}

lars_status_t lars_last_step_skipped(lars_handle_t h, int32_t* skipped) {
  if (!h || !skipped) return LARS_ERR_INVALID_ARG;
  if (h->device < 0) return LARS_ERR_NO_DEVICE;
  const DevBufs* b = h->last ? h->last : &h->full;
  DeviceGuard dg(h->device);
  CUDA_OR(cudaStreamSynchronize(h->last_stream));
  CUDA_OR(cudaMemcpy(skipped, b->sc.skip, sizeof(int32_t), cudaMemcpyDeviceToHost));
  return LARS_OK;
}

lars_status_t lars_destroy(lars_handle_t h) {
  if (!h) return LARS_ERR_INVALID_ARG;
  if (h->device >= 0) {
    DeviceGuard dg(h->device);
    if (h->comm) {
      auto& f = h->fused;
      if (f.dc_ok) ncclDevCommDestroy(h->comm, &f.dc);
      if (f.wwin) ncclCommWindowDeregister(h->comm, f.wwin);
      if (f.gwin) ncclCommWindowDeregister(h->comm, f.gwin);
      if (f.gwin2) ncclCommWindowDeregister(h->comm, f.gwin2);
      if (f.xwin) ncclCommWindowDeregister(h->comm, f.xwin);
      if (h->hwin) ncclCommWindowDeregister(h->comm, h->hwin);
      if (h->whalf && h->whalf_nccl_mem) ncclMemFree(h->whalf);
      if (h->whalf && !h->whalf_nccl_mem) cudaFree(h->whalf);
      if (f.w) ncclMemFree(f.w);
      if (f.g) ncclMemFree(f.g);
      if (f.g2) ncclMemFree(f.g2);
      if (f.x) ncclMemFree(f.x);
      cudaFree(f.gred32);
      cudaFree(f.state);
      for (auto e : h->ev)
        if (e) cudaEventDestroy(e);
      for (auto e : h->gev)
        if (e) cudaEventDestroy(e);
      if (h->cs) cudaStreamDestroy(h->cs);
      if (h->gcomm) ncclCommDestroy(h->gcomm);
      ncclCommDestroy(h->comm);
    }
    cudaFree(h->lr_d);
    cudaFree(h->full.mem);
    cudaFree(h->shard.mem);
    cudaFree(h->gred);
    cudaFree(h->gstage);
    if (h->hcs) {
      cudaStreamSynchronize(h->hcs);
      cudaStreamDestroy(h->hcs);
    }
    for (int b = 0; b < 2; ++b) {
      cudaFree(h->hstage[b]);
      if (h->hcopied[b]) cudaEventDestroy(h->hcopied[b]);
      if (h->hconsumed[b]) cudaEventDestroy(h->hconsumed[b]);
    }
    cudaFree(h->init_mem);
    if (h->pinned) cudaFreeHost(h->pinned);
    for (auto& st : h->prof.pending)
      for (auto e : st)
        if (e) cudaEventDestroy(e);
    for (auto e : h->prof.pool) cudaEventDestroy(e);
  }
  delete h;
  return LARS_OK;
}

}  // extern "C"
