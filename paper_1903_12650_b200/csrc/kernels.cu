// Hot-path kernels for sm_100a (B200). HBM-bound streaming: no tensor cores (nothing here is a
// dense contraction).
//
//  K1 lars_norms_kernel  — the "special GPU kernel for batched norm computations" (PAPER.md:130-135,
//     §III-B-2): ONE launch computes sum(w^2) and sum(g^2) of every layer, then, per layer, the trust
//     ratio lambda = eta*||w||/(||G|| + beta*||w|| + eps) (reading #1/#3/#4) and the
//     per-layer coefficient lr(t)*lambda. Work is split into tiles of equal
//     element count (one per CTA), so a 64-element BN vector and a 2.4M-element conv weight cost the
//     same per byte. fp64 accumulation of exact fp64 squares; the per-layer finish sums the per-segment
//     partials in a fixed order (bit-reproducible for a fixed plan). The last finisher of the step
//     decides the whole-step skip flag (non-finite norm -> skip; reading #13).
//  K2 lars_update_kernel — fused unscale (s*g, fp16/bf16 -> fp32 exact), weight decay, momentum and
//     update ("update own weights using single precision"):
//         v <- mu*v + lr*lambda*(s*g + beta_l*w);   w <- w - v          (reading #2)
//     streaming w, g, m exactly once (20 B/param fp32 g, 18 B/param fp16 g). Each CTA walks its tile
//     BACKWARDS, so it first re-reads the bytes K1 read last — the ones still in L2 (K1 loads with
//     L2::evict_last, K2's momentum traffic and stores use L2::evict_first).
// Both kernels are launched with programmatic dependent launch (griddepcontrol) so the next
// kernel's launch overlaps the previous one's tail.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <nccl.h>
#include <nccl_device.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>

#include "internal.h"

namespace lars {

// Device-side bounds and invariant checks (tools/checked_build.py builds the library with
// -DLARS_DEVICE_CHECKS; compute-sanitizer is not available on the GPU pool). Off in the product build.
#ifdef LARS_DEVICE_CHECKS
#define LARS_DCHECK(cond)                                                                         \
  do {                                                                                            \
    if (!(cond)) {                                                                                \
      printf("LARS_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__,  \
             (int)blockIdx.x, (int)threadIdx.x);                                                  \
      __trap();                                                                                   \
    }                                                                                             \
  } while (0)
#else
#define LARS_DCHECK(cond) \
  do {                    \
  } while (0)
#endif

// Every access of w, g, m goes through a chunk: it must lie inside the flat buffer, start 32-byte aligned
// (256-bit vectors) and belong to a local tensor of the work list.
__device__ __forceinline__ void check_chunk(const DevWork& wk, int32_t c, const Seg& ck) {
  LARS_DCHECK(c >= 0 && c < wk.nchunks);
  LARS_DCHECK(ck.begin >= 0 && ck.len > 0 && ck.len <= kChunk && ck.begin + ck.len <= wk.elem_end);
  LARS_DCHECK((ck.begin & 7) == 0);
  LARS_DCHECK(ck.tensor >= 0 && ck.tensor < wk.ntensors);
}

// ---------------------------------------------------------------- 256-bit / 128-bit accessors
struct F8 { float v[8]; };

__device__ __forceinline__ F8 ld8_keep(const float* p) {  // read-only, keep in L2 for K2
  uint32_t r[8];
  asm("ld.global.nc.L1::no_allocate.L2::evict_last.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p));
  F8 o;
#pragma unroll
  for (int i = 0; i < 8; ++i) o.v[i] = __uint_as_float(r[i]);
  return o;
}
__device__ __forceinline__ F8 ld8_nc(const float* p) {  // read-only in this kernel
  uint32_t r[8];
  asm("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p));
  F8 o;
#pragma unroll
  for (int i = 0; i < 8; ++i) o.v[i] = __uint_as_float(r[i]);
  return o;
}
__device__ __forceinline__ F8 ld8_rw(const float* p) {  // read then overwritten by the same thread
  uint32_t r[8];
  asm volatile("ld.global.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p));
  F8 o;
#pragma unroll
  for (int i = 0; i < 8; ++i) o.v[i] = __uint_as_float(r[i]);
  return o;
}
__device__ __forceinline__ void st8(float* p, const F8& o) {
  asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               ::"l"(p), "r"(__float_as_uint(o.v[0])), "r"(__float_as_uint(o.v[1])), "r"(__float_as_uint(o.v[2])),
               "r"(__float_as_uint(o.v[3])), "r"(__float_as_uint(o.v[4])), "r"(__float_as_uint(o.v[5])),
               "r"(__float_as_uint(o.v[6])), "r"(__float_as_uint(o.v[7]))
               : "memory");
}
// Store with no compiler memory clobber: lets later (non-aliasing) loads be hoisted above it.
__device__ __forceinline__ void st8_noclobber(float* p, const F8& o) {
  asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               ::"l"(p), "r"(__float_as_uint(o.v[0])), "r"(__float_as_uint(o.v[1])), "r"(__float_as_uint(o.v[2])),
               "r"(__float_as_uint(o.v[3])), "r"(__float_as_uint(o.v[4])), "r"(__float_as_uint(o.v[5])),
               "r"(__float_as_uint(o.v[6])), "r"(__float_as_uint(o.v[7])));
}
__device__ __forceinline__ uint4 ld16_nc(const void* p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// Gradient access by wire dtype. Widening fp16/bf16 -> fp32 is exact.
template <int DT> struct Grad;
// Raw (undecoded) 8-element vectors: lets a caller issue many loads before decoding any of them.
template <int DT> struct GradRaw { using T = uint4; };
template <> struct GradRaw<LARS_F32> { using T = F8; };

template <> struct Grad<LARS_F32> {
  __device__ __forceinline__ static F8 load8_keep(const void* g, int64_t i) { return ld8_keep((const float*)g + i); }
  __device__ __forceinline__ static F8 load8(const void* g, int64_t i) { return ld8_nc((const float*)g + i); }
  __device__ __forceinline__ static float load1(const void* g, int64_t i) { return __ldg((const float*)g + i); }
  __device__ __forceinline__ static F8 raw8(const void* g, int64_t i) { return ld8_nc((const float*)g + i); }
  __device__ __forceinline__ static F8 widen(const F8& r) { return r; }
};
__device__ __forceinline__ F8 widen_h8(uint4 r) {
  F8 o;
  const uint32_t u[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __half22float2(*reinterpret_cast<const __half2*>(&u[i]));
    o.v[2 * i] = f.x;
    o.v[2 * i + 1] = f.y;
  }
  return o;
}
__device__ __forceinline__ F8 widen_b8(uint4 r) {
  F8 o;
  const uint32_t u[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    o.v[2 * i] = __uint_as_float(u[i] << 16);
    o.v[2 * i + 1] = __uint_as_float(u[i] & 0xffff0000u);
  }
  return o;
}
template <> struct Grad<LARS_F16> {
// 16-bit gradients carry NO L2 keep hint in K1: the .L2::evict_last qualifier exists for 256-bit loads
// only, and a 128-bit load with an evict_last cache-hint policy measured 13.7 us (fp16) / 6.8 us (bf16)
// slower per step than a plain load (profiles/r02_h16_keep_sweep.txt).
  __device__ __forceinline__ static F8 load8_keep(const void* g, int64_t i) { return widen_h8(ld16_nc((const __half*)g + i)); }
  __device__ __forceinline__ static F8 load8(const void* g, int64_t i) { return widen_h8(ld16_nc((const __half*)g + i)); }
  __device__ __forceinline__ static float load1(const void* g, int64_t i) { return __half2float(((const __half*)g)[i]); }
  __device__ __forceinline__ static uint4 raw8(const void* g, int64_t i) { return ld16_nc((const __half*)g + i); }
  __device__ __forceinline__ static F8 widen(const uint4& r) { return widen_h8(r); }
};
template <> struct Grad<LARS_BF16> {
  __device__ __forceinline__ static F8 load8_keep(const void* g, int64_t i) { return widen_b8(ld16_nc((const uint16_t*)g + i)); }
  __device__ __forceinline__ static F8 load8(const void* g, int64_t i) { return widen_b8(ld16_nc((const uint16_t*)g + i)); }
  __device__ __forceinline__ static float load1(const void* g, int64_t i) {
    return __uint_as_float((uint32_t)((const uint16_t*)g)[i] << 16);
  }
  __device__ __forceinline__ static uint4 raw8(const void* g, int64_t i) { return ld16_nc((const uint16_t*)g + i); }
  __device__ __forceinline__ static F8 widen(const uint4& r) { return widen_b8(r); }
};

#ifdef LARS_TRACE
// Diagnostics build only (tools/trace_build.py): per-CTA [start ns, end ns, smid, tiles] per kernel.
__device__ unsigned long long* g_trace = nullptr;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}
#define TRACE_BEGIN unsigned long long _t0 = gtimer();
#define TRACE_END(k)                                                          \
  if (threadIdx.x == 0 && g_trace) {                                          \
    unsigned long long* _p = g_trace + ((size_t)(k) * 4096 + blockIdx.x) * 4; \
    _p[0] = _t0; _p[1] = gtimer(); _p[2] = smid(); _p[3] = gridDim.x;         \
  }
#define TRACE_MARK(k)                                                         \
  if (threadIdx.x == 0 && g_trace) g_trace[((size_t)(k) * 4096 + blockIdx.x) * 4 + 2] = gtimer();
#define TRACE_MARK_AT(k, c) \
  if (threadIdx.x == 0 && g_trace) g_trace[((size_t)(k) * 4096 + blockIdx.x) * 4 + (c)] = gtimer();
extern "C" int lars_trace_arm(void* buf) {
  return (int)cudaMemcpyToSymbol(g_trace, &buf, sizeof buf);
}
#else
#define TRACE_BEGIN
#define TRACE_END(k)
#define TRACE_MARK(k)
#define TRACE_MARK_AT(k, c)
#endif

// ---------------------------------------------------------------- gradient sources for K1
// Plain: the (already combined) gradient in local memory; element e lives at g[e - shift].
template <int DT>
struct LocalGrad {
  static constexpr bool kBulk = true;  // may stream through the bulk-copy engine (stream_tile_bulk)
  static constexpr int kDt = DT;
  static constexpr int kPeers = 0;
  __device__ __forceinline__ int nsrc() const { return 1; }
  __device__ __forceinline__ const void* src(int, int64_t e) const {
    return (const char*)g + (e - shift) * (DT == LARS_F32 ? 4 : 2);
  }
  static constexpr int kUnroll = kNormUnroll;  // (w, g) groups per lane per iteration
  static constexpr int kUnrollG = LARS_NORM_UNROLL_G;  // g-only groups per lane per iteration (carried norms)
  const void* g;
  int64_t shift;
  __device__ __forceinline__ F8 load8(int64_t e) const { return Grad<DT>::load8_keep(g, e - shift); }
  // keep = false: the chunk is one K2 reads late (after L2 has turned over): do not displace kept lines
  __device__ __forceinline__ F8 load8(int64_t e, bool keep) const {
    return keep ? Grad<DT>::load8_keep(g, e - shift) : Grad<DT>::load8(g, e - shift);
  }
  __device__ __forceinline__ float load1(int64_t e) const { return Grad<DT>::load1(g, e - shift); }
};

// Fused data-parallel reduce-scatter (dp fused path): element e of this rank's shard is the sum over the
// P ranks' gradient buffers (symmetric NCCL window, read over NVLink), accumulated in fp32 in rank order;
// the sum is also stored once into the local fp32 shard buffer the update kernel reads.
// Reading #29 (gradients are communicated in half precision): the combined gradient is a
// wire-format value, so a sum whose magnitude rounds to infinity in the wire dtype IS infinite — the
// fp32 sum saturates to +-Inf at the wire dtype's round-to-nearest-even overflow threshold, the norm goes
// non-finite and the whole step is skipped, as on the NCCL path (fp16 sums) and in the oracle.
template <int DT> struct WireMax { static constexpr float v = 3.4028234663852886e38f; };  // fp32: none
template <> struct WireMax<LARS_F16> { static constexpr float v = 65520.0f; };  // (65504 + 65536) / 2
template <> struct WireMax<LARS_BF16> { static constexpr float v = 3.3961775292304958e38f; };  // 0x7F7F8000
template <int DT>
__device__ __forceinline__ float wire_saturate(float x) {
  if constexpr (DT == LARS_F32) return x;
  return fabsf(x) >= WireMax<DT>::v ? copysignf(__int_as_float(0x7f800000), x) : x;
}
constexpr int kMaxRanks = 8;
template <int DT, int NP>  // NP: compile-time upper bound of the rank count (2, 4 or 8)
struct PeerSumGrad {
  static constexpr bool kBulk = true;
  static constexpr int kDt = DT;
  static constexpr int kPeers = NP;
  const void* gp[NP];         // gradient buffer of every rank (index = rank < nranks), same flat layout
  int nranks;
  float* gred;                // local fp32 reduced shard: element e at gred[e - begin]
  int64_t begin;
  static constexpr int kUnroll = 1;                 // (w, g) groups per lane per iteration (register budget)
  static constexpr int kUnrollG = NP <= 2 ? LARS_DP_UNROLL_G2 : 1;  // g-only groups per lane per iteration (carry)
  static constexpr int kBatch = NP < 4 ? NP : 4;   // peer loads issued back to back before decoding
  __device__ __forceinline__ F8 load8(int64_t e) const {
    F8 acc;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc.v[i] = 0.f;
#pragma unroll
    for (int p0 = 0; p0 < NP; p0 += kBatch) {  // rank order 0..nranks-1, in batches of kBatch loads
      typename GradRaw<DT>::T r[kBatch];
#pragma unroll
      for (int q = 0; q < kBatch; ++q)
        if (p0 + q < nranks) r[q] = Grad<DT>::raw8(gp[p0 + q], e);
#pragma unroll
      for (int q = 0; q < kBatch; ++q)
        if (p0 + q < nranks) {
          const F8 x = Grad<DT>::widen(r[q]);
#pragma unroll
          for (int i = 0; i < 8; ++i) acc.v[i] += x.v[i];
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) acc.v[i] = wire_saturate<DT>(acc.v[i]);
    st8_noclobber(gred + (e - begin), acc);
    return acc;
  }
  __device__ __forceinline__ F8 load8(int64_t e, bool) const { return load8(e); }
  __device__ __forceinline__ int nsrc() const { return nranks; }
  __device__ __forceinline__ const void* src(int p, int64_t e) const {
    return (const char*)gp[p] + e * (DT == LARS_F32 ? 4 : 2);
  }
  __device__ __forceinline__ void store8(int64_t e, const F8& x) const { st8_noclobber(gred + (e - begin), x); }
  __device__ __forceinline__ float load1(int64_t e) const {
    float acc = 0.f;
    for (int p = 0; p < nranks; ++p) acc += Grad<DT>::load1(gp[p], e);
    acc = wire_saturate<DT>(acc);
    gred[e - begin] = acc;
    return acc;
  }
};

// Asynchronous global -> shared copies (LDGSTS): issued early, waited for with cp_async_wait_all().
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ---------------------------------------------------------------- bulk copies (TMA engine) + mbarriers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  } while (!ok);
}
// order this thread's earlier generic-proxy accesses of shared memory before later async-proxy (bulk copy) ones
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// global -> shared bulk copy by the TMA engine; completes `bytes` of transaction count on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}

__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Launch with programmatic dependent launch: the kernel may become resident while its predecessor
// drains and must call pdl_wait() before touching anything the predecessor writes. coop: cooperative
// launch — the driver guarantees every CTA of the grid is co-resident (F1's CTAs wait on CTA 0's flag).
template <typename K, typename... Args>
static cudaError_t launch_pdl_smem(K kernel, int grid, cudaStream_t stream, bool coop, size_t smem, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = coop ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}
template <typename K, typename... Args>
static cudaError_t launch_pdl_ex(K kernel, int grid, cudaStream_t stream, bool coop, Args... args) {
  return launch_pdl_smem(kernel, grid, stream, coop, 0, args...);
}
template <typename K, typename... Args>
static cudaError_t launch_pdl(K kernel, int grid, cudaStream_t stream, Args... args) {
  return launch_pdl_ex(kernel, grid, stream, false, args...);
}

// Sum of squares added to a fp64 accumulator: exact fp64 squares of the fp32 values, fp64 adds (reading #15).
// (Summing each 8-element group in fp32 and widening once, with an fp64 redo for out-of-range groups, was
// measured: -1 us on fp32/fp16 gradients, +5 us on bf16 — the conversions are not what bounds K1. Not kept.)
__device__ __forceinline__ void acc8(double& a, const F8& x) {
#pragma unroll
  for (int i = 0; i < 8; ++i) a = fma((double)x.v[i], (double)x.v[i], a);
}
__device__ __forceinline__ void acc4(double& a, const float4& x) {
  a = fma((double)x.x, (double)x.x, a);
  a = fma((double)x.y, (double)x.y, a);
  a = fma((double)x.z, (double)x.z, a);
  a = fma((double)x.w, (double)x.w, a);
}

// ---------------------------------------------------------------- K1: segmented norms + finish
// Deterministic warp sum of x[a..b): lane i adds elements a+i, a+i+32, ... in order, then a fixed
// xor butterfly. The result (identical in every lane) depends only on the plan, never on timing.
__device__ __forceinline__ void warp_sum2(const double* xa, const double* xb, int32_t a, int32_t b, int lane,
                                          double& ra, double& rb) {
  double sa = 0.0, sb = 0.0;
  int32_t i = a + lane;
  for (; i + 96 < b; i += 128) {  // four loads of each in flight, added in the same order as one at a time
    const double a0 = __ldcg(xa + i), a1 = __ldcg(xa + i + 32), a2 = __ldcg(xa + i + 64), a3 = __ldcg(xa + i + 96);
    const double b0 = __ldcg(xb + i), b1 = __ldcg(xb + i + 32), b2 = __ldcg(xb + i + 64), b3 = __ldcg(xb + i + 96);
    sa += a0;
    sa += a1;
    sa += a2;
    sa += a3;
    sb += b0;
    sb += b1;
    sb += b2;
    sb += b3;
  }
  for (; i < b; i += 32) {
    sa += __ldcg(xa + i);
    sb += __ldcg(xb + i);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
    sb += __shfl_xor_sync(0xffffffffu, sb, o);
  }
  ra = sa;
  rb = sb;
}

// Per-layer finish from the layer's complete sums: ||w||, ||G|| = |s| sqrt(sum g^2), lambda, lr*lambda.
// Returns true when a norm is non-finite (the step will be skipped).
// lr(t) of this step and whether t is inside the schedule (read once per thread, early, off the critical path)
struct StepLr {
  double lr;
  bool in_range;
};
__device__ __forceinline__ StepLr step_lr(const Hyper& hy) {
  const int64_t t = hy.iter_dev ? *(volatile const int64_t*)hy.iter_dev : hy.iter;
  const bool in_range = t >= 0 && t < hy.total_iters;  // host-given iterations are validated on the host
  return StepLr{in_range ? hy.lr_table[t] : 0.0, in_range};
}

__device__ __forceinline__ bool finish_core(int32_t l, int32_t lars, double sw, double sg, const DevScratch& sc,
                                            const Hyper& hy, const StepLr& slr) {
  const double wn = sqrt(sw);
  const double gn = fabs(hy.grad_scale) * sqrt(sg);
  double lam = 1.0, beta = 0.0;
  if (lars) {  // weight kind: trust ratio + decay (reading #1, #3); skip kinds keep 1, 0 (#4)
    beta = hy.weight_decay;
    const double den = gn + hy.weight_decay * wn + hy.eps;
    // lambda = 1 when ||w|| = 0 or the denominator does not exceed the guard (reading #3)
    if (wn > 0.0 && den > hy.eps) lam = hy.eta * wn / den;
  }
  sc.w_norm[l] = wn;
  sc.g_norm[l] = gn;
  sc.lambda[l] = lam;
  sc.coef[l] = slr.in_range ? (float)(slr.lr * lam) : 0.0f;
  sc.beta[l] = (float)beta;
  return !(isfinite(wn) && isfinite(gn) && slr.in_range);
}
__device__ __forceinline__ bool finish_core(int32_t l, double sw, double sg, const DevWork& wk, const DevScratch& sc,
                                            const Hyper& hy) {
  return finish_core(l, wk.tlars[l], sw, sg, sc, hy, step_lr(hy));
}

// K1 phase A through the bulk-copy engine (single GPU / NCCL path, hy.k1_bulk): every warp streams its
// chunks (c0 + warp, c0 + warp + 8, ...) as pieces of <= 2 KB (pe elements of g, plus w when the weight
// norms are not carried) through kBulkStages private shared-memory stages. Lane 0 keeps kBulkStages pieces in
// flight with cp.async.bulk (no registers held per byte in flight, unlike the register loop, whose loads in
// flight per lane are capped by the 64-register budget); each stage has an mbarrier completed by the copy's
// transaction count. The warp sums squares from shared memory in fp64 (fixed order: lane, piece, then the
// xor butterfly), the < 8 ragged elements at a tensor's end straight from global memory. Gradient and
// weight bytes are fetched with an L2 evict_last policy (K2 re-reads them).
#ifndef LARS_BULK_STAGES
#define LARS_BULK_STAGES 3
#endif
#ifndef LARS_BULK_STAGE_BYTES
#define LARS_BULK_STAGE_BYTES 2048
#endif
constexpr int kBulkStages = LARS_BULK_STAGES;  // per warp
constexpr int kBulkStageBytes = LARS_BULK_STAGE_BYTES;
constexpr int kBulkSmem = kThreads / 32 * kBulkStages * kBulkStageBytes;  // 48 KB dynamic shared memory

// GL: LocalGrad<DT> (K1: one gradient source) or PeerSumGrad<DT, NP> (F1: the gradient of every rank, read
// over NVLink from the symmetric window; the consumer sums the ranks in order in fp32, applies the wire
// saturation, stores the sum into the fp32 reduced shard and accumulates its square).
template <class GL>
__device__ __forceinline__ void stream_tile_bulk(int32_t c0, int32_t c1, const DevWork& wk, const float* __restrict__ w,
                                                 const GL& gl, bool carried, double* sm_cw, double* sm_cg,
                                                 unsigned char* stages, uint64_t* bars, uint32_t& q) {
  constexpr int DT = GL::kDt;
  constexpr int kEs = DT == LARS_F32 ? 4 : 2;
  constexpr int kWarps = kThreads / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nsrc = gl.nsrc();
  const int32_t cw0 = c0 + warp;
  const int32_t nk = cw0 < c1 ? (c1 - cw0 + kWarps - 1) / kWarps : 0;  // this warp's chunks (<= 32)
  LARS_DCHECK(nk <= 32);
  // lane k holds the descriptor of this warp's k-th chunk (shuffled to the whole warp when needed)
  const Seg my = lane < nk ? wk.chunks[cw0 + kWarps * lane] : Seg{0, 0, 0};
  // piece elements: one stage holds w (unless carried) and every source's gradient for pe elements
  const int32_t pe = kBulkStageBytes / (nsrc * kEs + (carried ? 0 : 4)) / 8 * 8;
  const int32_t goff = carried ? 0 : pe * 4;  // gradient sub-buffers start here, pe * kEs bytes each
  const uint64_t pol = l2_policy_evict_last();
  unsigned char* wst = stages + warp * kBulkStages * kBulkStageBytes;
  uint64_t* wbar = bars + warp * kBulkStages;
  int32_t pk = 0, pj = 0;  // producer cursor: chunk pk, element pj inside it
  uint32_t pq = q;         // next piece to produce (piece q lives in stage q % kBulkStages)
  auto produce = [&]() {   // warp-uniform; lane 0 issues
    if (pk >= nk) return;
    const int64_t begin = __shfl_sync(0xffffffffu, my.begin, pk);
    const int32_t len = __shfl_sync(0xffffffffu, my.len, pk);
    const int32_t n = min(pe, len - pj), nb = n & ~7;
    if (lane == 0) {
      const uint32_t st = pq % kBulkStages;
      unsigned char* dst = wst + st * kBulkStageBytes;
      fence_proxy_async_smem();  // this warp's reads of the stage's previous piece precede the copy
      mbar_arrive_expect_tx(wbar + st, (uint32_t)nb * (nsrc * kEs + (carried ? 0 : 4)));
      if (nb > 0) {
        const int64_t e = begin + pj;
        if (!carried) bulk_g2s(dst, w + e, (uint32_t)nb * 4u, wbar + st, pol);
        for (int p = 0; p < nsrc; ++p)
          bulk_g2s(dst + goff + p * pe * kEs, gl.src(p, e), (uint32_t)nb * kEs, wbar + st, pol);
      }
    }
    ++pq;
    pj += pe;
    if (pj >= len) {
      pj = 0;
      ++pk;
    }
  };
#pragma unroll
  for (int i = 0; i < kBulkStages; ++i) produce();
  for (int32_t k = 0; k < nk; ++k) {
    const int64_t begin = __shfl_sync(0xffffffffu, my.begin, k);
    const int32_t len = __shfl_sync(0xffffffffu, my.len, k);
    double aw = 0.0, ag = 0.0;
    for (int32_t j = 0; j < len; j += pe) {
      const uint32_t st = q % kBulkStages;
      mbar_wait(wbar + st, (q / kBulkStages) & 1u);
      const int32_t n = min(pe, len - j), nb = n & ~7;
      const unsigned char* src = wst + st * kBulkStageBytes;
      if (!carried)
        for (int32_t i = 4 * lane; i < nb; i += 128) {
          acc4(aw, *reinterpret_cast<const float4*>(src + 4 * i));
        }
      if constexpr (GL::kPeers == 0) {
        const unsigned char* gs = src + goff;
        if constexpr (DT == LARS_F32) {
          for (int32_t i = 4 * lane; i < nb; i += 128) {
            acc4(ag, *reinterpret_cast<const float4*>(gs + 4 * i));
          }
        } else {
          for (int32_t i = 8 * lane; i < nb; i += 256) acc8(ag, Grad<DT>::widen(*reinterpret_cast<const uint4*>(gs + 2 * i)));
        }
      } else {  // rank sum (rank order, fp32) of 8-element groups, stored to the reduced shard
        for (int32_t i = 8 * lane; i < nb; i += 256) {
          F8 acc;
#pragma unroll
          for (int t = 0; t < 8; ++t) acc.v[t] = 0.f;
          for (int p = 0; p < nsrc; ++p) {
            const unsigned char* gs = src + goff + p * pe * kEs + i * kEs;
            F8 x;
            if constexpr (DT == LARS_F32) {
              const float4 x0 = *reinterpret_cast<const float4*>(gs), x1 = *reinterpret_cast<const float4*>(gs + 16);
              x = F8{{x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w}};
            } else {
              x = Grad<DT>::widen(*reinterpret_cast<const uint4*>(gs));
            }
#pragma unroll
            for (int t = 0; t < 8; ++t) acc.v[t] += x.v[t];
          }
#pragma unroll
          for (int t = 0; t < 8; ++t) acc.v[t] = wire_saturate<DT>(acc.v[t]);
          gl.store8(begin + j + i, acc);
          acc8(ag, acc);
        }
      }
      for (int32_t i = nb + lane; i < n; i += 32) {  // ragged tensor tail (< 8 elements), from global memory
        const int64_t e = begin + j + i;
        if (!carried) aw = fma((double)w[e], (double)w[e], aw);
        const double y = (double)gl.load1(e);
        ag = fma(y, y, ag);
      }
      __syncwarp();  // every lane is done with the stage before lane 0 refills it
      ++q;
      produce();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {  // fixed butterfly: deterministic
      aw += __shfl_xor_sync(0xffffffffu, aw, o);
      ag += __shfl_xor_sync(0xffffffffu, ag, o);
    }
    if (lane == 0) {
      const int32_t c = cw0 + kWarps * k;
      sm_cg[c - c0] = ag;
      if (!carried) sm_cw[c - c0] = aw;
    }
  }
}

template <class GL, bool REG_PATH = true>  // REG_PATH = false: bulk-copy streaming only (F1 BULK instances)
__device__ __forceinline__ void norms_tile(int32_t tile, const DevWork& wk, const DevScratch& sc, const Hyper& hy,
                                           const float* __restrict__ w, const GL& gl, double* sm_cw,
                                           double* sm_cg, unsigned* sm_done, unsigned* sm_nonfinite, bool carried,
                                           const StepLr& slr, unsigned char* stages = nullptr,
                                           uint64_t* bars = nullptr, uint32_t* bulk_q = nullptr) {
  constexpr int kWarps = kThreads / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int32_t s0 = wk.tile_seg[tile], s1 = wk.tile_seg[tile + 1];
  // Copied into shared memory under the chunk stream (cp.async, no registers held): every warp's first
  // segment finish record, and in carry mode the tile's carried chunk sums of w^2 (<= kMaxTileChunks ==
  // kThreads, one per thread).
  __shared__ __align__(16) SegInfo sm_si[kThreads / 32];
  static_assert(kMaxTileChunks <= kThreads, "one carried chunk partial per thread");
  // Phase A: the warps of the CTA stream the tile's chunks independently (no block barrier per layer);
  // chunk partials stay in shared memory.
  const int32_t c0 = wk.tile_chunk[tile], c1 = wk.tile_chunk[tile + 1];
  LARS_DCHECK(c0 >= 0 && c0 <= c1 && c1 - c0 <= kMaxTileChunks && c1 <= wk.nchunks);
  LARS_DCHECK(s0 < s1 || wk.ntensors == 0);
  if (carried && tid < c1 - c0) cp_async8(sm_cw + tid, sc.cpart_wnext + c0 + tid);
  if (lane < 2 && s0 + warp < s1) cp_async16((char*)(sm_si + warp) + 16 * lane, (const char*)(wk.seginfo + s0 + warp) + 16 * lane);
  bool bulk = false;
  if constexpr (GL::kBulk) {
    if (stages) {
      stream_tile_bulk(c0, c1, wk, w, gl, carried, sm_cw, sm_cg, stages, bars, *bulk_q);
      bulk = true;
    }
  }
  // chunk descriptors are prefetched one iteration ahead (their load would otherwise add a round trip
  // in front of every chunk's data loads)
  Seg nxt = (REG_PATH && !bulk && c0 + warp < c1) ? wk.chunks[c0 + warp] : Seg{0, 0, 0};
  for (int32_t c = c0 + warp; REG_PATH && !bulk && c < c1; c += kWarps) {
    const Seg ck = nxt;
    check_chunk(wk, c, ck);
    if (c + kWarps < c1) nxt = wk.chunks[c + kWarps];
    const float* wp = w + ck.begin;
    const int64_t gi = ck.begin;  // element index handed to the gradient source
    const int32_t ng = ck.len >> 3;
    if (carried) {  // sum(w^2) of this chunk was produced by the previous K2: stream g only
      double ag = 0.0, ag1 = 0.0;
      int32_t j = lane;
      constexpr int U = GL::kUnrollG;  // local source: 4 x 32 B in flight per lane
      // K2 walks every tile's parts last-to-first: only the tail of each tile can still be in L2 then
      const bool keep = (int64_t)(c - c0) * 100 >= (int64_t)(c1 - c0) * (100 - LARS_K1_KEEP_PCT);
      for (; j + (U - 1) * 32 < ng; j += U * 32) {
        F8 gv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) gv[u] = gl.load8(gi + 8 * (j + 32 * u), keep);
#pragma unroll
        for (int u = 0; u < U; u += 2) {
          acc8(ag, gv[u]);
          if (u + 1 < U) acc8(ag1, gv[u + 1]);
        }
      }
      for (; j < ng; j += 32) acc8(ag, gl.load8(gi + 8 * j));
      ag += ag1;
      for (int32_t i = (ng << 3) + lane; i < ck.len; i += 32) {
        const double y = (double)gl.load1(gi + i);
        ag = fma(y, y, ag);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ag += __shfl_xor_sync(0xffffffffu, ag, o);
      if (lane == 0) sm_cg[c - c0] = ag;
      continue;
    }
    double aw = 0.0, ag = 0.0, aw1 = 0.0, ag1 = 0.0;
    int32_t j = lane;
    constexpr int U = GL::kUnroll;
    const bool keep = (int64_t)(c - c0) * 100 >= (int64_t)(c1 - c0) * (100 - LARS_K1_KEEP_PCT);
    for (; j + (U - 1) * 32 < ng; j += U * 32) {
      F8 wv[U], gv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {  // all loads first: 2*U x 32 B in flight per lane
        wv[u] = keep ? ld8_keep(wp + 8 * (j + u * 32)) : ld8_nc(wp + 8 * (j + u * 32));
        gv[u] = gl.load8(gi + 8 * (j + u * 32), keep);
      }
#pragma unroll
      for (int u = 0; u < U; u += 2) {
        acc8(aw, wv[u]);
        acc8(ag, gv[u]);
        if (u + 1 < U) {
          acc8(aw1, wv[u + 1]);
          acc8(ag1, gv[u + 1]);
        }
      }
    }
    for (; j < ng; j += 32) {
      const F8 w0 = keep ? ld8_keep(wp + 8 * j) : ld8_nc(wp + 8 * j);
      const F8 g0 = gl.load8(gi + 8 * j, keep);
      acc8(aw, w0);
      acc8(ag, g0);
    }
    aw += aw1;
    ag += ag1;
    for (int32_t i = (ng << 3) + lane; i < ck.len; i += 32) {  // ragged tensor tail (< 8 elements)
      const double x = (double)wp[i], y = (double)gl.load1(gi + i);
      aw = fma(x, x, aw);
      ag = fma(y, y, ag);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {  // fixed butterfly: deterministic
      aw += __shfl_xor_sync(0xffffffffu, aw, o);
      ag += __shfl_xor_sync(0xffffffffu, ag, o);
    }
    if (lane == 0) {
      sm_cw[c - c0] = aw;
      sm_cg[c - c0] = ag;
    }
  }
  cp_async_wait_all();
  __syncthreads();  // every chunk partial of this tile is in shared memory
  TRACE_MARK_AT(4, 0)
  // Phase B: one warp per segment sums its chunk partials (fixed order). A layer that lies inside this
  // tile is finished right here (no global traffic beyond its outputs); a layer spread over several
  // tiles publishes the segment partial and the warp that brings in its last segment finishes it.
  for (int32_t s = s0 + warp; s < s1; s += kWarps) {
    const SegInfo si = (s == s0 + warp) ? sm_si[warp] : wk.seginfo[s];
    const int32_t a = si.a - c0, b = si.b - c0;
    LARS_DCHECK(a >= 0 && a < b && b <= c1 - c0);  // the segment's chunk partials are this tile's
    LARS_DCHECK(si.tensor >= 0 && si.tensor < wk.ntensors && si.nseg >= 1);
    LARS_DCHECK(si.split < wk.nsplit_total);
    double tw = 0.0, tg = 0.0;
    for (int32_t i = a + lane; i < b; i += 32) {
      tw += sm_cw[i];
      tg += sm_cg[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tw += __shfl_xor_sync(0xffffffffu, tw, o);
      tg += __shfl_xor_sync(0xffffffffu, tg, o);
    }
    const int32_t l = si.tensor;
    const int32_t nseg = si.nseg;
    const int32_t split = si.split;
    if (hy.defer) {  // K2 finishes the layer: leave the segment partial (and whether it is finite)
      if (lane == 0) {
        sc.part_w[s] = tw;
        sc.part_g[s] = tg;
        if (!(isfinite(tw) && isfinite(tg))) atomicOr(sm_nonfinite, 1u);
      }
      continue;
    }
    if (nseg == 1) {
      if (lane == 0) {
        if (split >= 0) {  // straddles ranks: publish this rank's share for the C3 allreduce
          sc.c3[1 + 2 * split] = tw;
          sc.c3[2 + 2 * split] = tg;
        } else if (finish_core(l, si.lars, tw, tg, sc, hy, slr)) {
          atomicOr(sm_nonfinite, 1u);
        }
        atomicAdd(sm_done, 1u);
      }
      continue;
    }
    unsigned prev = 0;
    if (lane == 0) {
      sc.part_w[s] = tw;
      sc.part_g[s] = tg;
      __threadfence();
      prev = atomicAdd(sc.seg_done + l, 1u);
    }
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (prev == (unsigned)nseg - 1u) {  // last segment of layer l: this warp finishes it
      __threadfence();
      const int32_t sb = si.tseg_begin;
      double sw = 0.0, sg = 0.0;
      for (int32_t i = sb + lane; i < sb + nseg; i += 32) {
        sw += __ldcg(sc.part_w + i);
        sg += __ldcg(sc.part_g + i);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sw += __shfl_xor_sync(0xffffffffu, sw, o);
        sg += __shfl_xor_sync(0xffffffffu, sg, o);
      }
      if (lane == 0) {
        sc.seg_done[l] = 0u;  // all of this step's arrivals are in: rearm for the next step
        if (split >= 0) {
          sc.c3[1 + 2 * split] = sw;
          sc.c3[2 + 2 * split] = sg;
        } else if (finish_core(l, si.lars, sw, sg, sc, hy, slr)) {
          atomicOr(sm_nonfinite, 1u);
        }
        atomicAdd(sm_done, 1u);
      }
    }
  }
}

// K1 body, shared by the single-GPU / NCCL kernel and the fused data-parallel kernel (they differ only
// in where the gradient comes from). Static persistent schedule: CTA b owns tiles b, b + grid, ... (one
// tile per resident CTA by construction of the work list; dynamically scheduled tiles measured slower).
// Returns true on thread 0 of the CTA that completed the step's layer count (data-parallel mode: the
// caller then publishes this rank's C3 shares).
template <bool CARRY, class GL, bool REG_PATH = true>
__device__ __forceinline__ bool norms_body(const DevWork& wk, const DevScratch& sc, const Hyper& hy,
                                           const float* __restrict__ w, const GL& gl,
                                           unsigned char* stages = nullptr) {
  __shared__ double sm_cw[kMaxTileChunks], sm_cg[kMaxTileChunks];
  __shared__ unsigned sm_done, sm_nonfinite;
  __shared__ uint64_t sm_bars[kThreads / 32 * kBulkStages];
  uint32_t bulk_q = 0;  // pieces this warp has consumed (its stages' mbarrier phases)
  if (threadIdx.x == 0) {
    sm_done = 0u;
    sm_nonfinite = 0u;
  }
  if (stages && (threadIdx.x & 31) == 0) {
    for (int i = 0; i < kBulkStages; ++i) mbar_init(sm_bars + (threadIdx.x >> 5) * kBulkStages + i, 1u);
    mbar_init_fence();
  }
  __syncthreads();
  // carry mode: the previous K2 left sum(w_new^2) per chunk; valid until the host invalidates it
  const bool carried = CARRY && *(volatile const int32_t*)sc.wnext_valid != 0;
  const StepLr slr = step_lr(hy);
  for (int32_t tile = blockIdx.x; tile < wk.ntiles; tile += gridDim.x) {
    __syncthreads();  // shared chunk partials of the previous tile fully consumed
    norms_tile<GL, REG_PATH>(tile, wk, sc, hy, w, gl, sm_cw, sm_cg, &sm_done, &sm_nonfinite, carried, slr, stages,
                             sm_bars, &bulk_q);
  }
  __syncthreads();
  if (hy.defer) {  // no cross-CTA finish here: one flag per CTA, and the iteration K2 will use
    if (threadIdx.x == 0) {
      sc.nf_cta[blockIdx.x] = sm_nonfinite ? 1 : 0;
      if (blockIdx.x == 0 && hy.iter_dev) *sc.step_iter = *(volatile const int64_t*)hy.iter_dev;
    }
    return false;
  }
  // Count this CTA's finished layers once; the CTA that completes the count decides the step's skip.
  if (threadIdx.x == 0 && sm_done > 0u) {
    if (sm_nonfinite) atomicOr(sc.nonfinite, 1u);
    __threadfence();
    const unsigned before = atomicAdd(sc.tensors_done, sm_done);
    if (before + sm_done == (unsigned)wk.ntensors) {
      __threadfence();
      const unsigned nf = atomicExch(sc.nonfinite, 0u);
      *(volatile unsigned*)sc.tensors_done = 0u;
      if (sc.c3) {  // data parallel: the decision is global, taken after the C3 exchange
        *(volatile double*)sc.c3 = nf ? 1.0 : 0.0;
        return true;
      }
      int32_t status = nf ? 1 : 0;
      if (hy.iter_dev) {  // every layer has read the iteration: advance it (graph replays walk the schedule)
        const int64_t t = *(volatile int64_t*)hy.iter_dev;
        if (t < 0 || t >= hy.total_iters) status = 2;
        *(volatile int64_t*)hy.iter_dev = t + 1;
      }
      *(volatile int32_t*)sc.skip = status;
      return true;
    }
  }
  return false;
}

// BULK: a separate instance streaming through bulk-copy stages (its shared-memory attributes — 48 KB of
// dynamic stages, the max-shared carveout — must not touch the register-loop instance, which runs faster
// with the default L1/shared split).
template <int DT, bool CARRY, bool BULK = false>
__global__ void __launch_bounds__(kThreads, kCtasPerSm) lars_norms_kernel(DevWork wk, DevScratch sc, Hyper hy,
                                                                          const float* __restrict__ w,
                                                                          const void* __restrict__ g,
                                                                          int64_t g_shift) {
  // wait, then release the dependent K2 (K2 reads only the static work list before its own wait)
  extern __shared__ __align__(128) unsigned char k1_stages[];  // kBulkSmem bytes when BULK
#if LARS_K1_PREFETCH_LINES > 0
  // while the previous step's K2 drains: pull the head of each warp's first chunk of g into L2 (the work
  // list is static; an L2 prefetch cannot go stale, L2 being the device's point of coherence). fp32 only:
  // for 16-bit gradients it measured slower (profiles/r02_k1_prefetch_sweep.txt)
  if (!BULK && DT == LARS_F32 && (int32_t)blockIdx.x < wk.ntiles) {
    const int32_t c = wk.tile_chunk[blockIdx.x] + (int32_t)(threadIdx.x >> 5);
    if (c < wk.tile_chunk[blockIdx.x + 1]) {
      const Seg ck = wk.chunks[c];
      const char* p = (const char*)g + (ck.begin - g_shift) * 4;
      const int32_t bytes = min(ck.len * 4, LARS_K1_PREFETCH_LINES * 128);
      for (int32_t o = (int32_t)(threadIdx.x & 31) * 128; o < bytes; o += 32 * 128)
        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p + o));
    }
  }
#endif
  pdl_wait();
  pdl_trigger();
  TRACE_BEGIN
  norms_body<CARRY, LocalGrad<DT>, !BULK>(wk, sc, hy, w, LocalGrad<DT>{g, g_shift}, BULK ? k1_stages : nullptr);
  TRACE_END(0)
}

// ---------------------------------------------------------------- K2: fused update
__device__ __forceinline__ void upd8(F8& w, F8& m, const F8& g, float s, float c, float b, float mu, bool apply) {
  if (!apply) {  // reading #2: lr*lambda inside the velocity
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float u = fmaf(b, w.v[i], s * g.v[i]);  // s*g + beta_l*w
      const float v = fmaf(mu, m.v[i], c * u);       // mu*v + lr*lambda*(...)
      w.v[i] = w.v[i] - v;
      m.v[i] = v;
    }
  } else {       // velocity of (s*g + beta_l*w), lr*lambda at the weight step
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float u = fmaf(b, w.v[i], s * g.v[i]);
      const float v = fmaf(mu, m.v[i], u);
      w.v[i] = fmaf(-c, v, w.v[i]);
      m.v[i] = v;
    }
  }
}

__device__ __forceinline__ void accw8(double& a, const F8& x) { acc8(a, x); }

// Extra destinations of the updated weights: none (single GPU / NCCL all-gather), or every other rank's
// weight buffer over NVLink (dp fused path: the all-gather happens as the update is written).
struct NoPeers {
  __device__ __forceinline__ void store8(int64_t, const F8&) const {}
  __device__ __forceinline__ void store1(int64_t, float) const {}
};
struct PeerWeights {
  float* pw[kMaxRanks - 1];  // the other ranks' weight buffers (symmetric window, same flat layout)
  int n;
  __device__ __forceinline__ void store8(int64_t e, const F8& x) const {
    for (int p = 0; p < n; ++p) {
      float* d = pw[p] + e;
      asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(d), "r"(__float_as_uint(x.v[0])),
                   "r"(__float_as_uint(x.v[1])), "r"(__float_as_uint(x.v[2])), "r"(__float_as_uint(x.v[3])),
                   "r"(__float_as_uint(x.v[4])), "r"(__float_as_uint(x.v[5])), "r"(__float_as_uint(x.v[6])),
                   "r"(__float_as_uint(x.v[7]))
                   : "memory");
    }
  }
  __device__ __forceinline__ void store1(int64_t e, float x) const {
    for (int p = 0; p < n; ++p) pw[p][e] = x;
  }
};

// LARS_FLAG_HALF_WEIGHTS: the new weights rounded to the wire dtype (round to nearest even) go to this
// rank's compute-weight buffer and (fused path) every other rank's, 16 B per 8 elements.
template <int HDT>
__device__ __forceinline__ uint32_t pack2_rn(float a, float b) {
  if (HDT == LARS_F16) {
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
  }
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
template <int HDT>
__device__ __forceinline__ uint4 pack8_rn(const F8& x) {
  return make_uint4(pack2_rn<HDT>(x.v[0], x.v[1]), pack2_rn<HDT>(x.v[2], x.v[3]), pack2_rn<HDT>(x.v[4], x.v[5]),
                    pack2_rn<HDT>(x.v[6], x.v[7]));
}
__device__ __forceinline__ void st16(void* p, uint4 v) {
  asm volatile("st.global.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
template <int HDT>
__device__ __forceinline__ uint16_t half_rn(float x) {
  if (HDT == LARS_F16) {
    const __half h = __float2half_rn(x);
    return *reinterpret_cast<const uint16_t*>(&h);
  }
  const __nv_bfloat16 h = __float2bfloat16_rn(x);
  return *reinterpret_cast<const uint16_t*>(&h);
}
template <int HDT>
struct LocalHalf {  // NCCL path: this rank's part of the compute weights (the all-gather follows)
  uint16_t* wh;
  __device__ __forceinline__ void store8(int64_t e, const F8& x) const { st16(wh + e, pack8_rn<HDT>(x)); }
  __device__ __forceinline__ void store1(int64_t e, float x) const { wh[e] = half_rn<HDT>(x); }
};
template <int HDT>
struct PeerHalf {  // fused path: every rank's compute weights, this one's included
  uint16_t* ph[kMaxRanks];
  int n;
  __device__ __forceinline__ void store8(int64_t e, const F8& x) const {
    const uint4 v = pack8_rn<HDT>(x);
    for (int p = 0; p < n; ++p) st16(ph[p] + e, v);
  }
  __device__ __forceinline__ void store1(int64_t e, float x) const {
    const uint16_t v = half_rn<HDT>(x);
    for (int p = 0; p < n; ++p) ph[p][e] = v;
  }
};

// LARS_FLAG_HALF_WEIGHTS on a step that is NOT applied (skipped, or before any applied step): the compute
// weights must still be RNE(master) — a skipped step publishes the unchanged master weights of the work
// list, so the all-gather that follows never spreads stale (or initial zero) compute weights.
template <typename WS>
__device__ __forceinline__ void publish_half_tiles(const DevWork& wk, const float* __restrict__ w, const WS& ws) {
  constexpr int kWarps = kThreads / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int32_t tile = blockIdx.x; tile < wk.ntiles; tile += gridDim.x)
    for (int32_t c = wk.tile_chunk[tile] + warp; c < wk.tile_chunk[tile + 1]; c += kWarps) {
      const Seg ck = wk.chunks[c];
      check_chunk(wk, c, ck);
      const int32_t ng = ck.len >> 3;
      for (int32_t j = lane; j < ng; j += 32) ws.store8(ck.begin + 8 * j, ld8_nc(w + ck.begin + 8 * j));
      for (int32_t i = (ng << 3) + lane; i < ck.len; i += 32) ws.store1(ck.begin + i, w[ck.begin + i]);
    }
}

// NVLS: one multicast store per vector reaches every rank's weight buffer (the NVSwitch replicates it), so
// the SM issues 1x the bytes instead of (P-1)x. multimem.st is at most 128-bit.
struct McastWeights {
  float* mc;  // multicast address of the weight window (ncclGetLsaMultimemPointer)
  __device__ __forceinline__ void store8(int64_t e, const F8& x) const {
    float* d = mc + e;
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(d), "f"(x.v[0]), "f"(x.v[1]),
                 "f"(x.v[2]), "f"(x.v[3]) : "memory");
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(d + 4), "f"(x.v[4]), "f"(x.v[5]),
                 "f"(x.v[6]), "f"(x.v[7]) : "memory");
  }
  __device__ __forceinline__ void store1(int64_t e, float x) const {
    asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(mc + e), "f"(x) : "memory");
  }
};

// One warp chunk of K2 (and F2): unscale + weight decay + momentum + update of <= kChunk elements, every new
// weight also handed to `ws` (the other ranks' buffers on the fused path); carry mode also leaves the chunk's
// sum(w_new^2) for the next step's K1.
// Deferred finish (K2 prologue): the coefficients of the layers of the CTA's current tile, indexed by
// local tensor id - base, and the tile's segment records.
__shared__ float k2_coef[kMaxTileChunks], k2_beta[kMaxTileChunks];
__shared__ __align__(16) SegInfo k2_seg[kMaxTileChunks];

// DEFER: lr*lambda and beta_l come from the CTA's shared copies (k2_coef/k2_beta, index tensor - base),
// otherwise from the scratch arrays K1 (or the split finisher) wrote.
// PAIRS: two 8-element groups per lane per iteration (more stores in flight: the fused F2, whose peer stores
// bound it, measured 1.8 us faster at P = 2) or one (K2: spill-free at 59 registers, 3.0-3.5 us faster).
template <int DT, bool CARRY, typename WS = NoPeers, bool DEFER = false, bool PAIRS = false>
__device__ __forceinline__ void update_chunk(int32_t c, const DevWork& wk, const DevScratch& sc, const Hyper& hy,
                                             float* __restrict__ w, const void* __restrict__ g, int64_t g_shift,
                                             float* __restrict__ m, const WS& ws, int32_t base) {
  const int lane = threadIdx.x & 31;
  const float s = hy.grad_scale_f, mu = hy.mu;
  const Seg ck = wk.chunks[c];
  check_chunk(wk, c, ck);
  const float cf = DEFER ? k2_coef[ck.tensor - base] : sc.coef[ck.tensor];
  const float b = DEFER ? k2_beta[ck.tensor - base] : sc.beta[ck.tensor];
  float* wp = w + ck.begin;
  float* mp = m + ck.begin;
  const int64_t gi = ck.begin - g_shift;
  const int32_t ng = ck.len >> 3;
  double aw = 0.0;  // CARRY: sum(w_new^2) of this chunk for the next step's K1
  for (int32_t i = (ng << 3) + lane; i < ck.len; i += 32) {  // ragged tensor tail (< 8 elements)
    const float wv = wp[i], mv = mp[i];
    const float u = fmaf(b, wv, s * Grad<DT>::load1(g, gi + i));
    const float v = hy.lr_at_apply ? fmaf(mu, mv, u) : fmaf(mu, mv, cf * u);
    const float wn = hy.lr_at_apply ? fmaf(-cf, v, wv) : wv - v;
    wp[i] = wn;
    mp[i] = v;
    ws.store1(ck.begin + i, wn);
    if (CARRY) aw = fma((double)wn, (double)wn, aw);
  }
  int32_t j = ng - 1 - lane;
  for (; PAIRS && j - 32 >= 0; j -= 64) {
    const int32_t j1 = j - 32;
    F8 w0 = ld8_rw(wp + 8 * j), w1 = ld8_rw(wp + 8 * j1);
    const F8 g0 = Grad<DT>::load8(g, gi + 8 * j), g1 = Grad<DT>::load8(g, gi + 8 * j1);
    F8 m0 = ld8_rw(mp + 8 * j), m1 = ld8_rw(mp + 8 * j1);
    upd8(w0, m0, g0, s, cf, b, mu, hy.lr_at_apply);
    upd8(w1, m1, g1, s, cf, b, mu, hy.lr_at_apply);
    st8(wp + 8 * j, w0);
    st8(mp + 8 * j, m0);
    st8(wp + 8 * j1, w1);
    st8(mp + 8 * j1, m1);
    ws.store8(ck.begin + 8 * j, w0);
    ws.store8(ck.begin + 8 * j1, w1);
    if (CARRY) {  // one fp64 accumulator (a second one for ILP cost spills at the 64-register budget)
      accw8(aw, w0);
      accw8(aw, w1);
    }
  }
  for (; j >= 0; j -= 32) {  // (!PAIRS: one 8-element group per lane per iteration throughout)
    F8 w0 = ld8_rw(wp + 8 * j), m0 = ld8_rw(mp + 8 * j);
    const F8 g0 = Grad<DT>::load8(g, gi + 8 * j);
    upd8(w0, m0, g0, s, cf, b, mu, hy.lr_at_apply);
    st8(wp + 8 * j, w0);
    st8(mp + 8 * j, m0);
    ws.store8(ck.begin + 8 * j, w0);
    if (CARRY) accw8(aw, w0);
  }
  if (CARRY) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) aw += __shfl_xor_sync(0xffffffffu, aw, o);
    if (lane == 0) sc.cpart_wnext[c] = aw;
  }
}

template <int DT, bool CARRY, typename WS = NoPeers, bool DEFER = false, bool PAIRS = false>
__device__ __forceinline__ void update_item(int32_t item, const DevWork& wk, const DevScratch& sc, const Hyper& hy,
                                            float* __restrict__ w, const void* __restrict__ g, int64_t g_shift,
                                            float* __restrict__ m, const WS& ws = WS(), int32_t base = 0) {
  constexpr int kWarps = kThreads / 32;
  const int warp = threadIdx.x >> 5;
  // item -> (part q, tile): all tiles' last parts first (the bytes K1 read last, still in L2), then the
  // next-to-last parts, ...; inside a part the chunks run backwards.
  const int32_t q = kUpdateSplit - 1 - item / wk.ntiles, tile = item % wk.ntiles;
  const int32_t t0 = wk.tile_chunk[tile], tn = wk.tile_chunk[tile + 1] - t0;
  const int32_t c0 = t0 + (int32_t)((int64_t)tn * q / kUpdateSplit);
  const int32_t c1 = t0 + (int32_t)((int64_t)tn * (q + 1) / kUpdateSplit);
  LARS_DCHECK(tile >= 0 && tile < wk.ntiles && q >= 0 && q < kUpdateSplit && c0 <= c1 && c1 <= wk.nchunks);
  for (int32_t c = c1 - 1 - warp; c >= c0; c -= kWarps)  // backwards: K1's most recent reads first
    update_chunk<DT, CARRY, WS, DEFER, PAIRS>(c, wk, sc, hy, w, g, g_shift, m, ws, base);
}

// Deferred finish (single GPU, hy.defer). K1 has left every segment's partial sums, one non-finite flag
// per K1 CTA and (device iteration) the step's iteration. Before griddepcontrol.wait (while K1 drains) a
// K2 CTA copies its tile's segment records (static work list) into shared memory; after the wait it reads
// the flags and the partials of its tile's layers — one round of loads.
// The step is skipped when any flag is set (a layer norm is non-finite exactly when one of its partials is:
// the partials are sums of <= 2^31 fp32 squares and |s| <= 2^64, so no finite sum overflows the norm) or the
// iteration is out of range; every CTA takes the same decision, CTA 0 records it and advances a device
// iteration (every K1 CTA has read it; the next K1 reads it after this grid completes).
__device__ __forceinline__ void deferred_prefetch_segs(int32_t tile, const DevWork& wk) {
  SegInfo* sm_seg = k2_seg;
  const int32_t s0 = wk.tile_seg[tile], n = wk.tile_seg[tile + 1] - s0;
  LARS_DCHECK(n >= 1 && n <= kMaxTileChunks);
  for (int32_t i = threadIdx.x; i < 2 * n; i += blockDim.x)
    cp_async16((char*)(sm_seg + i / 2) + 16 * (i & 1), (const char*)(wk.seginfo + s0 + i / 2) + 16 * (i & 1));
}

__device__ __forceinline__ bool deferred_skip(const DevWork& wk, const DevScratch& sc, const Hyper& hy, int bad) {
  bad = __syncthreads_or(bad);
  const int64_t t = hy.iter_dev ? __ldcg(sc.step_iter) : hy.iter;
  const bool in_range = t >= 0 && t < hy.total_iters;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *(volatile int32_t*)sc.skip = !in_range ? 2 : bad ? 1 : 0;
    if (hy.iter_dev) *(volatile int64_t*)hy.iter_dev = t + 1;
  }
  return bad || !in_range;
}

// The layers of `tile` (its segments, one per layer, consecutive local tensor ids; records in sm_seg): each
// layer's norms from ALL its segment partials in the same fixed order as K1's own finish (lane-strided sum,
// xor butterfly: every CTA that touches the layer computes the same bits), then lambda and lr*lambda into
// the CTA's shared arrays (index = tensor - base, base returned). The CTA holding a layer's first segment
// also writes the layer's outputs (lars_last_norms). `first`: also reduce the K1 flags into the skip decision
// (their loads are issued beside the partials').
__device__ __forceinline__ int32_t deferred_finish_tile(int32_t tile, const DevWork& wk, const DevScratch& sc,
                                                        const Hyper& hy, bool first, bool* skip) {
  const SegInfo* sm_seg = k2_seg;
  float* sm_coef = k2_coef;
  float* sm_beta = k2_beta;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int32_t s0 = wk.tile_seg[tile], s1 = wk.tile_seg[tile + 1];
  // every load of the prologue is issued before any of them is used: the K1 flags (first tile; OR-ed at
  // the end), the iteration, then — once the segment records are in — the partials
  int f0 = 0, f1 = 0, f2 = 0;
  if (first) {
    const int32_t i = threadIdx.x;
    if (i < wk.grid) f0 = __ldcg(sc.nf_cta + i);
    if (i + kThreads < wk.grid) f1 = __ldcg(sc.nf_cta + i + kThreads);
    if (i + 2 * kThreads < wk.grid) f2 = __ldcg(sc.nf_cta + i + 2 * kThreads);
    for (int32_t j = i + 3 * kThreads; j < wk.grid; j += kThreads) f2 |= __ldcg(sc.nf_cta + j);
  }
  const int64_t t = hy.iter_dev ? __ldcg(sc.step_iter) : hy.iter;
  const bool in_range = t >= 0 && t < hy.total_iters;
  const double lr = !in_range ? 0.0 : hy.iter_dev ? hy.lr_table[t] : hy.lr_host;
  cp_async_wait_all();
  __syncthreads();  // the tile's segment records are in shared memory
  if (first) {
    TRACE_MARK_AT(5, 1)
  }
  const int32_t base = sm_seg[0].tensor;
  const int32_t n = s1 - s0;
  auto finish = [&](int32_t k, const SegInfo& si, double sw, double sg) {
    const double wn = sqrt(sw), gn = fabs(hy.grad_scale) * sqrt(sg);
    double lam = 1.0, beta = 0.0;
    if (si.lars) {  // reading #1, #3, #4 (same arithmetic as finish_core)
      beta = hy.weight_decay;
      const double den = gn + hy.weight_decay * wn + hy.eps;
      if (wn > 0.0 && den > hy.eps) lam = hy.eta * wn / den;
    }
    const float cf = in_range ? (float)(lr * lam) : 0.0f;
    sm_coef[k] = cf;
    sm_beta[k] = (float)beta;
    if (s0 + k == si.tseg_begin) {
      const int32_t l = si.tensor;
      sc.w_norm[l] = wn;
      sc.g_norm[l] = gn;
      sc.lambda[l] = lam;
      sc.coef[l] = cf;
      sc.beta[l] = (float)beta;
    }
  };
  // A tile's interior segments are whole layers (one partial each): one thread per layer, all loads at once.
  for (int32_t k = threadIdx.x; k < n; k += blockDim.x) {
    const SegInfo si = sm_seg[k];
    LARS_DCHECK(si.tensor - base == k && k < kMaxTileChunks);
    LARS_DCHECK(si.nseg == 1 || k == 0 || k == n - 1);
    if (si.nseg == 1) finish(k, si, __ldcg(sc.part_w + si.tseg_begin), __ldcg(sc.part_g + si.tseg_begin));
  }
  if (first) {
    TRACE_MARK_AT(5, 2)
  }
  // Only the first and the last segment can belong to a layer spread over several tiles: the two last warps
  // (idle in the pass above unless the tile has > 192 layers) sum those layers' partials (the fixed order
  // of K1's own finish).
  constexpr int kW0 = kThreads / 32 - 2;
  if (warp >= kW0 && (warp == kW0 || n > 1)) {
    const int32_t k = warp == kW0 ? 0 : n - 1;
    const SegInfo si = sm_seg[k];
    if (si.nseg > 1) {
      double sw, sg;
      warp_sum2(sc.part_w, sc.part_g, si.tseg_begin, si.tseg_begin + si.nseg, lane, sw, sg);
      if (lane == 0) finish(k, si, sw, sg);
    }
  }
  if (first) *skip = deferred_skip(wk, sc, hy, f0 | f1 | f2);  // (its __syncthreads_or also publishes sm_coef)
  else __syncthreads();
  return base;
}

// K2. Same persistent schedule as K1 (CTA b owns tiles b, b + grid, ...; identical grid and resources,
// so CTA b runs on the same SM in both kernels) and each tile's chunks walked backwards: the gradient
// bytes K1 streamed last into this SM's L2 slice are re-read first.
template <int DT, bool CARRY, bool HALF = false, bool DEFER = false>
__global__ void __launch_bounds__(kThreads, kCtasPerSm) lars_update_kernel(DevWork wk, DevScratch sc, Hyper hy,
                                                                           float* __restrict__ w,
                                                                           const void* __restrict__ g,
                                                                           int64_t g_shift, float* __restrict__ m) {
  static_assert(!(HALF && DEFER), "the deferred finish is the whole-layout step's");
  pdl_trigger();
  if constexpr (DEFER) deferred_prefetch_segs(blockIdx.x, wk);  // static work list: before the wait
#if LARS_K2_PREFETCH_LINES > 0
  // while K1 drains: pull the head of w and m of each warp's first chunk (the tile's last) into L2. Both
  // were last written by the previous K2, complete before K1 passed its own wait and released this grid.
  // fp32 gradients only: 16-bit measured +0.7 us (profiles/r02_k2_prefetch_sweep.txt)
  if (!HALF && DT == LARS_F32 && (int32_t)blockIdx.x < wk.ntiles) {
    const int32_t c = wk.tile_chunk[blockIdx.x + 1] - 1 - (int32_t)(threadIdx.x >> 5);
    if (c >= wk.tile_chunk[blockIdx.x]) {
      const Seg ck = wk.chunks[c];
      const int32_t bytes = min(ck.len * 4, LARS_K2_PREFETCH_LINES * 128);
      for (int32_t o = (int32_t)(threadIdx.x & 31) * 128; o < bytes; o += 32 * 128) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)(w + ck.begin) + o));
        asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)(m + ck.begin) + o));
      }
    }
  }
#endif
  pdl_wait();
  bool skip = false;
  TRACE_BEGIN
  if constexpr (DEFER) {
    for (int32_t tile = blockIdx.x; tile < wk.ntiles; tile += gridDim.x) {
      const bool first = tile == (int32_t)blockIdx.x;
      if (!first) deferred_prefetch_segs(tile, wk);
      const int32_t base = deferred_finish_tile(tile, wk, sc, hy, first, &skip);
      if (first) {
        TRACE_MARK_AT(5, 0)  // (diagnostics build) prologue done
      }
      if (!skip)
        for (int32_t q = kUpdateSplit - 1; q >= 0; --q)
          update_item<DT, CARRY, NoPeers, true>((kUpdateSplit - 1 - q) * wk.ntiles + tile, wk, sc, hy, w, g, g_shift,
                                                m, NoPeers(), base);
      __syncthreads();  // the tile's coefficients are consumed before the next tile's overwrite them
    }
  } else {
    skip = *(volatile const int32_t*)sc.skip != 0;  // whole step skipped (non-finite norm)
    if (!skip)
      for (int32_t tile = blockIdx.x; tile < wk.ntiles; tile += gridDim.x)
        for (int32_t q = kUpdateSplit - 1; q >= 0; --q)
          if constexpr (HALF)
            update_item<DT, CARRY, LocalHalf<DT>>((kUpdateSplit - 1 - q) * wk.ntiles + tile, wk, sc, hy, w, g,
                                                  g_shift, m, LocalHalf<DT>{(uint16_t*)hy.w_half});
          else
            update_item<DT, CARRY>((kUpdateSplit - 1 - q) * wk.ntiles + tile, wk, sc, hy, w, g, g_shift, m);
  }
  if constexpr (HALF)
    if (skip) publish_half_tiles(wk, w, LocalHalf<DT>{(uint16_t*)hy.w_half});
  // every chunk's sum(w_new^2) is written once this grid completes; the next K1 (stream-ordered after
  // the whole grid) may use them. A skipped step leaves w — and therefore the old sums — valid.
  if (CARRY && !skip && blockIdx.x == 0 && threadIdx.x == 0) *(volatile int32_t*)sc.wnext_valid = 1;
  TRACE_END(1)
}

// A rank that owns no layer still advances a device iteration and reports its range check.
__global__ void empty_step_kernel(int64_t* iter_dev, int64_t total_iters, int32_t* skip) {
  const int64_t t = *iter_dev;
  *skip = (t < 0 || t >= total_iters) ? 2 : 0;
  *iter_dev = t + 1;
}

// Data-parallel finish, after C3 = allreduce(sum) of [non-finite count, split-layer partial sums]:
// every rank sees the same global sums, so every rank takes the same skip decision (reading #13) and
// each rank finishes the split layers it touches exactly like K1 finishes whole ones.
// Consumes the global C3 sums in sc.c3 (one warp): every rank sees the same sums, so every rank takes the
// same decision; zeroes sc.c3 for the next step's shares.
__device__ __forceinline__ void split_finish_body(const DevWork& wk, const DevScratch& sc, const Hyper& hy) {
  const int lane = threadIdx.x;
  const int32_t n = 1 + 2 * wk.nsplit_total;
  bool bad = false;
  for (int32_t i = lane; i < n; i += 32) {
    const double x = sc.c3[i];
    bad |= (i == 0) ? (x > 0.0) : !isfinite(x);
  }
  for (int32_t k = lane; k < wk.nsplit_local; k += 32) {
    const int32_t l = wk.split_locals[k], j = wk.tsplit[l];
    bad |= finish_core(l, sc.c3[1 + 2 * j], sc.c3[2 + 2 * j], wk, sc, hy);
  }
  bad = __any_sync(0xffffffffu, bad);
  __syncwarp();
  for (int32_t i = lane; i < n; i += 32) sc.c3[i] = 0.0;  // next step's shares start from zero
  if (lane == 0) {
    int32_t status = bad ? 1 : 0;
    if (hy.iter_dev) {
      const int64_t t = *hy.iter_dev;
      if (t < 0 || t >= hy.total_iters) status = 2;
      *hy.iter_dev = t + 1;
    }
    *sc.skip = status;
  }
}

__global__ void lars_split_finish_kernel(DevWork wk, DevScratch sc, Hyper hy) { split_finish_body(wk, sc, hy); }

// ---------------------------------------------------------------- fused data-parallel path (NEXT-f1)
// Gradient and weight buffers live in NCCL symmetric windows (ncclMemAlloc + ncclCommWindowRegister), so
// every rank can load and store every other rank's buffers over NVLink with plain ld/st (LSA pointers).
// The reduce-scatter is fused into K1 (each rank sums its shard over all ranks' gradients in fp32), the
// C3 exchange rides on F1's tail and F2's head (epoch-tagged words, no extra kernel), and the all-gather is fused
// into K2 (each updated weight is stored locally and into every peer). One LSA barrier at F1's entry (taken by
// CTA 0) and one at F2's exit (taken by the last CTA) order the steps across ranks.
//
//   F1 lars_dp_reduce_norms_kernel : barrier(b) -> shard sum over ranks + norms; the final CTA publishes
//                                    this rank's C3 shares into every rank's exchange slot (epoch-tagged words)
//   F2 lars_dp_update_gather_kernel: wait for all ranks' shares, fixed-order sum, finish split layers, skip
//                                    -> update + store w to every peer -> barrier(b)
// The C3 shares [non-finite flag, split-layer sums] travel as EPOCH-TAGGED words: value i of rank p lands in
// slot p of every rank's exchange window as two 64-bit words, (epoch << 32) | low 32 bits and
// (epoch << 32) | high 32 bits of the double. Every word is written and read whole (single-copy atomic), so
// a reader that sees the step's epoch in a word has that word's payload: no release fence and no separate
// flag, i.e. no NVLink round trip on the critical path between F1's last tile and F2's start (the
// fence + flag protocol cost ~4 us here). Epochs only grow (the 32-bit tag wraps after 4e9 steps).
__device__ __forceinline__ unsigned long long share_word(uint32_t epoch, uint32_t half) {
  return ((unsigned long long)epoch << 32) | half;
}

// End of F1 (one thread): this rank's shares go into slot [rank] of every rank's exchange window. The
// iteration of this step is recorded (and a device iteration advanced) here, after every layer of this rank
// has read it.
__device__ void dp_publish_shares(const DevWork& wk, const DevScratch& sc, const Hyper& hy, const DpFused& f) {
  // one warp: every (rank, value) word pair by its own lane, all loads of the shares in flight at once
  const int lane = threadIdx.x & 31;
  const int32_t n = 1 + 2 * wk.nsplit_total;
  unsigned long long epoch = 0;
  if (lane == 0) {
    epoch = *f.epoch + 1ull;
    *f.epoch = epoch;
    const int64_t t = hy.iter_dev ? *(volatile int64_t*)hy.iter_dev : hy.iter;
    *f.step_iter = t;
    if (hy.iter_dev) *(volatile int64_t*)hy.iter_dev = t + 1;
  }
  const uint32_t e32 = (uint32_t)__shfl_sync(0xffffffffu, epoch, 0);
  for (int32_t k = lane; k < f.nranks * n; k += 32) {
    const int p = k / n, i = k % n;
    const unsigned long long bits = (unsigned long long)__double_as_longlong(__ldcg(sc.c3 + i));
    unsigned long long* slot =
        (unsigned long long*)ncclGetLsaPointer(f.xwin, (size_t)f.rank * 2 * n * sizeof(unsigned long long), p);
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_system> lo(slot[2 * i]), hi(slot[2 * i + 1]);
    lo.store(share_word(e32, (uint32_t)bits), cuda::memory_order_relaxed);
    hi.store(share_word(e32, (uint32_t)(bits >> 32)), cuda::memory_order_relaxed);
  }
  __syncwarp();  // every lane has read the shares
  for (int32_t i = lane; i < n; i += 32) sc.c3[i] = 0.0;  // next step's shares start from zero
}

// Start of F2 (warp 0 of every CTA): wait until every word of every rank's shares carries this step's
// epoch, sum the shares in rank order (identical on every rank), finish the split layers this rank touches,
// decide the skip. Returns the step status (0 apply, 1 non-finite, 2 iteration out of range) to every lane
// of warp 0.
// The split layer lane k of warp 0 finishes (static work list: loaded before F2's griddepcontrol.wait, so the
// chain split_locals -> tsplit -> tlars is off the critical path).
struct SplitPre {
  int32_t l = -1, j = 0, lars = 0;
};
__device__ __forceinline__ SplitPre load_split_pre(const DevWork& wk) {
  SplitPre sp;
  const int lane = threadIdx.x & 31;
  LARS_DCHECK(wk.nsplit_local <= 32);
  if (lane < wk.nsplit_local) {
    sp.l = wk.split_locals[lane];
    sp.j = wk.tsplit[sp.l];
    sp.lars = wk.tlars[sp.l];
  }
  return sp;
}

__device__ int32_t dp_collect_shares(const DevWork& wk, const DevScratch& sc, const Hyper& hy, const DpFused& f,
                                     const SplitPre& sp) {
  const int lane = threadIdx.x & 31;
  const int32_t n = 1 + 2 * wk.nsplit_total;
  const uint32_t e32 = (uint32_t)*(volatile unsigned long long*)f.epoch;
  // the step's iteration as recorded by F1 (a device iteration has moved on already); its lr(t) from the host
  // unless the iteration lives on the device
  const int64_t t = *(volatile const int64_t*)f.step_iter;
  unsigned long long* x = (unsigned long long*)ncclGetLocalPointer(f.xwin, 0);
  for (int32_t k = lane; k < f.nranks * 2 * n; k += 32) {
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_system> word(x[k]);
    while ((uint32_t)(word.load(cuda::memory_order_relaxed) >> 32) != e32) __nanosleep(32);
  }
  __syncwarp();
  TRACE_MARK_AT(6, 1)
  auto val = [&](int p, int32_t i) {  // every word of this step is in: plain reads
    const unsigned long long* w = x + ((size_t)p * n + i) * 2;
    const unsigned long long lo = *(volatile const unsigned long long*)w, hi = *(volatile const unsigned long long*)(w + 1);
    return __longlong_as_double((long long)((hi << 32) | (lo & 0xffffffffull)));
  };
  bool bad = false;
  for (int32_t i = lane; i < n; i += 32) {
    double tot = 0.0;
    for (int p = 0; p < f.nranks; ++p) tot += val(p, i);  // rank order
    bad |= (i == 0) ? (tot > 0.0) : !isfinite(tot);
  }
  const bool in_range = t >= 0 && t < hy.total_iters;
  if (sp.l >= 0) {
    double sw = 0.0, sg = 0.0;
    for (int p = 0; p < f.nranks; ++p) {
      sw += val(p, 1 + 2 * sp.j);
      sg += val(p, 2 + 2 * sp.j);
    }
    const StepLr slr{!in_range ? 0.0 : hy.iter_dev ? hy.lr_table[t] : hy.lr_host, in_range};
    bad |= finish_core(sp.l, sp.lars, sw, sg, sc, hy, slr);  // identical values from every CTA (benign duplicates)
  }
  bad = __any_sync(0xffffffffu, bad);
  return !in_range ? 2 : bad ? 1 : 0;
}

// BULK: the rank sum streams through bulk-copy stages (stream_tile_bulk; peer reads by the TMA engine, no
// registers per byte in flight), so every peer-count instance fits 4 CTAs per SM.
template <int DT, bool CARRY, int NP, bool BULK>
__global__ void __launch_bounds__(kThreads, BULK ? kCtasPerSm : dp_norm_ctas_per_sm(NP))
    lars_dp_reduce_norms_kernel(DevWork wk, DevScratch sc, Hyper hy, const float* w, DpFused f) {
  extern __shared__ __align__(128) unsigned char f1_stages[];  // kBulkSmem bytes when BULK
  TRACE_BEGIN
  pdl_trigger();  // F2's CTAs may be scheduled as F1's retire (they wait in griddepcontrol.wait)
  pdl_wait();
  // Entry: every rank's gradient for this step is complete once every rank's F1 is running. CTA 0 alone
  // syncs with the other ranks (one LSA barrier instead of one per CTA); the others wait for its go flag.
  // The step epoch cannot move during the entry: it is advanced by the CTA that completes the layer
  // count, which needs every tile-owning CTA past its entry. A CTA that owns no tile (the launcher caps
  // the grid at one CTA per tile; this guards any other grid) leaves before reading the epoch: it could
  // otherwise read the NEXT epoch and wait for a go flag that never comes.
  if (blockIdx.x != 0 && (int32_t)blockIdx.x >= wk.ntiles) return;
  {
    const unsigned long long E = *(volatile const unsigned long long*)f.epoch;
    if (blockIdx.x == 0) {
      ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), f.dc, ncclTeamTagLsa(), 0);
      bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
      if (threadIdx.x == 0) {
        cuda::atomic_ref<unsigned long long, cuda::thread_scope_system> go(*f.go);
        go.store(E + 1, cuda::memory_order_release);
      }
    } else {
      if (threadIdx.x == 0) {
        cuda::atomic_ref<unsigned long long, cuda::thread_scope_system> go(*f.go);
        while (go.load(cuda::memory_order_acquire) < E + 1) __nanosleep(32);
      }
    }
    __syncthreads();
  }
  TRACE_MARK(5)
  LARS_DCHECK(f.nranks >= 1 && f.nranks <= NP && f.rank >= 0 && f.rank < f.nranks);
  PeerSumGrad<DT, NP> gl;
#pragma unroll
  for (int p = 0; p < NP; ++p) gl.gp[p] = p < f.nranks ? ncclGetLsaPointer(f.gwin, 0, p) : nullptr;
  gl.nranks = f.nranks;
  gl.gred = f.gred;
  gl.begin = f.begin;
  // static tiles (one per CTA): measured faster than 4x finer dynamically scheduled tiles, whose per-tile
  // overhead outweighs the shorter tail (tools/trace_dp.py)
  const bool final_cta = norms_body<CARRY, PeerSumGrad<DT, NP>, !BULK>(wk, sc, hy, w, gl, BULK ? f1_stages : nullptr);
  TRACE_MARK(4)
  __shared__ int s_publish;
  if (threadIdx.x == 0) s_publish = final_cta || (wk.ntensors == 0 && blockIdx.x == 0);
  __syncthreads();
  if (s_publish && threadIdx.x < 32) dp_publish_shares(wk, sc, hy, f);
  __syncthreads();
  TRACE_END(2)
}

template <bool CARRY, bool MCAST, int HDT = 0>  // HDT: compute-weight dtype (LARS_FLAG_HALF_WEIGHTS), 0 = fp32 all-gather
__global__ void __launch_bounds__(kThreads, kCtasPerSm) lars_dp_update_gather_kernel(DevWork wk, DevScratch sc,
                                                                                     Hyper hy, float* w, float* m,
                                                                                     DpFused f) {
  __shared__ int32_t s_status;
  TRACE_BEGIN
  pdl_trigger();
  SplitPre sp;
  if (threadIdx.x < 32) sp = load_split_pre(wk);
#if LARS_F2_PREFETCH_LINES > 0
  // while F1 drains: the head of w and m of each warp's first chunk into L2 (as K2; this rank's shard of
  // w and m is written only by this rank's previous F2, complete before F1 started)
  if ((int32_t)blockIdx.x < wk.ntiles) {
    const int32_t c = wk.tile_chunk[blockIdx.x + 1] - 1 - (int32_t)(threadIdx.x >> 5);
    if (c >= wk.tile_chunk[blockIdx.x]) {
      const Seg ck = wk.chunks[c];
      const int32_t bytes = min(ck.len * 4, LARS_F2_PREFETCH_LINES * 128);
      for (int32_t o = (int32_t)(threadIdx.x & 31) * 128; o < bytes; o += 32 * 128) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)(w + ck.begin) + o));
        asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)(m + ck.begin) + o));
      }
    }
  }
#endif
  pdl_wait();  // F1 complete (its shares and reduced shard are visible)
  TRACE_MARK_AT(6, 0)
  if (threadIdx.x < 32) {
    const int32_t st = dp_collect_shares(wk, sc, hy, f, sp);
    if (threadIdx.x == 0) {
      s_status = st;
      if (blockIdx.x == 0) *(volatile int32_t*)sc.skip = st;
    }
  }
  __syncthreads();
  TRACE_MARK_AT(4, 0)
  const bool skip = s_status != 0;
  if constexpr (HDT != 0) {
    if (skip) {  // the compute weights stay RNE(master) on every rank
      PeerHalf<HDT> ws;
      ws.n = f.nranks;
      for (int p = 0; p < f.nranks; ++p) ws.ph[p] = (uint16_t*)ncclGetLsaPointer(f.hwin, 0, p);
      publish_half_tiles(wk, w, ws);
    }
  }
  // items ordered last-part-of-every-tile first (see update_item), striped statically over this grid
  if (!skip) {
    if constexpr (HDT != 0) {  // half-precision compute weights to every rank (this one included)
      PeerHalf<HDT> ws;
      ws.n = f.nranks;
      for (int p = 0; p < f.nranks; ++p) ws.ph[p] = (uint16_t*)ncclGetLsaPointer(f.hwin, 0, p);
      for (int32_t item = blockIdx.x; item < wk.ntiles * kUpdateSplit; item += gridDim.x)
        update_item<LARS_F32, CARRY, PeerHalf<HDT>, false, true>(item, wk, sc, hy, w, f.gred, f.begin, m, ws);
    } else if (MCAST) {
      const McastWeights ws{(float*)ncclGetLsaMultimemPointer(f.wwin, 0, f.dc)};
      for (int32_t item = blockIdx.x; item < wk.ntiles * kUpdateSplit; item += gridDim.x)
        update_item<LARS_F32, CARRY, McastWeights, false, true>(item, wk, sc, hy, w, f.gred, f.begin, m, ws);
    } else {
      PeerWeights ws;
      ws.n = 0;
      for (int p = 0; p < f.nranks; ++p)
        if (p != f.rank) ws.pw[ws.n++] = (float*)ncclGetLsaPointer(f.wwin, 0, p);
      for (int32_t item = blockIdx.x; item < wk.ntiles * kUpdateSplit; item += gridDim.x)
        update_item<LARS_F32, CARRY, PeerWeights, false, true>(item, wk, sc, hy, w, f.gred, f.begin, m, ws);
    }
  }
  if (MCAST) asm volatile("fence.acq_rel.sys;" ::: "memory");  // multicast stores before the barrier release
  if (CARRY && !skip && blockIdx.x == 0 && threadIdx.x == 0) *(volatile int32_t*)sc.wnext_valid = 1;
  __syncthreads();
  TRACE_END(3)
  // Exit: after this grid every rank's w must be complete. Each CTA makes its peer stores visible and
  // counts itself out; the last CTA of the grid syncs with the other ranks' last CTAs (one LSA barrier).
  __shared__ int s_last;
  if (threadIdx.x == 0) {
    __threadfence_system();
    s_last = atomicAdd(f.done, 1u) == gridDim.x - 1;
    if (s_last) *(volatile unsigned*)f.done = 0u;
  }
  __syncthreads();
  if (s_last) {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), f.dc, ncclTeamTagLsa(), 0);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  }
}

template <int DT, bool CARRY, bool BULK>
static void launch_reduce_norms_np(int np, int grid, cudaStream_t st, const DevWork& wk, const DevScratch& sc,
                                   const Hyper& hy, const float* w, const DpFused& f) {
  // cooperative: every CTA waits for CTA 0's entry flag, so the whole grid must be co-resident
  const size_t smem = BULK ? kBulkSmem : 0;
#ifndef LARS_F1_COOP
#define LARS_F1_COOP 1
#endif
  if (np <= 2)
    launch_pdl_smem(lars_dp_reduce_norms_kernel<DT, CARRY, 2, BULK>, grid, st, LARS_F1_COOP, smem, wk, sc, hy, w, f);
  else if (np <= 4)
    launch_pdl_smem(lars_dp_reduce_norms_kernel<DT, CARRY, 4, BULK>, grid, st, LARS_F1_COOP, smem, wk, sc, hy, w, f);
  else
    launch_pdl_smem(lars_dp_reduce_norms_kernel<DT, CARRY, 8, BULK>, grid, st, LARS_F1_COOP, smem, wk, sc, hy, w, f);
}

// Bulk-copy instances: static + dynamic shared memory exceeds the 48 KB a kernel gets without opting in,
// and 4 CTAs x ~53 KB per SM need the largest shared-memory carveout.
template <typename K>
static void prefer_shared(K kernel) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBulkSmem);
  cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
}

template <int DT, bool CARRY, bool BULK>
static int reduce_norms_occupancy_np(int np) {
  int n = 0;
  cudaError_t e;
  const size_t smem = BULK ? kBulkSmem : 0;
  if (BULK) {
    prefer_shared(lars_dp_reduce_norms_kernel<DT, CARRY, 2, BULK>);
    prefer_shared(lars_dp_reduce_norms_kernel<DT, CARRY, 4, BULK>);
    prefer_shared(lars_dp_reduce_norms_kernel<DT, CARRY, 8, BULK>);
  }
  if (np <= 2)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, lars_dp_reduce_norms_kernel<DT, CARRY, 2, BULK>, kThreads, smem);
  else if (np <= 4)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, lars_dp_reduce_norms_kernel<DT, CARRY, 4, BULK>, kThreads, smem);
  else
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, lars_dp_reduce_norms_kernel<DT, CARRY, 8, BULK>, kThreads, smem);
  return e == cudaSuccess ? n : 0;
}

template <bool BULK>
static int dp_blocks_per_sm(int32_t dt, bool carry, int np) {
  if (carry) {
    if (dt == LARS_F32) return reduce_norms_occupancy_np<LARS_F32, true, BULK>(np);
    if (dt == LARS_F16) return reduce_norms_occupancy_np<LARS_F16, true, BULK>(np);
    return reduce_norms_occupancy_np<LARS_BF16, true, BULK>(np);
  }
  if (dt == LARS_F32) return reduce_norms_occupancy_np<LARS_F32, false, BULK>(np);
  if (dt == LARS_F16) return reduce_norms_occupancy_np<LARS_F16, false, BULK>(np);
  return reduce_norms_occupancy_np<LARS_BF16, false, BULK>(np);
}
int dp_reduce_norms_blocks_per_sm(int32_t dt, bool carry, int np, bool bulk) {
  return bulk ? dp_blocks_per_sm<true>(dt, carry, np) : dp_blocks_per_sm<false>(dt, carry, np);
}

template <bool BULK>
static void launch_reduce_norms_b(int32_t dt, bool carry, int np, int grid, cudaStream_t st, const DevWork& wk,
                                  const DevScratch& sc, const Hyper& hy, const float* w, const DpFused& f) {
  if (carry) {
    if (dt == LARS_F32) launch_reduce_norms_np<LARS_F32, true, BULK>(np, grid, st, wk, sc, hy, w, f);
    else if (dt == LARS_F16) launch_reduce_norms_np<LARS_F16, true, BULK>(np, grid, st, wk, sc, hy, w, f);
    else launch_reduce_norms_np<LARS_BF16, true, BULK>(np, grid, st, wk, sc, hy, w, f);
  } else {
    if (dt == LARS_F32) launch_reduce_norms_np<LARS_F32, false, BULK>(np, grid, st, wk, sc, hy, w, f);
    else if (dt == LARS_F16) launch_reduce_norms_np<LARS_F16, false, BULK>(np, grid, st, wk, sc, hy, w, f);
    else launch_reduce_norms_np<LARS_BF16, false, BULK>(np, grid, st, wk, sc, hy, w, f);
  }
}
static void launch_reduce_norms(int32_t dt, bool carry, int np, int grid, cudaStream_t st, const DevWork& wk,
                                const DevScratch& sc, const Hyper& hy, const float* w, const DpFused& f) {
  if (f.bulk) launch_reduce_norms_b<true>(dt, carry, np, grid, st, wk, sc, hy, w, f);
  else launch_reduce_norms_b<false>(dt, carry, np, grid, st, wk, sc, hy, w, f);
}

cudaError_t launch_dp_fused(int32_t dt, const DevWork& wk, const DevScratch& sc, const Hyper& hy, float* w, float* m,
                            const DpFused& f, int grid_norm, int grid_update, cudaStream_t st, cudaEvent_t ev1,
                            cudaEvent_t ev2) {
  DevWork wg = wk;
  grid_norm = std::min(grid_norm, std::max(wk.ntiles, 1));  // one CTA per tile (F1's entry relies on it)
  wg.grid = grid_norm;
  launch_reduce_norms(dt, hy.carry, f.np_template, grid_norm, st, wg, sc, hy, w, f);
  if (ev1) cudaEventRecord(ev1, st);
  if (ev2) cudaEventRecord(ev2, st);  // (the exchange now lives inside F1's tail and F2's head)
  if (f.hwin) {
    if (dt == LARS_F16) {
      if (hy.carry) launch_pdl(lars_dp_update_gather_kernel<true, false, LARS_F16>, grid_update, st, wg, sc, hy, w, m, f);
      else launch_pdl(lars_dp_update_gather_kernel<false, false, LARS_F16>, grid_update, st, wg, sc, hy, w, m, f);
    } else {
      if (hy.carry) launch_pdl(lars_dp_update_gather_kernel<true, false, LARS_BF16>, grid_update, st, wg, sc, hy, w, m, f);
      else launch_pdl(lars_dp_update_gather_kernel<false, false, LARS_BF16>, grid_update, st, wg, sc, hy, w, m, f);
    }
  } else if (hy.carry) {
    if (f.mcast) launch_pdl(lars_dp_update_gather_kernel<true, true>, grid_update, st, wg, sc, hy, w, m, f);
    else launch_pdl(lars_dp_update_gather_kernel<true, false>, grid_update, st, wg, sc, hy, w, m, f);
  } else {
    if (f.mcast) launch_pdl(lars_dp_update_gather_kernel<false, true>, grid_update, st, wg, sc, hy, w, m, f);
    else launch_pdl(lars_dp_update_gather_kernel<false, false>, grid_update, st, wg, sc, hy, w, m, f);
  }
  return cudaGetLastError();
}

cudaError_t launch_split_finish(const DevWork& wk, const DevScratch& sc, const Hyper& hy, cudaStream_t st) {
  lars_split_finish_kernel<<<1, 32, 0, st>>>(wk, sc, hy);
  return cudaGetLastError();
}

template <int HDT>
__global__ void __launch_bounds__(kThreads) lars_publish_half_kernel(DevWork wk, const float* __restrict__ w,
                                                                    uint16_t* __restrict__ wh) {
  publish_half_tiles(wk, w, LocalHalf<HDT>{wh});
}

cudaError_t launch_publish_half(int32_t dt, const DevWork& wk, const float* w, void* w_half, cudaStream_t st) {
  if (wk.ntiles == 0) return cudaSuccess;
  if (dt == LARS_F16) lars_publish_half_kernel<LARS_F16><<<wk.grid, kThreads, 0, st>>>(wk, w, (uint16_t*)w_half);
  else if (dt == LARS_BF16) lars_publish_half_kernel<LARS_BF16><<<wk.grid, kThreads, 0, st>>>(wk, w, (uint16_t*)w_half);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

// ---------------------------------------------------------------- parallel deterministic initialization
// PAPER.md:119-127 (§III-B-1): every rank initializes the weights itself from the same seed — no broadcast.
// Each weight is a pure function of (seed, layer, element): Philox4x64-10 counter-based random numbers,
// truncated normal by inverse CDF (no rejection, so no data-dependent stream consumption).
__device__ __forceinline__ void philox4x64_10(uint64_t c[4], uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ull;
      k1 += 0xBB67AE8584CAA73Bull;
    }
    const uint64_t lo0 = 0xD2E7470EE14C6C93ull * c[0], hi0 = __umul64hi(0xD2E7470EE14C6C93ull, c[0]);
    const uint64_t lo1 = 0xCA5A826395121157ull * c[2], hi1 = __umul64hi(0xCA5A826395121157ull, c[2]);
    const uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
  }
}

__global__ void __launch_bounds__(kThreads) lars_init_weights_kernel(DevWork wk, InitTable it, float* __restrict__ w,
                                                                    uint64_t seed) {
  constexpr int kWarps = kThreads / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double phi_m2 = 0.022750131948179195;  // Phi(-2) = erfc(sqrt 2) / 2
  for (int32_t tile = blockIdx.x; tile < wk.ntiles; tile += gridDim.x) {
    const int32_t c0 = wk.tile_chunk[tile], c1 = wk.tile_chunk[tile + 1];
    for (int32_t c = c0 + warp; c < c1; c += kWarps) {
      const Seg ck = wk.chunks[c];
      const int32_t l = ck.tensor;
      const int32_t kind = it.kind[l];
      const int64_t i0 = ck.begin - it.offset[l];  // element index inside the layer (multiple of 4)
      for (int32_t q = 4 * lane; q < ck.len; q += 128) {
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (kind == LARS_KIND_WEIGHT) {
          uint64_t x[4] = {(uint64_t)(i0 + q) >> 2, (uint64_t)it.layer[l], 0ull, 0ull};
          philox4x64_10(x, seed, 0x4C415253ull);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const double u = (double)(x[k] >> 11) * 0x1.0p-53;
            const double p = phi_m2 + u * (1.0 - 2.0 * phi_m2);
            v[k] = (float)(it.sigma[l] * (1.4142135623730951 * erfinv(2.0 * p - 1.0)));
          }
        } else if (kind == LARS_KIND_BN_GAMMA) {
          v[0] = v[1] = v[2] = v[3] = 1.f;
        }
        for (int k = 0; k < 4 && q + k < ck.len; ++k) w[ck.begin + q + k] = v[k];
      }
    }
  }
}

cudaError_t launch_init_weights(const DevWork& wk, const InitTable& it, float* w, uint64_t seed, cudaStream_t st) {
  lars_init_weights_kernel<<<wk.grid, kThreads, 0, st>>>(wk, it, w, seed);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- launchers

template <int DT>
static cudaError_t launch_norms_t(const DevWork& wk, const DevScratch& sc, const Hyper& hy, const float* w,
                                  const void* g, int64_t g_shift, cudaStream_t st) {
  if (hy.k1_bulk) {
    if (hy.carry)
      return launch_pdl_smem(lars_norms_kernel<DT, true, true>, wk.grid, st, false, kBulkSmem, wk, sc, hy, w, g, g_shift);
    return launch_pdl_smem(lars_norms_kernel<DT, false, true>, wk.grid, st, false, kBulkSmem, wk, sc, hy, w, g, g_shift);
  }
  if (hy.carry) return launch_pdl(lars_norms_kernel<DT, true>, wk.grid, st, wk, sc, hy, w, g, g_shift);
  return launch_pdl(lars_norms_kernel<DT, false>, wk.grid, st, wk, sc, hy, w, g, g_shift);
}

// Resident K1 CTAs per SM with the bulk-copy stages (the work list assumes kCtasPerSm).
template <int DT, bool CARRY>
static int norms_bulk_occupancy() {
  int n = 0;
  prefer_shared(lars_norms_kernel<DT, CARRY, true>);
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, lars_norms_kernel<DT, CARRY, true>, kThreads, kBulkSmem) ==
                 cudaSuccess ? n : 0;
}
int norms_bulk_blocks_per_sm(int32_t dt, bool carry) {
  if (dt == LARS_F32) return carry ? norms_bulk_occupancy<LARS_F32, true>() : norms_bulk_occupancy<LARS_F32, false>();
  if (dt == LARS_F16) return carry ? norms_bulk_occupancy<LARS_F16, true>() : norms_bulk_occupancy<LARS_F16, false>();
  return carry ? norms_bulk_occupancy<LARS_BF16, true>() : norms_bulk_occupancy<LARS_BF16, false>();
}
template <int DT>
static cudaError_t launch_update_t(const DevWork& wk, const DevScratch& sc, const Hyper& hy, float* w,
                                   const void* g, int64_t g_shift, float* m, cudaStream_t st) {
  if constexpr (DT != LARS_F32) {
    if (hy.w_half) {
      if (hy.carry) return launch_pdl(lars_update_kernel<DT, true, true>, wk.grid, st, wk, sc, hy, w, g, g_shift, m);
      return launch_pdl(lars_update_kernel<DT, false, true>, wk.grid, st, wk, sc, hy, w, g, g_shift, m);
    }
  }
  if (hy.defer) {
    if (hy.carry) return launch_pdl(lars_update_kernel<DT, true, false, true>, wk.grid, st, wk, sc, hy, w, g, g_shift, m);
    return launch_pdl(lars_update_kernel<DT, false, false, true>, wk.grid, st, wk, sc, hy, w, g, g_shift, m);
  }
  if (hy.carry) return launch_pdl(lars_update_kernel<DT, true>, wk.grid, st, wk, sc, hy, w, g, g_shift, m);
  return launch_pdl(lars_update_kernel<DT, false>, wk.grid, st, wk, sc, hy, w, g, g_shift, m);
}

cudaError_t launch_norms(int32_t dt, const DevWork& wk, const DevScratch& sc, const Hyper& hy, const float* w,
                         const void* g, int64_t g_shift, cudaStream_t st) {
  if (wk.ntensors == 0) {  // nothing owned (P > number of layers): no norms, but keep the contract
    if (sc.c3) return cudaSuccess;  // data parallel: the finisher kernel decides (its shares stay 0)
    if (!hy.iter_dev) return cudaMemsetAsync(sc.skip, 0, sizeof(int32_t), st);
    empty_step_kernel<<<1, 1, 0, st>>>(hy.iter_dev, hy.total_iters, sc.skip);
    return cudaGetLastError();
  }
  switch (dt) {
    case LARS_F32: return launch_norms_t<LARS_F32>(wk, sc, hy, w, g, g_shift, st);
    case LARS_F16: return launch_norms_t<LARS_F16>(wk, sc, hy, w, g, g_shift, st);
    default: return launch_norms_t<LARS_BF16>(wk, sc, hy, w, g, g_shift, st);
  }
}

cudaError_t launch_update(int32_t dt, const DevWork& wk, const DevScratch& sc, const Hyper& hy, float* w,
                          const void* g, int64_t g_shift, float* m, cudaStream_t st) {
  if (wk.ntensors == 0) return cudaSuccess;
  switch (dt) {
    case LARS_F32: return launch_update_t<LARS_F32>(wk, sc, hy, w, g, g_shift, m, st);
    case LARS_F16: return launch_update_t<LARS_F16>(wk, sc, hy, w, g, g_shift, m, st);
    default: return launch_update_t<LARS_BF16>(wk, sc, hy, w, g, g_shift, m, st);
  }
}

cudaError_t launch_step(int32_t dt, const DevWork& wk, const DevScratch& sc, const Hyper& hy, float* w,
                        const void* g, int64_t g_shift, float* m, cudaStream_t st) {
  cudaError_t e = launch_norms(dt, wk, sc, hy, w, g, g_shift, st);
  if (e != cudaSuccess) return e;
  return launch_update(dt, wk, sc, hy, w, g, g_shift, m, st);
}

}  // namespace lars
