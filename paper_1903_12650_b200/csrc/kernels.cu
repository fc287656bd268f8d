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

#include <cstdint>

#include "internal.h"

namespace lars {

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
__device__ __forceinline__ uint4 ld16_nc(const void* p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// Gradient access by wire dtype. Widening fp16/bf16 -> fp32 is exact.
template <int DT> struct Grad;
template <> struct Grad<LARS_F32> {
  __device__ __forceinline__ static F8 load8_keep(const void* g, int64_t i) { return ld8_keep((const float*)g + i); }
  __device__ __forceinline__ static F8 load8(const void* g, int64_t i) { return ld8_nc((const float*)g + i); }
  __device__ __forceinline__ static float load1(const void* g, int64_t i) { return __ldg((const float*)g + i); }
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
  __device__ __forceinline__ static F8 load8_keep(const void* g, int64_t i) { return widen_h8(ld16_nc((const __half*)g + i)); }
  __device__ __forceinline__ static F8 load8(const void* g, int64_t i) { return widen_h8(ld16_nc((const __half*)g + i)); }
  __device__ __forceinline__ static float load1(const void* g, int64_t i) { return __half2float(((const __half*)g)[i]); }
};
template <> struct Grad<LARS_BF16> {
  __device__ __forceinline__ static F8 load8_keep(const void* g, int64_t i) { return widen_b8(ld16_nc((const uint16_t*)g + i)); }
  __device__ __forceinline__ static F8 load8(const void* g, int64_t i) { return widen_b8(ld16_nc((const uint16_t*)g + i)); }
  __device__ __forceinline__ static float load1(const void* g, int64_t i) {
    return __uint_as_float((uint32_t)((const uint16_t*)g)[i] << 16);
  }
};

__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void acc8(double& a, const F8& x) {
#pragma unroll
  for (int i = 0; i < 8; ++i) a = fma((double)x.v[i], (double)x.v[i], a);
}

// ---------------------------------------------------------------- K1: segmented norms + finish
__device__ void finish_tensor(int32_t l, const DevWork& wk, const DevScratch& sc, const Hyper& hy) {
  // Runs on ONE thread once all segments of local tensor l have published their partials.
  __threadfence();
  const int32_t b = wk.tseg_begin[l], c = wk.tseg_count[l];
  double sw = 0.0, sg = 0.0;
  for (int32_t i = 0; i < c; ++i) {  // fixed order -> bit-reproducible
    sw += __ldcg(sc.part_w + b + i);
    sg += __ldcg(sc.part_g + b + i);
  }
  sc.seg_done[l] = 0u;  // all of this step's arrivals are in: rearm for the next step
  const double wn = sqrt(sw);
  const double gn = fabs(hy.grad_scale) * sqrt(sg);
  double lam = 1.0, beta = 0.0;
  if (wk.tlars[l]) {
    beta = hy.weight_decay;
    const double den = gn + hy.weight_decay * wn + hy.eps;
    if (wn > 0.0 && den > 0.0) lam = hy.eta * wn / den;
  }
  sc.w_norm[l] = wn;
  sc.g_norm[l] = gn;
  sc.lambda[l] = lam;
  sc.coef[l] = (float)(hy.lr_table[hy.iter] * lam);
  sc.beta[l] = (float)beta;
  if (!(isfinite(wn) && isfinite(gn))) atomicOr(sc.nonfinite, 1u);
  __threadfence();
  if (atomicAdd(sc.tensors_done, 1u) == (unsigned)wk.ntensors - 1u) {
    __threadfence();
    const unsigned nf = atomicExch(sc.nonfinite, 0u);
    *(volatile int32_t*)sc.skip = nf ? 1 : 0;
    *(volatile unsigned*)sc.tensors_done = 0u;
  }
}

template <int DT>
__global__ void __launch_bounds__(kThreads) lars_norms_kernel(DevWork wk, DevScratch sc, Hyper hy,
                                                              const float* __restrict__ w,
                                                              const void* __restrict__ g, int64_t g_shift) {
  __shared__ double red_w[kThreads / 32], red_g[kThreads / 32];
  pdl_trigger();
  pdl_wait();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int32_t s0 = wk.tile_seg[blockIdx.x], s1 = wk.tile_seg[blockIdx.x + 1];
  for (int32_t s = s0; s < s1; ++s) {
    const Seg sg = wk.segs[s];
    const float* wp = w + sg.begin;
    const int64_t gi = sg.begin - g_shift;
    const int32_t ng = sg.len >> 3;
    double aw = 0.0, ag = 0.0, aw1 = 0.0, ag1 = 0.0;
    int32_t j = tid;
    for (; j + 3 * kThreads < ng; j += 4 * kThreads) {
      F8 w0 = ld8_keep(wp + 8 * j), w1 = ld8_keep(wp + 8 * (j + kThreads));
      F8 w2 = ld8_keep(wp + 8 * (j + 2 * kThreads)), w3 = ld8_keep(wp + 8 * (j + 3 * kThreads));
      F8 g0 = Grad<DT>::load8_keep(g, gi + 8 * j), g1 = Grad<DT>::load8_keep(g, gi + 8 * (j + kThreads));
      F8 g2 = Grad<DT>::load8_keep(g, gi + 8 * (j + 2 * kThreads));
      F8 g3 = Grad<DT>::load8_keep(g, gi + 8 * (j + 3 * kThreads));
      acc8(aw, w0); acc8(aw1, w1); acc8(aw, w2); acc8(aw1, w3);
      acc8(ag, g0); acc8(ag1, g1); acc8(ag, g2); acc8(ag1, g3);
    }
    aw += aw1;
    ag += ag1;
    for (; j < ng; j += kThreads) {
      F8 w0 = ld8_keep(wp + 8 * j);
      F8 g0 = Grad<DT>::load8_keep(g, gi + 8 * j);
      acc8(aw, w0);
      acc8(ag, g0);
    }
    for (int32_t i = (ng << 3) + tid; i < sg.len; i += kThreads) {  // ragged tensor tail
      const double x = (double)wp[i], y = (double)Grad<DT>::load1(g, gi + i);
      aw = fma(x, x, aw);
      ag = fma(y, y, ag);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      aw += __shfl_xor_sync(0xffffffffu, aw, o);
      ag += __shfl_xor_sync(0xffffffffu, ag, o);
    }
    if (lane == 0) { red_w[warp] = aw; red_g[warp] = ag; }
    __syncthreads();
    if (tid == 0) {
      double tw = 0.0, tg = 0.0;
#pragma unroll
      for (int i = 0; i < kThreads / 32; ++i) { tw += red_w[i]; tg += red_g[i]; }
      sc.part_w[s] = tw;
      sc.part_g[s] = tg;
      __threadfence();
      const unsigned prev = atomicAdd(sc.seg_done + sg.tensor, 1u);
      if (prev == (unsigned)wk.tseg_count[sg.tensor] - 1u) finish_tensor(sg.tensor, wk, sc, hy);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- K2: fused update
__device__ __forceinline__ void upd8(F8& w, F8& m, const F8& g, float s, float c, float b, float mu) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float u = fmaf(b, w.v[i], s * g.v[i]);  // s*g + beta_l*w
    const float v = fmaf(mu, m.v[i], c * u);       // mu*v + lr*lambda*(...)
    w.v[i] = w.v[i] - v;
    m.v[i] = v;
  }
}

template <int DT>
__global__ void __launch_bounds__(kThreads) lars_update_kernel(DevWork wk, DevScratch sc, Hyper hy,
                                                               float* __restrict__ w,
                                                               const void* __restrict__ g, int64_t g_shift,
                                                               float* __restrict__ m) {
  pdl_trigger();
  pdl_wait();
  if (*(volatile const int32_t*)sc.skip) return;  // whole step skipped (non-finite norm)
  const int tid = threadIdx.x;
  const float s = hy.grad_scale_f, mu = hy.mu;
  const int32_t s0 = wk.tile_seg[blockIdx.x], s1 = wk.tile_seg[blockIdx.x + 1];
  for (int32_t s_ = s1 - 1; s_ >= s0; --s_) {  // backwards: K1's most recent reads first
    const Seg sg = wk.segs[s_];
    const float c = sc.coef[sg.tensor], b = sc.beta[sg.tensor];
    float* wp = w + sg.begin;
    float* mp = m + sg.begin;
    const int64_t gi = sg.begin - g_shift;
    const int32_t ng = sg.len >> 3;
    for (int32_t i = (ng << 3) + tid; i < sg.len; i += kThreads) {  // ragged tail
      float wv = wp[i], mv = mp[i];
      const float u = fmaf(b, wv, s * Grad<DT>::load1(g, gi + i));
      const float v = fmaf(mu, mv, c * u);
      wp[i] = wv - v;
      mp[i] = v;
    }
    int32_t j = ng - 1 - tid;
    for (; j - kThreads >= 0; j -= 2 * kThreads) {
      const int32_t j1 = j - kThreads;
      F8 w0 = ld8_rw(wp + 8 * j), w1 = ld8_rw(wp + 8 * j1);
      F8 g0 = Grad<DT>::load8(g, gi + 8 * j), g1 = Grad<DT>::load8(g, gi + 8 * j1);
      F8 m0 = ld8_rw(mp + 8 * j), m1 = ld8_rw(mp + 8 * j1);
      upd8(w0, m0, g0, s, c, b, mu);
      upd8(w1, m1, g1, s, c, b, mu);
      st8(wp + 8 * j, w0); st8(mp + 8 * j, m0);
      st8(wp + 8 * j1, w1); st8(mp + 8 * j1, m1);
    }
    if (j >= 0) {
      F8 w0 = ld8_rw(wp + 8 * j), g0 = Grad<DT>::load8(g, gi + 8 * j), m0 = ld8_rw(mp + 8 * j);
      upd8(w0, m0, g0, s, c, b, mu);
      st8(wp + 8 * j, w0);
      st8(mp + 8 * j, m0);
    }
  }
}

// ---------------------------------------------------------------- launchers
template <typename K, typename... Args>
static cudaError_t launch_pdl(K kernel, int grid, cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <int DT>
static cudaError_t launch_norms_t(const DevWork& wk, const DevScratch& sc, const Hyper& hy, const float* w,
                                  const void* g, int64_t g_shift, cudaStream_t st) {
  return launch_pdl(lars_norms_kernel<DT>, wk.ntiles, st, wk, sc, hy, w, g, g_shift);
}
template <int DT>
static cudaError_t launch_update_t(const DevWork& wk, const DevScratch& sc, const Hyper& hy, float* w,
                                   const void* g, int64_t g_shift, float* m, cudaStream_t st) {
  return launch_pdl(lars_update_kernel<DT>, wk.ntiles, st, wk, sc, hy, w, g, g_shift, m);
}

cudaError_t launch_norms(int32_t dt, const DevWork& wk, const DevScratch& sc, const Hyper& hy, const float* w,
                         const void* g, int64_t g_shift, cudaStream_t st) {
  if (wk.ntensors == 0) return cudaMemsetAsync(sc.skip, 0, sizeof(int32_t), st);
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
