// Probe of the NCCL 2.28 device API on this box (not product code): symmetric window + LSA peer
// pointers + per-CTA LSA barrier, P processes forked from one launcher, one GPU each.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I<nccl>/include tools/nccl_dev_probe.cu \
//        -L<nccl>/lib -l:libnccl.so.2 -o build/nccl_dev_probe && build/nccl_dev_probe 2
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>
#include <sys/wait.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#define CK(x) do { auto e_ = (x); if (e_ != 0) { printf("rank %d: %s failed (%d) at %d\n", rank, #x, (int)e_, __LINE__); exit(1); } } while (0)

__global__ void probe(ncclDevComm dc, ncclWindow_t win, int rank, int P, int* out) {
  // every CTA b writes (rank, b) into slot [b][rank] of every peer, then syncs with CTA b of all peers
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    int* dst = (int*)ncclGetLsaPointer(win, ((size_t)blockIdx.x * P + rank) * sizeof(int), p);
    *dst = rank * 100000 + blockIdx.x;
  }
  ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), blockIdx.x);
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  int* local = (int*)ncclGetLocalPointer(win, 0);
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    const int v = local[blockIdx.x * P + p];
    if (v != p * 100000 + (int)blockIdx.x) atomicAdd(out, 1);
  }
}

// RS-like pattern: rank r reads slice r (n floats) from every other rank; AG-like: rank r writes slice r
// into every other rank. 128-bit or 256-bit vectors, unrolled.
template <int U>
__global__ void peer_read(ncclWindow_t win, int rank, int P, size_t n, float* sink) {
  float acc = 0.f;
  const size_t nv = n / 8;
  for (int p = 0; p < P; ++p) {
    if (p == rank) continue;
    const float* src = (const float*)ncclGetLsaPointer(win, (size_t)rank * n * 4, p);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nv; i += (size_t)gridDim.x * blockDim.x * U) {
      uint32_t r[U][8];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        size_t k = i + (size_t)u * gridDim.x * blockDim.x;
        if (k < nv)
          asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(r[u][0]), "=r"(r[u][1]), "=r"(r[u][2]),
                       "=r"(r[u][3]), "=r"(r[u][4]), "=r"(r[u][5]), "=r"(r[u][6]), "=r"(r[u][7]) : "l"(src + 8 * k));
        else
          for (int q = 0; q < 8; ++q) r[u][q] = 0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        for (int q = 0; q < 8; ++q) acc += __uint_as_float(r[u][q]);
    }
  }
  if (acc == 12345.f) *sink = acc;
}

// 128-bit non-coherent loads (what the fused F1 uses for fp16 gradients), all peers per element
template <int U>
__global__ void peer_read_v4nc(ncclWindow_t win, int rank, int P, size_t n, float* sink) {
  float acc = 0.f;
  const size_t nv = n / 4;
  const float* src[8];
  for (int p = 0; p < P; ++p) src[p] = (const float*)ncclGetLsaPointer(win, (size_t)rank * n * 4, p);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nv; i += (size_t)gridDim.x * blockDim.x * U) {
    uint32_t r[U][8][4];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int p = 0; p < 8; ++p)
        if (p < P && p != rank) {
          size_t k = i + (size_t)u * gridDim.x * blockDim.x;
          if (k >= nv) k = i;
          asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r[u][p][0]), "=r"(r[u][p][1]),
                       "=r"(r[u][p][2]), "=r"(r[u][p][3]) : "l"(src[p] + 4 * k));
        }
#pragma unroll
    for (int u = 0; u < U; ++u)
      for (int p = 0; p < 8; ++p)
        if (p < P && p != rank)
          for (int q = 0; q < 4; ++q) acc += __uint_as_float(r[u][p][q]);
  }
  if (acc == 12345.f) *sink = acc;
}

__global__ void peer_write(ncclWindow_t win, int rank, int P, size_t n) {
  const size_t nv = n / 8;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nv; i += (size_t)gridDim.x * blockDim.x) {
    for (int p = 0; p < P; ++p) {
      if (p == rank) continue;
      float* dst = (float*)ncclGetLsaPointer(win, (size_t)rank * n * 4, p) + 8 * i;
      asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst), "r"(1), "r"(2), "r"(3), "r"(4), "r"(5),
                   "r"(6), "r"(7), "r"(8) : "memory");
    }
  }
}

int main(int argc, char** argv) {
  int P = argc > 1 ? atoi(argv[1]) : 2;
  int rank = -1;
  ncclUniqueId id;
  CK(ncclGetUniqueId(&id));
  for (int r = 0; r < P; ++r) {
    if (fork() == 0) { rank = r; break; }
  }
  if (rank < 0) {
    int bad = 0, st = 0;
    for (int r = 0; r < P; ++r) { wait(&st); bad |= !(WIFEXITED(st) && WEXITSTATUS(st) == 0); }
    printf("probe P=%d: %s\n", P, bad ? "FAILED" : "ok");
    return bad;
  }
  CK(cudaSetDevice(rank));
  ncclComm_t comm;
  CK(ncclCommInitRank(&comm, P, id, rank));
  const int blocks = 148 * 4;
  void* buf = nullptr;
  size_t bytes = 1 << 22;
  CK(ncclMemAlloc(&buf, bytes));
  CK(cudaMemset(buf, 0, bytes));
  ncclWindow_t win;
  CK(ncclCommWindowRegister(comm, buf, bytes, &win, NCCL_WIN_COLL_SYMMETRIC));
  ncclDevCommRequirements reqs;
  memset(&reqs, 0, sizeof reqs);
  reqs.lsaBarrierCount = blocks;
  ncclDevComm dc;
  CK(ncclDevCommCreate(comm, &reqs, &dc));
  printf("rank %d: lsaRank %d lsaSize %d nRanks %d\n", rank, dc.lsaRank, dc.lsaSize, dc.nRanks);
  int* out;
  CK(cudaMalloc(&out, 4));
  CK(cudaMemset(out, 0, 4));
  for (int it = 0; it < 3; ++it) probe<<<blocks, 128>>>(dc, win, rank, P, out);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  int h = -1;
  CK(cudaMemcpy(&h, out, 4, cudaMemcpyDeviceToHost));
  // timing of an empty barrier round
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int it = 0; it < 100; ++it) probe<<<blocks, 128>>>(dc, win, rank, P, out);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("rank %d: mismatches %d, write+barrier kernel %.2f us\n", rank, h, ms * 10.0f);
  {  // bandwidth: 64 MB slice per rank
    const size_t n = (size_t)16 << 20;  // floats per slice
    void* big = nullptr;
    const size_t bb = n * 4 * P;
    CK(ncclMemAlloc(&big, bb));
    CK(cudaMemset(big, 0, bb));
    ncclWindow_t bw;
    CK(ncclCommWindowRegister(comm, big, bb, &bw, NCCL_WIN_COLL_SYMMETRIC));
    float* sink;
    CK(cudaMalloc(&sink, 4));
    for (int cfg = 0; cfg < 4; ++cfg) {
      const int grid = (cfg & 1) ? 148 * 8 : 148 * 4, thr = 256;
      for (int warm = 0; warm < 2; ++warm) {
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int it = 0; it < 10; ++it) {
          if (cfg < 2) peer_read<2><<<grid, thr>>>(bw, rank, P, n, sink);
          else peer_read<4><<<grid, thr>>>(bw, rank, P, n, sink);
        }
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
      }
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = (double)n * 4 * (P - 1);
      printf("rank %d: peer read (ingress) cfg %d: %.1f GB/s\n", rank, cfg, bytes / (ms / 10 * 1e-3) / 1e9);
    }
    for (int cfg = 0; cfg < 3; ++cfg) {
      const int grid = 148 * 4;
      for (int warm = 0; warm < 2; ++warm) {
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int it = 0; it < 10; ++it) {
          if (cfg == 0) peer_read_v4nc<1><<<grid, 256>>>(bw, rank, P, n, sink);
          else if (cfg == 1) peer_read_v4nc<2><<<grid, 256>>>(bw, rank, P, n, sink);
          else peer_read_v4nc<4><<<grid, 256>>>(bw, rank, P, n, sink);
        }
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
      }
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = (double)n * 4 * (P - 1);
      printf("rank %d: peer read v4.nc all-peers U=%d: %.1f GB/s\n", rank, 1 << cfg, bytes / (ms / 10 * 1e-3) / 1e9);
    }
    for (int cfg = 0; cfg < 2; ++cfg) {
      const int grid = cfg ? 148 * 8 : 148 * 4;
      for (int warm = 0; warm < 2; ++warm) {
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int it = 0; it < 10; ++it) peer_write<<<grid, 256>>>(bw, rank, P, n);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
      }
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = (double)n * 4 * (P - 1);
      printf("rank %d: peer write (egress) cfg %d: %.1f GB/s\n", rank, cfg, bytes / (ms / 10 * 1e-3) / 1e9);
    }
  }
  CK(ncclDevCommDestroy(comm, &dc));
  CK(ncclCommWindowDeregister(comm, win));
  CK(ncclMemFree(buf));
  CK(ncclCommDestroy(comm));
  return h == 0 ? 0 : 1;
}
