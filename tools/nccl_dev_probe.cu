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
  CK(ncclDevCommDestroy(comm, &dc));
  CK(ncclCommWindowDeregister(comm, win));
  CK(ncclMemFree(buf));
  CK(ncclCommDestroy(comm));
  return h == 0 ? 0 : 1;
}
