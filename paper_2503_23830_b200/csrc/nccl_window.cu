// The peer addresses of an NCCL symmetric-memory window (NCCL 2.28 device API:
// ncclCommWindowRegister with NCCL_WIN_COLL_SYMMETRIC, ncclGetPeerPointer), so
// the fused put can store into windows NCCL allocated and mapped
// (orch_window_create_nccl in dispatch.cu). Its own translation unit: the
// device API headers and dispatch.cu's anonymous-namespace kernels do not mix.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

namespace orchb {

__global__ void k_nccl_window_peers(ncclWindow_t win, int P, char** __restrict__ peers) {
  const int r = threadIdx.x;
  if (r < P) peers[r] = static_cast<char*>(ncclGetPeerPointer(win, 0, r));
}

cudaError_t nccl_window_peers(ncclWindow_t win, int P, char** peers_dev) {
  k_nccl_window_peers<<<1, 32>>>(win, P, peers_dev);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  return e;
}

}  // namespace orchb
