// kernels_metrics.cu -- nearest-neighbour search for the Chamfer distance of
// the genome evaluation (metrics.cpp:14-22, search.cpp:256-262).
//
// The reference builds a kd-tree per cloud; its pruning (diff^2 < best) is
// exact in float, so every query's result is the exact minimum of
// squared_norm(p - q) over the cloud. Here that minimum is taken by brute
// force: a query per thread, the point cloud streamed through shared memory
// in tiles, the squared distance spelled as the reference computes it
// (geom.hpp:28-33: ((dx*dx + dy*dy) + dz*dz), separate roundings, no FMA).
// |a|·|b| = 2048^2 distances per evaluation mesh pair: microseconds.
#include "prenom_device.cuh"

namespace prenom {
namespace {

constexpr int kNnThreads = 256;
constexpr int kNnTile = 1024;

__global__ void __launch_bounds__(kNnThreads) k_nearest_sq(int nq, const float* __restrict__ q, int np,
                                                           const float* __restrict__ p, float* __restrict__ out) {
  __shared__ float tile[kNnTile * 3];
  const int i = blockIdx.x * kNnThreads + threadIdx.x;
  float qx = 0.f, qy = 0.f, qz = 0.f;
  if (i < nq) {
    qx = q[3 * i];
    qy = q[3 * i + 1];
    qz = q[3 * i + 2];
  }
  float best = INFINITY;
  for (int t0 = 0; t0 < np; t0 += kNnTile) {
    const int nt = min(kNnTile, np - t0);
    __syncthreads();
    for (int j = threadIdx.x; j < nt * 3; j += kNnThreads) tile[j] = p[3 * (size_t)t0 + j];
    __syncthreads();
    if (i < nq)
      for (int j = 0; j < nt; ++j) {
        const float dx = __fsub_rn(tile[3 * j], qx), dy = __fsub_rn(tile[3 * j + 1], qy),
                    dz = __fsub_rn(tile[3 * j + 2], qz);
        const float d = __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
        best = d < best ? d : best;
      }
  }
  if (i < nq) out[i] = best;
}

}  // namespace

cudaError_t launch_nearest_sq(int nq, const float* q, int np, const float* p, float* out, cudaStream_t st) {
  if (nq <= 0) return cudaSuccess;
  k_nearest_sq<<<(nq + kNnThreads - 1) / kNnThreads, kNnThreads, 0, st>>>(nq, q, np, p, out);
  return cudaGetLastError();
}

}  // namespace prenom
