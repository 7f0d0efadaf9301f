// kernels_umma_test.cu -- single-tile tcgen05 GEMM used by
// prenom_debug_umma_gemm to validate the descriptor / TMEM layout toolkit
// (umma.cuh) on the device: D[M][N] = A[M][K] * B[N][K]^T in bf16 -> fp32,
// with A and B staged K-major or MN-major.
#include "prenom_device.cuh"
#include "umma.cuh"

namespace prenom {
namespace {

__global__ void __launch_bounds__(128) k_umma_gemm(int M, int N, int K, int a_mn, int b_mn, const float* A,
                                                   const float* B, float* D) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* sa = sm;
  unsigned char* sb = sm + (size_t)M * K * 2;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // stage operands as bf16 core-matrix tiles
  for (int i = tid; i < M * K; i += 128) {
    const int m = i / K, k = i % K;
    const __nv_bfloat16 v = __float2bfloat16_rn(A[i]);
    const uint32_t off = a_mn ? umma::cm_offset(k, m, M) : umma::cm_offset(m, k, K);
    *reinterpret_cast<__nv_bfloat16*>(sa + off) = v;
  }
  for (int i = tid; i < N * K; i += 128) {
    const int n = i / K, k = i % K;
    const __nv_bfloat16 v = __float2bfloat16_rn(B[i]);
    const uint32_t off = b_mn ? umma::cm_offset(k, n, N) : umma::cm_offset(n, k, K);
    *reinterpret_cast<__nv_bfloat16*>(sb + off) = v;
  }
  uint32_t ncols = 32;
  while ((int)ncols < N) ncols <<= 1;
  if (warp == 0) umma::tmem_alloc(&tbase, ncols);
  if (tid == 0) {
    umma::mbar_init(&bar, 1);
    umma::fence_mbar_init();
  }
  umma::fence_proxy_async();
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tm = tbase;
  if (tid == 0) {
    const uint32_t idesc = umma::idesc_bf16(M, N, a_mn, b_mn);
    for (int ks = 0; ks < K / 16; ++ks) {
      const uint64_t da = a_mn ? umma::desc_mnmajor(sa, M, ks) : umma::desc_kmajor(sa, K, ks);
      const uint64_t db = b_mn ? umma::desc_mnmajor(sb, N, ks) : umma::desc_kmajor(sb, K, ks);
      umma::mma_bf16(tm, da, db, idesc, ks > 0);
    }
    umma::commit(&bar);
  }
  umma::mbar_wait(&bar, 0);
  umma::fence_after_sync();
  // M = 128: row = lane of the warp's quadrant. M = 64: rows 16q..16q+15 in lanes 32q..32q+15.
  const int row = M == 128 ? 32 * warp + lane : (lane < 16 ? 16 * warp + lane : -1);
  for (int c = 0; c < N; c += 8) {
    float v[8];
    umma::tmem_ld8(umma::taddr(tm, 32 * warp, c), v);
    umma::tmem_wait_ld();
    if (row >= 0)
      for (int j = 0; j < 8; ++j) D[(size_t)row * N + c + j] = v[j];
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tm, ncols);
}

}  // namespace

cudaError_t launch_umma_gemm(int M, int N, int K, int a_mn, int b_mn, const float* A, const float* B, float* D,
                             cudaStream_t st) {
  const size_t smem = (size_t)(M + N) * K * 2;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_umma_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_umma_gemm<<<1, 128, smem, st>>>(M, N, K, a_mn, b_mn, A, B, D);
  return cudaGetLastError();
}

}  // namespace prenom
