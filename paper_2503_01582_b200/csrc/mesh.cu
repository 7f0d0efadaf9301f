// mesh.cu -- isosurface extraction on the GPU, right after the density query
// (train_track's final refresh_grid + choose_iso +
// marching_cubes, mapper.cpp:186-187; marching_cubes.cpp:125-180).
//
// Output is the reference's Mesh exactly: the same vertex positions (bit
// for bit), the same triangles in the same order, vertices numbered in order
// of first use by the kept triangles (what cleanup_mesh leaves,
// mesh.cpp:30-54). The serial reference welds vertices through a hash map in
// cell order; here every step is a data-parallel pass over the lattice:
//
//   1. cells:  config + triangle count per cell; block totals          (k_mc_count)
//   2. scan of the block totals                                        (k_scan_blocks)
//   3. cells:  block-local scan -> every triangle's slot; its 3 welded
//              vertex keys (canonical lattice edge, as the reference's
//              edge_vertex key) and the zero-area test of cleanup_mesh (k_mc_emit)
//   4. keep-flag compaction of the triangles (generic scan)
//   5. first use of each edge key by a kept triangle (atomicMin)       (k_mc_first_use)
//   6. slot q is a vertex's first use iff first_use[key] == q; a scan of
//      those flags numbers the vertices; vertices and triangles are written (k_mc_write)
//
// Layout in HBM: the grid is R^3 fp32 x-fastest (refresh_grid layout);
// first_use is a dense u32 array over the 3 R^3 lattice edges (key =
// ((z R + y) R + x) 3 + axis, 200 MB at R = 256).
#include <algorithm>
#include <array>
#include <cstring>
#include <tuple>
#include <vector>

#include "prenom_device.cuh"

namespace prenom {
namespace {

// Cube conventions of the reference's table (marching_cubes.cpp:10-13): corner
// offsets and the 12 edges as corner pairs (vertex placement on crossed edges).
constexpr int kCorner[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                               {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
constexpr int kEdge[12][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}, {4, 5}, {5, 6},
                              {6, 7}, {7, 4}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};
constexpr int kMaxTri = 16;  // per configuration (the reference's table needs <= 12)

struct CaseTableDev {
  unsigned char count[256];
  unsigned char tri[256][kMaxTri][3];  // cube-edge indices
};
__constant__ CaseTableDev c_case;
__constant__ unsigned char c_edge_axis[12];     // 0/1/2
__constant__ unsigned char c_edge_lo[12][3];    // offset of the lower (canonical) endpoint

struct F3 {
  float x, y, z;
};

// The reference's case table (cube_case_triangles, marching_cubes.cpp:115-117),
// generated from its golden fixture by scripts/gen_mc_table.py.
#include "mc_case_table.inc"

const CaseTableDev& host_case_table() {
  static const CaseTableDev t = [] {
    CaseTableDev c;
    std::memset(&c, 0, sizeof c);
    for (int cfg = 0; cfg < 256; ++cfg) {
      c.count[cfg] = kMcCaseCount[cfg];
      for (int i = 0; i < kMcCaseCount[cfg]; ++i)
        for (int k = 0; k < 3; ++k) c.tri[cfg][i][k] = kMcCaseTri[cfg][i][k];
    }
    return c;
  }();
  return t;
}

// ------------------------------------------------------------------ device
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

struct McArgs {
  const float* grid;
  int R;
  float iso;
  long long ncells;  // (R-1)^3
};

__device__ __forceinline__ int cell_config(const McArgs& a, long long c, int& i, int& j, int& k) {
  const int C = a.R - 1;
  i = (int)(c % C);
  j = (int)((c / C) % C);
  k = (int)(c / ((long long)C * C));
  int cfg = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    // kCorner[q] = (x, y, z) = ((q ^ q >> 1) & 1, q >> 1 & 1, q >> 2)
    const int ox = (q ^ (q >> 1)) & 1, oy = (q >> 1) & 1, oz = q >> 2;
    const float v = a.grid[((size_t)(k + oz) * a.R + (j + oy)) * a.R + (i + ox)];
    if (v > a.iso) cfg |= 1 << q;  // "inside" = value > iso
  }
  return cfg;
}

__device__ __forceinline__ uint32_t cell_tris(const McArgs& a, long long c) {
  if (c >= a.ncells) return 0;
  int i, j, k;
  const int cfg = cell_config(a, c, i, j, k);
  return (cfg == 0 || cfg == 255) ? 0u : (uint32_t)c_case.count[cfg];
}

// Block-wide exclusive scan of ITEMS values per thread (warp shuffles + smem).
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* s_warp, uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    s_warp[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  total = s_warp[(blockDim.x >> 5) - 1];
  const uint32_t base = warp ? s_warp[warp - 1] : 0u;
  __syncthreads();
  return base + x - v;
}

__global__ void __launch_bounds__(kScanThreads) k_mc_count(McArgs a, uint32_t* block_sum) {
  __shared__ uint32_t s_warp[32];
  const long long c0 = (long long)blockIdx.x * kScanTile + (long long)threadIdx.x * kScanItems;
  uint32_t v = 0;
#pragma unroll
  for (int t = 0; t < kScanItems; ++t) v += cell_tris(a, c0 + t);
  uint32_t total;
  block_exclusive_scan(v, s_warp, total);
  if (threadIdx.x == 0) block_sum[blockIdx.x] = total;
}

// Exclusive scan of n block sums in place (one CTA, n <= kScanTile * chunks);
// writes the grand total to *total.
__global__ void __launch_bounds__(kScanThreads) k_scan_blocks(uint32_t* sums, int n, uint32_t* total) {
  __shared__ uint32_t s_warp[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < n; base += kScanTile) {
    uint32_t v[kScanItems], s = 0;
#pragma unroll
    for (int t = 0; t < kScanItems; ++t) {
      const int idx = base + threadIdx.x * kScanItems + t;
      v[t] = idx < n ? sums[idx] : 0u;
      s += v[t];
    }
    uint32_t tot;
    uint32_t ex = block_exclusive_scan(s, s_warp, tot) + carry;
#pragma unroll
    for (int t = 0; t < kScanItems; ++t) {
      const int idx = base + threadIdx.x * kScanItems + t;
      if (idx < n) sums[idx] = ex;
      ex += v[t];
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__device__ __forceinline__ F3 dev_vertex(const McArgs& a, uint32_t key, float scale) {
  const int axis = (int)(key % 3u);
  const uint32_t lin = key / 3u;
  const int ax = (int)(lin % (uint32_t)a.R), ay = (int)((lin / (uint32_t)a.R) % (uint32_t)a.R),
            az = (int)(lin / ((uint32_t)a.R * (uint32_t)a.R));
  const int bx = ax + (axis == 0), by = ay + (axis == 1), bz = az + (axis == 2);
  const float fa = a.grid[((size_t)az * a.R + ay) * a.R + ax];
  const float fb = a.grid[((size_t)bz * a.R + by) * a.R + bx];
  float t = __fdiv_rn(__fsub_rn(a.iso, fa), __fsub_rn(fb, fa));
  t = t < 0.f ? 0.f : (1.f < t ? 1.f : t);  // std::clamp
  const float pax = __fmul_rn((float)ax, scale), pay = __fmul_rn((float)ay, scale), paz = __fmul_rn((float)az, scale);
  const float pbx = __fmul_rn((float)bx, scale), pby = __fmul_rn((float)by, scale), pbz = __fmul_rn((float)bz, scale);
  return F3{__fadd_rn(pax, __fmul_rn(__fsub_rn(pbx, pax), t)), __fadd_rn(pay, __fmul_rn(__fsub_rn(pby, pay), t)),
            __fadd_rn(paz, __fmul_rn(__fsub_rn(pbz, paz), t))};
}

// cleanup_mesh's zero-area test (mesh.cpp:16-19, 35-38): area =
// 0.5 sqrt(double(dot(n, n))), n = cross(b - a, c - a), all in float.
__device__ __forceinline__ bool dev_nonzero_area(F3 p, F3 q, F3 r) {
  const float ux = __fsub_rn(q.x, p.x), uy = __fsub_rn(q.y, p.y), uz = __fsub_rn(q.z, p.z);
  const float vx = __fsub_rn(r.x, p.x), vy = __fsub_rn(r.y, p.y), vz = __fsub_rn(r.z, p.z);
  const float nx = __fsub_rn(__fmul_rn(uy, vz), __fmul_rn(uz, vy));
  const float ny = __fsub_rn(__fmul_rn(uz, vx), __fmul_rn(ux, vz));
  const float nz = __fsub_rn(__fmul_rn(ux, vy), __fmul_rn(uy, vx));
  const float d = __fadd_rn(__fadd_rn(__fmul_rn(nx, nx), __fmul_rn(ny, ny)), __fmul_rn(nz, nz));
  const double area = 0.5 * sqrt((double)d);
  return !(area <= 0.0);
}

__device__ __forceinline__ uint32_t edge_key(int R, int i, int j, int k, int e) {
  const int x = i + c_edge_lo[e][0], y = j + c_edge_lo[e][1], z = k + c_edge_lo[e][2];
  return (((uint32_t)z * (uint32_t)R + (uint32_t)y) * (uint32_t)R + (uint32_t)x) * 3u + c_edge_axis[e];
}

__global__ void __launch_bounds__(kScanThreads) k_mc_emit(McArgs a, const uint32_t* block_off, uint4* tris,
                                                          uint32_t* keep) {
  __shared__ uint32_t s_warp[32];
  const long long c0 = (long long)blockIdx.x * kScanTile + (long long)threadIdx.x * kScanItems;
  uint32_t cnt[kScanItems], v = 0;
#pragma unroll
  for (int t = 0; t < kScanItems; ++t) {
    cnt[t] = cell_tris(a, c0 + t);
    v += cnt[t];
  }
  uint32_t total;
  uint32_t slot = block_off[blockIdx.x] + block_exclusive_scan(v, s_warp, total);
  const float scale = 1.f / (float)(a.R - 1);
#pragma unroll
  for (int t = 0; t < kScanItems; ++t) {
    if (!cnt[t]) continue;
    int i, j, k;
    const int cfg = cell_config(a, c0 + t, i, j, k);
    for (uint32_t m = 0; m < cnt[t]; ++m, ++slot) {
      const uint32_t k0 = edge_key(a.R, i, j, k, c_case.tri[cfg][m][0]);
      const uint32_t k1 = edge_key(a.R, i, j, k, c_case.tri[cfg][m][1]);
      const uint32_t k2 = edge_key(a.R, i, j, k, c_case.tri[cfg][m][2]);
      tris[slot] = make_uint4(k0, k1, k2, 0u);
      keep[slot] = dev_nonzero_area(dev_vertex(a, k0, scale), dev_vertex(a, k1, scale), dev_vertex(a, k2, scale))
                       ? 1u : 0u;
    }
  }
}

// Generic exclusive scan, phase 1 / 3 (phase 2 = k_scan_blocks).
__global__ void __launch_bounds__(kScanThreads) k_scan_sum(const uint32_t* in, long long n, uint32_t* block_sum) {
  __shared__ uint32_t s_warp[32];
  const long long i0 = (long long)blockIdx.x * kScanTile + (long long)threadIdx.x * kScanItems;
  uint32_t v = 0;
#pragma unroll
  for (int t = 0; t < kScanItems; ++t) v += i0 + t < n ? in[i0 + t] : 0u;
  uint32_t total;
  block_exclusive_scan(v, s_warp, total);
  if (threadIdx.x == 0) block_sum[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_apply(const uint32_t* in, long long n,
                                                             const uint32_t* block_off, uint32_t* out) {
  __shared__ uint32_t s_warp[32];
  const long long i0 = (long long)blockIdx.x * kScanTile + (long long)threadIdx.x * kScanItems;
  uint32_t v[kScanItems], s = 0;
#pragma unroll
  for (int t = 0; t < kScanItems; ++t) {
    v[t] = i0 + t < n ? in[i0 + t] : 0u;
    s += v[t];
  }
  uint32_t total;
  uint32_t ex = block_off[blockIdx.x] + block_exclusive_scan(s, s_warp, total);
#pragma unroll
  for (int t = 0; t < kScanItems; ++t) {
    if (i0 + t < n) out[i0 + t] = ex;
    ex += v[t];
  }
}

// Compact the kept triangles (stable) and record each edge key's first use.
__global__ void k_mc_compact(const uint4* tris, const uint32_t* keep, const uint32_t* keep_off, long long ntri,
                             uint4* kept, uint32_t* first_use) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < ntri;
       t += (long long)gridDim.x * blockDim.x) {
    if (!keep[t]) continue;
    const uint32_t q = keep_off[t];
    const uint4 k = tris[t];
    kept[q] = k;
    atomicMin(first_use + k.x, 3u * q + 0u);
    atomicMin(first_use + k.y, 3u * q + 1u);
    atomicMin(first_use + k.z, 3u * q + 2u);
  }
}

__global__ void k_mc_mark(const uint4* kept, long long nslot, const uint32_t* first_use, uint32_t* mark) {
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < nslot;
       q += (long long)gridDim.x * blockDim.x) {
    const uint4 k = kept[q / 3];
    const uint32_t key = (q % 3 == 0) ? k.x : (q % 3 == 1 ? k.y : k.z);
    mark[q] = first_use[key] == (uint32_t)q ? 1u : 0u;
  }
}

__global__ void k_mc_write(McArgs a, const uint4* kept, long long nkept, const uint32_t* first_use,
                           const uint32_t* mark, const uint32_t* vid, float* verts, int* tris_out) {
  const float scale = 1.f / (float)(a.R - 1);
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < 3 * nkept;
       q += (long long)gridDim.x * blockDim.x) {
    const uint4 k = kept[q / 3];
    const uint32_t key = (q % 3 == 0) ? k.x : (q % 3 == 1 ? k.y : k.z);
    const uint32_t first = first_use[key];
    tris_out[q] = (int)vid[first];
    if (mark[q]) {
      const F3 p = dev_vertex(a, key, scale);
      const uint32_t v = vid[q];
      verts[3 * (size_t)v + 0] = p.x;
      verts[3 * (size_t)v + 1] = p.y;
      verts[3 * (size_t)v + 2] = p.z;
    }
  }
}

__global__ void k_grid_max(const float* g, long long n, float* out) {
  float m = -INFINITY;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    m = fmaxf(m, g[i]);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<int*>(out), __float_as_int(m));  // m >= 0 on grids
}

bool g_tables_uploaded[64] = {};

cudaError_t upload_tables(cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && g_tables_uploaded[dev]) return cudaSuccess;
  unsigned char axis[12], lo[12][3];
  for (int e = 0; e < 12; ++e) {
    const int* ca = kCorner[kEdge[e][0]];
    const int* cb = kCorner[kEdge[e][1]];
    // canonical endpoint: the lexicographically smaller of (x, y, z) (marching_cubes.cpp:137-141)
    const bool b_first = std::make_tuple(cb[0], cb[1], cb[2]) < std::make_tuple(ca[0], ca[1], ca[2]);
    const int* l = b_first ? cb : ca;
    const int* h = b_first ? ca : cb;
    axis[e] = (unsigned char)(h[0] != l[0] ? 0 : (h[1] != l[1] ? 1 : 2));
    for (int d = 0; d < 3; ++d) lo[e][d] = (unsigned char)l[d];
  }
  cudaError_t e = cudaMemcpyToSymbolAsync(c_case, &host_case_table(), sizeof(CaseTableDev), 0,
                                          cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyToSymbolAsync(c_edge_axis, axis, sizeof axis, 0, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyToSymbolAsync(c_edge_lo, lo, sizeof lo, 0, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // the host table must outlive the copy
  if (e == cudaSuccess && dev < 64) g_tables_uploaded[dev] = true;
  return e;
}

}  // namespace

// exclusive scan of n u32 -> out; returns the total through a host read
cudaError_t scan_exclusive_u32(const uint32_t* in, long long n, uint32_t* out, MeshBuf<uint32_t>& tmp, uint32_t* d_total,
                     uint32_t* h_total, cudaStream_t st) {
  const long long nb = (n + kScanTile - 1) / kScanTile;
  cudaError_t e = tmp.ensure((size_t)std::max<long long>(nb, 1));
  if (e != cudaSuccess) return e;
  if (n > 0) {
    k_scan_sum<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, tmp.p);
    k_scan_blocks<<<1, kScanThreads, 0, st>>>(tmp.p, (int)nb, d_total);
    k_scan_apply<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, tmp.p, out);
  } else {
    e = cudaMemsetAsync(d_total, 0, sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
  }
  e = cudaMemcpyAsync(h_total, d_total, sizeof(uint32_t), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return e == cudaSuccess ? cudaGetLastError() : e;
}


int mc_case_triangles(int config, int* edges) {
  if (config < 0 || config > 255) return -1;
  const CaseTableDev& t = host_case_table();
  for (int i = 0; i < t.count[config]; ++i)
    for (int k = 0; k < 3; ++k) edges[3 * i + k] = t.tri[config][i][k];
  return t.count[config];
}

cudaError_t launch_grid_max(const float* grid, long long n, float* d_out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(d_out, 0, sizeof(float), st);
  if (e != cudaSuccess) return e;
  k_grid_max<<<(unsigned)std::min<long long>((n + 255) / 256, 148 * 8), 256, 0, st>>>(grid, n, d_out);
  return cudaGetLastError();
}

// Marching cubes of an R^3 device grid (scratch `m`) into the mesh `out`.
cudaError_t run_marching_cubes(const float* d_grid, int R, float iso, McScratch& m, McMesh& out, cudaStream_t st,
                               int* launches) {
  out.n_vertices = out.n_triangles = 0;
  if (R < 2) return cudaSuccess;
  cudaError_t e = upload_tables(st);
  if (e != cudaSuccess) return e;
  auto& block = m.block;
  auto& tmp = m.tmp;
  auto& keep = m.keep;
  auto& keep_off = m.keep_off;
  auto& first_use = m.first_use;
  auto& mark = m.mark;
  auto& vid = m.vid;
  auto& total = m.total;
  auto& tris = m.tri_keys;
  auto& kept = m.kept;
  McArgs a{d_grid, R, iso, (long long)(R - 1) * (R - 1) * (R - 1)};
  const long long nb = (a.ncells + kScanTile - 1) / kScanTile;
  if ((e = block.ensure((size_t)nb)) != cudaSuccess || (e = total.ensure(1)) != cudaSuccess) return e;
  uint32_t ntri = 0, nkept = 0, nvert = 0;
  k_mc_count<<<(unsigned)nb, kScanThreads, 0, st>>>(a, block.p);
  k_scan_blocks<<<1, kScanThreads, 0, st>>>(block.p, (int)nb, total.p);
  if ((e = cudaMemcpyAsync(&ntri, total.p, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  *launches += 2;
  if (ntri == 0) return cudaGetLastError();
  if ((e = tris.ensure(ntri)) != cudaSuccess || (e = keep.ensure(ntri)) != cudaSuccess ||
      (e = keep_off.ensure(ntri)) != cudaSuccess)
    return e;
  k_mc_emit<<<(unsigned)nb, kScanThreads, 0, st>>>(a, block.p, tris.p, keep.p);
  if ((e = scan_exclusive_u32(keep.p, ntri, keep_off.p, tmp, total.p, &nkept, st)) != cudaSuccess) return e;
  *launches += 4;
  if (nkept == 0) return cudaSuccess;
  const size_t nkeys = (size_t)3 * R * R * R;
  if ((e = kept.ensure(nkept)) != cudaSuccess || (e = first_use.ensure(nkeys)) != cudaSuccess ||
      (e = mark.ensure(3 * (size_t)nkept)) != cudaSuccess || (e = vid.ensure(3 * (size_t)nkept)) != cudaSuccess)
    return e;
  if ((e = cudaMemsetAsync(first_use.p, 0xFF, nkeys * sizeof(uint32_t), st)) != cudaSuccess) return e;
  const unsigned g = (unsigned)std::min<long long>((ntri + 255) / 256, 148 * 16);
  k_mc_compact<<<g, 256, 0, st>>>(tris.p, keep.p, keep_off.p, ntri, kept.p, first_use.p);
  const long long nslot = 3LL * nkept;
  const unsigned gs = (unsigned)std::min<long long>((nslot + 255) / 256, 148 * 16);
  k_mc_mark<<<gs, 256, 0, st>>>(kept.p, nslot, first_use.p, mark.p);
  if ((e = scan_exclusive_u32(mark.p, nslot, vid.p, tmp, total.p, &nvert, st)) != cudaSuccess) return e;
  if ((e = out.verts.ensure(3 * (size_t)nvert)) != cudaSuccess || (e = out.tris.ensure(nslot)) != cudaSuccess) return e;
  k_mc_write<<<gs, 256, 0, st>>>(a, kept.p, nkept, first_use.p, mark.p, vid.p, out.verts.p, out.tris.p);
  *launches += 6;
  out.n_vertices = nvert;
  out.n_triangles = nkept;
  return cudaGetLastError();
}

}  // namespace prenom
