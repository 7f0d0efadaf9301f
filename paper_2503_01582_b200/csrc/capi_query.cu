// capi_query.cu -- C ABI: render, density query, mesh extraction, batched field_eval, metric NN.
#include "capi_internal.cuh"

using namespace prenom;
using namespace prenom_capi;

extern "C" {
prenom_status prenom_render(prenom_object_t o, int n_rays, const float* origins, const float* dirs,
                            float* rgb_out, float* depth_out) {
  NvtxRange nvtx_("prenom.render");
  if (!o || !origins || !dirs) return fail(PRENOM_USAGE, "NULL argument");
  if (n_rays < 1) return fail(PRENOM_USAGE, "n_rays must be >= 1");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  STATUS_TRY(drop_prefetch(o));  // render reuses the sample buffers a prefetched step would read
  const int S = o->cfg.samples_per_ray;
  STATUS_TRY(ensure_scratch(o, n_rays, S));
  cudaStream_t st = o->ctx->stream;
  DevBuf<float> d_o, d_d, d_rgb, d_dep;
  CUDA_TRY(d_o.ensure(3 * (size_t)n_rays));
  CUDA_TRY(d_d.ensure(3 * (size_t)n_rays));
  CUDA_TRY(d_rgb.ensure(3 * (size_t)n_rays));
  CUDA_TRY(d_dep.ensure(n_rays));
  CUDA_TRY(cudaMemcpyAsync(d_o.p, origins, 3 * sizeof(float) * n_rays, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_d.p, dirs, 3 * sizeof(float) * n_rays, cudaMemcpyHostToDevice, st));
  RaySource src;
  std::memset(&src, 0, sizeof src);
  src.mode = 1;
  src.origins = d_o.p;
  src.dirs = d_d.p;
  const SampleBufs sb = bufs(o);
  CUDA_TRY(launch_sample(src, sampler_cfg(o, n_rays, o->cfg.prior_sampling, PRENOM_TAG_RENDER,
                                          (uint32_t)o->render_calls++), sb, nullptr, st));
  if (uses_tc(o))
    CUDA_TRY(launch_fwd_tc(o->fd, o->params.p, (long long)n_rays * S, S, sb.count, sb.pos_depth, o->feat_tc.p,
                           o->out.p, o->flag.p, o->tile_ctr.p, tc_split(o), st));
  else
    CUDA_TRY(launch_field_fwd_train(o->fd, o->params.p, n_rays, S, sb, o->feat_t.p, o->out.p, o->flag.p, st));
  CompositeArgs ca;
  std::memset(&ca, 0, sizeof ca);
  ca.B = n_rays;
  ca.S = S;
  ca.pos_depth = sb.pos_depth;
  ca.delta = sb.delta;
  ca.target = sb.target;
  ca.kind = sb.kind;
  ca.count = sb.count;
  ca.out = o->out.p;
  ca.color_out = d_rgb.p;
  ca.depth_out = d_dep.p;
  CUDA_TRY(cudaMemsetAsync(d_rgb.p, 0, 3 * sizeof(float) * n_rays, st));
  CUDA_TRY(cudaMemsetAsync(d_dep.p, 0, sizeof(float) * n_rays, st));
  CUDA_TRY(launch_composite(ca, st));
  o->ctx->launches += 3;
  if (rgb_out) CUDA_TRY(cudaMemcpyAsync(rgb_out, d_rgb.p, 3 * sizeof(float) * n_rays, cudaMemcpyDeviceToHost, st));
  if (depth_out) CUDA_TRY(cudaMemcpyAsync(depth_out, d_dep.p, sizeof(float) * n_rays, cudaMemcpyDeviceToHost, st));
  return check_flag(o);
}

prenom_status prenom_density_query(prenom_object_t o, int R, float* out, int update) {
  NvtxRange nvtx_("prenom.density_query");
  if (!o) return fail(PRENOM_USAGE, "NULL object");
  if (R < 2 || R > 1024) return fail(PRENOM_DATA, "grid resolution out of range");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  cudaStream_t st = o->ctx->stream;
  const size_t n = (size_t)R * R * R;
  DevBuf<float>& d = o->query;  // kept across calls (no per-query cudaMalloc/cudaFree)
  CUDA_TRY(d.ensure(n));  // (never the live sampling grid: update swaps the two)
  CUDA_TRY(launch_refresh_grid(o->fd, o->params.p, R, d.p, o->flag.p, st));
  o->ctx->launches += 1;
  if (out) CUDA_TRY(cudaMemcpyAsync(out, d.p, n * sizeof(float), cudaMemcpyDeviceToHost, st));
  if (update) {
    STATUS_TRY(drop_prefetch(o));  // the sampling grid is replaced
    CUDA_TRY(cudaStreamSynchronize(st));
    std::swap(o->grid.p, d.p);
    std::swap(o->grid.n, d.n);
    o->R = R;
  }
  return check_flag(o);
}

// train_track's tail (mapper.cpp:186-187): refresh_grid at R, choose_iso
// (density_grid.cpp:134-136) unless iso is given, marching_cubes
// (marching_cubes.cpp:125-180) -- all on the device; the mesh stays in the
// object until prenom_get_mesh copies it out.
prenom_status prenom_extract_mesh(prenom_object_t o, int R, float iso, float iso_floor, float* iso_used,
                                  int64_t* n_vertices, int64_t* n_triangles) {
  NvtxRange nvtx_("prenom.extract_mesh");
  if (!o) return fail(PRENOM_USAGE, "NULL object");
  if (R < 2 || R > 1024) return fail(PRENOM_DATA, "grid resolution out of range");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  cudaStream_t st = o->ctx->stream;
  const size_t n = (size_t)R * R * R;
  McScratch& m = o->ctx->mc;
  CUDA_TRY(m.grid.ensure(n));
  o->ctx->mc_grid_owner = nullptr;
  CUDA_TRY(launch_refresh_grid(o->fd, o->params.p, R, m.grid.p, o->flag.p, st));
  o->ctx->launches += 1;
  STATUS_TRY(check_flag(o));
  float level = iso;
  if (std::isnan(iso)) {
    CUDA_TRY(m.gmax.ensure(1));
    CUDA_TRY(launch_grid_max(m.grid.p, (long long)n, m.gmax.p, st));
    o->ctx->launches += 1;
    float mx = 0.f;
    CUDA_TRY(cudaMemcpyAsync(&mx, m.gmax.p, sizeof(float), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    level = std::fmax(0.5f * mx, iso_floor);
  }
  int launches = 0;
  o->mesh.R = R;
  o->ctx->mc_grid_owner = o;
  CUDA_TRY(run_marching_cubes(m.grid.p, R, level, m, o->mesh, st, &launches));
  o->ctx->launches += launches;
  if (iso_used) *iso_used = level;
  if (n_vertices) *n_vertices = o->mesh.n_vertices;
  if (n_triangles) *n_triangles = o->mesh.n_triangles;
  return PRENOM_OK;
}

prenom_status prenom_get_mesh_grid(prenom_object_t o, int* res, float* grid) {
  if (!o || !res) return fail(PRENOM_USAGE, "NULL argument");
  if (o->mesh.R < 2) return fail(PRENOM_USAGE, "prenom_get_mesh_grid: no mesh extracted yet");
  if (o->ctx->mc_grid_owner != o)
    return fail(PRENOM_USAGE, "prenom_get_mesh_grid: the lattice was replaced by a later extraction on this context");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  *res = o->mesh.R;
  if (grid) {
    const size_t n = (size_t)o->mesh.R * o->mesh.R * o->mesh.R;
    CUDA_TRY(cudaMemcpyAsync(grid, o->ctx->mc.grid.p, n * sizeof(float), cudaMemcpyDeviceToHost, o->ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(o->ctx->stream));
  }
  return PRENOM_OK;
}

prenom_status prenom_get_mesh(prenom_object_t o, float* vertices, int32_t* triangles) {
  if (!o) return fail(PRENOM_USAGE, "NULL object");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  cudaStream_t st = o->ctx->stream;
  const McMesh& m = o->mesh;
  if (vertices && m.n_vertices)
    CUDA_TRY(cudaMemcpyAsync(vertices, m.verts.p, 3 * sizeof(float) * m.n_vertices, cudaMemcpyDeviceToHost, st));
  if (triangles && m.n_triangles)
    CUDA_TRY(cudaMemcpyAsync(triangles, m.tris.p, 3 * sizeof(int32_t) * m.n_triangles, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return PRENOM_OK;
}

prenom_status prenom_debug_marching_cubes(prenom_ctx_t c, int R, const float* grid, float iso, int64_t* n_vertices,
                                          int64_t* n_triangles) {
  if (!c || !grid) return fail(PRENOM_USAGE, "NULL argument");
  if (R < 1 || R > 1024) return fail(PRENOM_DATA, "grid resolution out of range");
  CUDA_TRY(cudaSetDevice(c->device));
  McScratch& m = c->mc;
  c->mc_grid_owner = nullptr;
  const size_t n = (size_t)R * R * R;
  CUDA_TRY(m.grid.ensure(n));
  CUDA_TRY(cudaMemcpyAsync(m.grid.p, grid, n * sizeof(float), cudaMemcpyHostToDevice, c->stream));
  int launches = 0;
  CUDA_TRY(run_marching_cubes(m.grid.p, R, iso, m, c->mc_dbg, c->stream, &launches));
  c->launches += launches;
  if (n_vertices) *n_vertices = c->mc_dbg.n_vertices;
  if (n_triangles) *n_triangles = c->mc_dbg.n_triangles;
  return PRENOM_OK;
}

prenom_status prenom_debug_mesh_get(prenom_ctx_t c, float* vertices, int32_t* triangles) {
  if (!c) return fail(PRENOM_USAGE, "NULL context");
  CUDA_TRY(cudaSetDevice(c->device));
  const McMesh& m = c->mc_dbg;
  if (vertices && m.n_vertices)
    CUDA_TRY(cudaMemcpyAsync(vertices, m.verts.p, 3 * sizeof(float) * m.n_vertices, cudaMemcpyDeviceToHost,
                             c->stream));
  if (triangles && m.n_triangles)
    CUDA_TRY(cudaMemcpyAsync(triangles, m.tris.p, 3 * sizeof(int32_t) * m.n_triangles, cudaMemcpyDeviceToHost,
                             c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return PRENOM_OK;
}

int prenom_mc_case_triangles(int config, int* edges) {
  if (!edges) return -1;
  return mc_case_triangles(config, edges);
}

// metrics.cpp:14-22's nearest-neighbour step (kernels_metrics.cu): per query,
// the exact minimum squared distance to the cloud.
prenom_status prenom_nearest_sq(prenom_ctx_t c, int n_queries, const float* queries, int n_points,
                                const float* points, float* min_sq) {
  if (!c || (n_queries > 0 && (!queries || !min_sq)) || (n_points > 0 && !points))
    return fail(PRENOM_USAGE, "NULL argument");
  if (n_queries < 0 || n_points < 1) return fail(PRENOM_DATA, "nearest_sq: empty cloud");
  CUDA_TRY(cudaSetDevice(c->device));
  DevBuf<float> dq, dp, dout;
  CUDA_TRY(dq.ensure(3 * (size_t)n_queries));
  CUDA_TRY(dp.ensure(3 * (size_t)n_points));
  CUDA_TRY(dout.ensure((size_t)n_queries));
  CUDA_TRY(cudaMemcpyAsync(dq.p, queries, 12 * (size_t)n_queries, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(dp.p, points, 12 * (size_t)n_points, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(launch_nearest_sq(n_queries, dq.p, n_points, dp.p, dout.p, c->stream));
  c->launches += 1;
  CUDA_TRY(cudaMemcpyAsync(min_sq, dout.p, 4 * (size_t)n_queries, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return PRENOM_OK;
}

prenom_status prenom_field_eval(prenom_object_t o, int n, const float* xyz, float* sigma, float* rgb) {
  if (!o || !xyz) return fail(PRENOM_USAGE, "NULL argument");
  if (n < 0) return fail(PRENOM_USAGE, "n < 0");
  if (n == 0) return PRENOM_OK;
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  cudaStream_t st = o->ctx->stream;
  DevBuf<float> dx, ds, dr;
  CUDA_TRY(dx.ensure(3 * (size_t)n));
  CUDA_TRY(ds.ensure(n));
  CUDA_TRY(dr.ensure(3 * (size_t)n));
  CUDA_TRY(cudaMemcpyAsync(dx.p, xyz, 3 * sizeof(float) * n, cudaMemcpyHostToDevice, st));
  CUDA_TRY(launch_field_points(o->fd, o->params.p, n, dx.p, ds.p, dr.p, nullptr, nullptr, o->flag.p, st));
  o->ctx->launches += 1;
  if (sigma) CUDA_TRY(cudaMemcpyAsync(sigma, ds.p, sizeof(float) * n, cudaMemcpyDeviceToHost, st));
  if (rgb) CUDA_TRY(cudaMemcpyAsync(rgb, dr.p, 3 * sizeof(float) * n, cudaMemcpyDeviceToHost, st));
  return check_flag(o);
}
}  // extern "C"
