// capi_debug.cu -- C ABI: single-stage entry points the parity tests drive (Philox, encode, field,
// backward, Adam, sampler, loss, ray generation, tcgen05 tile GEMM).
#include "capi_internal.cuh"

using namespace prenom;
using namespace prenom_capi;

extern "C" {
// ------------------------------------------------------------- debug
prenom_status prenom_debug_philox(prenom_ctx_t ctx, int n, const uint32_t* ck, uint32_t* out) {
  if (!ctx || !ck || !out || n < 0) return fail(PRENOM_USAGE, "bad arguments");
  CUDA_TRY(cudaSetDevice(ctx->device));
  DevBuf<uint32_t> a, b;
  CUDA_TRY(a.ensure(6 * (size_t)n));
  CUDA_TRY(b.ensure(4 * (size_t)n));
  CUDA_TRY(cudaMemcpyAsync(a.p, ck, 6 * sizeof(uint32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(launch_philox(n, a.p, b.p, ctx->stream));
  ctx->launches += 1;
  CUDA_TRY(cudaMemcpyAsync(out, b.p, 4 * sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return PRENOM_OK;
}

prenom_status prenom_debug_hash_encode(prenom_ctx_t ctx, const prenom_field_arch* arch, const float* params, int n,
                                       const float* xyz, float* features) {
  if (!ctx || !params || !xyz || !features || n < 0) return fail(PRENOM_USAGE, "bad arguments");
  STATUS_TRY(validate_arch(arch));
  if (n == 0) return PRENOM_OK;
  CUDA_TRY(cudaSetDevice(ctx->device));
  const FieldDesc fd = make_desc(*arch);
  const size_t P = param_count_host(*arch);
  DevBuf<float> dp, dx, df;
  DevBuf<int> flag;
  CUDA_TRY(dp.ensure(P));
  CUDA_TRY(dx.ensure(3 * (size_t)n));
  CUDA_TRY(df.ensure((size_t)n * fd.in_dim));
  CUDA_TRY(flag.ensure(1));
  cudaStream_t st = ctx->stream;
  CUDA_TRY(cudaMemcpyAsync(dp.p, params, P * sizeof(float), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(dx.p, xyz, 3 * sizeof(float) * n, cudaMemcpyHostToDevice, st));
  CUDA_TRY(launch_field_points(fd, dp.p, n, dx.p, nullptr, nullptr, nullptr, df.p, flag.p, st));
  ctx->launches += 1;
  CUDA_TRY(cudaMemcpyAsync(features, df.p, sizeof(float) * n * fd.in_dim, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return PRENOM_OK;
}

namespace {
// prenom_debug_field_eval precision selecting the fp32 SIMT tile forward
constexpr int kDebugTileFp32 = 3;

// Points as B = n one-sample "rays" through the train-path tile kernels.
struct PointBatch {
  DevBuf<float> params, feat_t, dfeat_t, grad;
  DevBuf<unsigned char> feat_tc;
  DevBuf<float4> pos, out, dout;
  DevBuf<int> count, flag, ctr;
  SampleBufs sb;
  prenom_status init(const FieldDesc& fd, size_t P, int n, const float* h_params, const float* xyz,
                     cudaStream_t st) {
    const size_t npad = ((size_t)n + kTile - 1) / kTile * kTile;
    CUDA_TRY(params.ensure(P));
    CUDA_TRY(feat_t.ensure(npad * fd.in_dim));
    CUDA_TRY(dfeat_t.ensure(npad * fd.in_dim));
    if (tc_supported(fd)) CUDA_TRY(feat_tc.ensure(tc_feature_bytes(fd, n, 1)));  // (split-sized: fits both modes)
    CUDA_TRY(pos.ensure(npad));
    CUDA_TRY(out.ensure(npad));
    CUDA_TRY(dout.ensure(npad));
    CUDA_TRY(count.ensure(n));
    CUDA_TRY(flag.ensure(1));
    CUDA_TRY(ctr.ensure(4));
    CUDA_TRY(cudaMemset(ctr.p, 0, 4 * sizeof(int)));
    CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(int), st));
    CUDA_TRY(cudaMemcpyAsync(params.p, h_params, P * sizeof(float), cudaMemcpyHostToDevice, st));
    std::vector<float4> hp(n);
    std::vector<int> hc(n, 1);
    for (int i = 0; i < n; ++i) hp[i] = make_float4(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], 0.f);
    CUDA_TRY(cudaMemcpyAsync(pos.p, hp.data(), sizeof(float4) * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(count.p, hc.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    std::memset(&sb, 0, sizeof sb);
    sb.pos_depth = pos.p;
    sb.count = count.p;
    return PRENOM_OK;
  }
};
}  // namespace

prenom_status prenom_debug_field_eval(prenom_ctx_t ctx, const prenom_field_arch* arch, const float* params, int n,
                                      const float* xyz, float* sigma, float* rgb, float* raw, int precision) {
  if (!ctx || !params || !xyz || n < 0) return fail(PRENOM_USAGE, "bad arguments");
  STATUS_TRY(validate_arch(arch));
  if (n == 0) return PRENOM_OK;
  CUDA_TRY(cudaSetDevice(ctx->device));
  const FieldDesc fd = make_desc(*arch);
  const size_t P = param_count_host(*arch);
  cudaStream_t st = ctx->stream;
  int hflag = 0;
  if (precision == PRENOM_MLP_FP32) {
    DevBuf<float> dp, dx, ds, dr, dw;
    DevBuf<int> flag;
    CUDA_TRY(dp.ensure(P));
    CUDA_TRY(dx.ensure(3 * (size_t)n));
    CUDA_TRY(ds.ensure(n));
    CUDA_TRY(dr.ensure(3 * (size_t)n));
    CUDA_TRY(dw.ensure(4 * (size_t)n));
    CUDA_TRY(flag.ensure(1));
    CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(int), st));
    CUDA_TRY(cudaMemcpyAsync(dp.p, params, P * sizeof(float), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(dx.p, xyz, 3 * sizeof(float) * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(launch_field_points(fd, dp.p, n, dx.p, ds.p, dr.p, dw.p, nullptr, flag.p, st));
    ctx->launches += 1;
    if (sigma) CUDA_TRY(cudaMemcpyAsync(sigma, ds.p, sizeof(float) * n, cudaMemcpyDeviceToHost, st));
    if (rgb) CUDA_TRY(cudaMemcpyAsync(rgb, dr.p, 3 * sizeof(float) * n, cudaMemcpyDeviceToHost, st));
    if (raw) CUDA_TRY(cudaMemcpyAsync(raw, dw.p, 4 * sizeof(float) * n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(&hflag, flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
  } else if (precision == kDebugTileFp32 || precision == PRENOM_MLP_BF16 || precision == PRENOM_MLP_BF16X3) {
    // the train-path tile forward: fp32 smem GEMMs (kDebugTileFp32) or tcgen05
    // (bf16 / split bf16)
    const bool tc = precision != kDebugTileFp32;
    if (tc && !tc_supported(fd)) return fail(PRENOM_USAGE, "arch not supported by the tensor-core path");
    PointBatch pb;
    STATUS_TRY(pb.init(fd, P, n, params, xyz, st));
    if (tc)
      CUDA_TRY(launch_fwd_tc(fd, pb.params.p, n, 1, pb.count.p, pb.pos.p, pb.feat_tc.p, pb.out.p, pb.flag.p, pb.ctr.p,
                             precision == PRENOM_MLP_BF16X3, st));
    else
      CUDA_TRY(launch_field_fwd_train(fd, pb.params.p, n, 1, pb.sb, pb.feat_t.p, pb.out.p, pb.flag.p, st));
    ctx->launches += 1;
    std::vector<float4> h(n);
    CUDA_TRY(cudaMemcpyAsync(h.data(), pb.out.p, sizeof(float4) * n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(&hflag, pb.flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    for (int i = 0; i < n; ++i) {
      if (sigma) sigma[i] = h[i].x;
      if (rgb) {
        rgb[3 * i] = h[i].y;
        rgb[3 * i + 1] = h[i].z;
        rgb[3 * i + 2] = h[i].w;
      }
    }
    if (raw) std::memset(raw, 0, sizeof(float) * 4 * n);
  } else {
    return fail(PRENOM_USAGE, "unsupported mlp precision for debug_field_eval");
  }
  if (hflag) return fail(PRENOM_NUMERIC, "field_eval produced a non-finite output");
  return PRENOM_OK;
}

prenom_status prenom_debug_field_backward(prenom_ctx_t ctx, const prenom_field_arch* arch, const float* params,
                                          int n, const float* xyz, const float* d_sigma, const float* d_rgb,
                                          float* grad, int precision) {
  if (!ctx || !params || !xyz || !d_sigma || !d_rgb || !grad || n < 0) return fail(PRENOM_USAGE, "bad arguments");
  STATUS_TRY(validate_arch(arch));
  const FieldDesc fd = make_desc(*arch);
  const size_t P = param_count_host(*arch);
  if (n == 0) {
    std::memset(grad, 0, P * sizeof(float));
    return PRENOM_OK;
  }
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  PointBatch pb;
  STATUS_TRY(pb.init(fd, P, n, params, xyz, st));
  CUDA_TRY(pb.grad.ensure(P));
  CUDA_TRY(cudaMemsetAsync(pb.grad.p, 0, P * sizeof(float), st));
  std::vector<float4> hd(n);
  for (int i = 0; i < n; ++i) hd[i] = make_float4(d_sigma[i], d_rgb[3 * i], d_rgb[3 * i + 1], d_rgb[3 * i + 2]);
  CUDA_TRY(cudaMemcpyAsync(pb.dout.p, hd.data(), sizeof(float4) * n, cudaMemcpyHostToDevice, st));
  if (precision == PRENOM_MLP_BF16 || precision == PRENOM_MLP_BF16X3) {
    if (!tc_supported(fd)) return fail(PRENOM_USAGE, "arch not supported by the tensor-core path");
    const int split = precision == PRENOM_MLP_BF16X3;
    CUDA_TRY(init_feature_tiles(fd, pb.feat_tc.p, tc_feature_bytes(fd, n, split), split, st));
    CUDA_TRY(launch_fwd_tc(fd, pb.params.p, n, 1, pb.count.p, pb.pos.p, pb.feat_tc.p, pb.out.p, pb.flag.p, pb.ctr.p,
                           split, st));
    CUDA_TRY(launch_bwd_tc(fd, pb.params.p, pb.grad.p, n, 1, pb.count.p, pb.pos.p, pb.feat_tc.p, pb.dout.p,
                           pb.ctr.p + 2, split, nullptr, 0, st));
  } else {
    CUDA_TRY(launch_field_fwd_train(fd, pb.params.p, n, 1, pb.sb, pb.feat_t.p, pb.out.p, pb.flag.p, st));
    CUDA_TRY(launch_mlp_bwd_train(fd, pb.params.p, pb.grad.p, n, 1, pb.count.p, pb.feat_t.p, pb.dout.p,
                                  pb.dfeat_t.p, st));
    CUDA_TRY(launch_encode_bwd(fd, pb.params.p, pb.grad.p, n, 1, pb.count.p, pb.pos.p, pb.dfeat_t.p, st));
  }
  ctx->launches += 3;
  CUDA_TRY(cudaMemcpyAsync(grad, pb.grad.p, P * sizeof(float), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return PRENOM_OK;
}

prenom_status prenom_debug_adam(prenom_ctx_t ctx, size_t n, float* params, const float* grads, float* m, float* v,
                                int64_t* step, float lr, float b1, float b2, float eps) {
  if (!ctx || !params || !grads || !m || !v || !step) return fail(PRENOM_USAGE, "NULL argument");
  if (n == 0) return PRENOM_OK;
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  DevBuf<float> dp, dg, dm, dv;
  CUDA_TRY(dp.ensure(n));
  CUDA_TRY(dg.ensure(n));
  CUDA_TRY(dm.ensure(n));
  CUDA_TRY(dv.ensure(n));
  CUDA_TRY(cudaMemcpyAsync(dp.p, params, n * 4, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(dg.p, grads, n * 4, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(dm.p, m, n * 4, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(dv.p, v, n * 4, cudaMemcpyHostToDevice, st));
  *step += 1;
  const float c1 = 1.f - std::pow(b1, (float)*step), c2 = 1.f - std::pow(b2, (float)*step);
  CUDA_TRY(launch_adam(n, dp.p, dg.p, dm.p, dv.p, lr, b1, b2, eps, c1, c2, 0, st));
  ctx->launches += 1;
  CUDA_TRY(cudaMemcpyAsync(params, dp.p, n * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(m, dm.p, n * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(v, dv.p, n * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return PRENOM_OK;
}

prenom_status prenom_debug_sample_rays(prenom_ctx_t ctx, int n_rays, const float* origins, const float* dirs,
                                       const float box_min[3], const float box_max[3], int prior, int grid_res,
                                       const float* grid, int n_coarse, int n_fine, float eps, uint64_t seed,
                                       int64_t step, float* depths, float* deltas, float* positions, int* count,
                                       float* t_entry, float* t_exit) {
  if (!ctx || !origins || !dirs || !box_min || !box_max || n_rays < 0) return fail(PRENOM_USAGE, "bad arguments");
  if (prior && (!grid || grid_res < 2)) return fail(PRENOM_USAGE, "prior sampling needs a grid");
  if (n_fine < 1 || n_fine > 1024 || (prior && (n_coarse < 1 || n_coarse > 1024)))
    return fail(PRENOM_USAGE, "sample counts out of range");
  if (n_rays == 0) return PRENOM_OK;
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const size_t N = (size_t)n_rays * n_fine;
  DevBuf<float> d_o, d_d, d_g, d_delta, d_te, d_tx;
  DevBuf<float4> d_pd, d_tgt;
  DevBuf<int> d_kind, d_cnt;
  CUDA_TRY(d_o.ensure(3 * (size_t)n_rays));
  CUDA_TRY(d_d.ensure(3 * (size_t)n_rays));
  CUDA_TRY(d_pd.ensure(N));
  CUDA_TRY(d_delta.ensure(N));
  CUDA_TRY(d_tgt.ensure(n_rays));
  CUDA_TRY(d_kind.ensure(n_rays));
  CUDA_TRY(d_cnt.ensure(n_rays));
  CUDA_TRY(d_te.ensure(n_rays));
  CUDA_TRY(d_tx.ensure(n_rays));
  CUDA_TRY(cudaMemcpyAsync(d_o.p, origins, 12 * (size_t)n_rays, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_d.p, dirs, 12 * (size_t)n_rays, cudaMemcpyHostToDevice, st));
  if (prior) {
    const size_t gv = (size_t)grid_res * grid_res * grid_res;
    CUDA_TRY(d_g.ensure(gv));
    CUDA_TRY(cudaMemcpyAsync(d_g.p, grid, gv * 4, cudaMemcpyHostToDevice, st));
  }
  CUDA_TRY(cudaMemsetAsync(d_pd.p, 0, N * sizeof(float4), st));
  CUDA_TRY(cudaMemsetAsync(d_delta.p, 0, N * sizeof(float), st));
  RaySource src;
  std::memset(&src, 0, sizeof src);
  src.mode = 1;
  src.origins = d_o.p;
  src.dirs = d_d.p;
  SamplerCfg c;
  std::memset(&c, 0, sizeof c);
  c.B = n_rays;
  c.S = n_fine;
  c.prior = prior;
  c.n_coarse = n_coarse;
  c.eps = eps;
  c.grid_res = grid_res;
  c.grid = d_g.p;
  std::memcpy(c.bmin, box_min, 12);
  std::memcpy(c.bmax, box_max, 12);
  c.seed = seed;
  c.tag = PRENOM_TAG_FINE;
  c.step = (uint32_t)step;
  SampleBufs sb;
  std::memset(&sb, 0, sizeof sb);
  sb.pos_depth = d_pd.p;
  sb.delta = d_delta.p;
  sb.target = d_tgt.p;
  sb.kind = d_kind.p;
  sb.count = d_cnt.p;
  sb.t_entry = d_te.p;
  sb.t_exit = d_tx.p;
  CUDA_TRY(launch_sample(src, c, sb, nullptr, st));
  ctx->launches += 1;
  std::vector<float4> hpd(N);
  CUDA_TRY(cudaMemcpyAsync(hpd.data(), d_pd.p, N * sizeof(float4), cudaMemcpyDeviceToHost, st));
  if (deltas) CUDA_TRY(cudaMemcpyAsync(deltas, d_delta.p, N * 4, cudaMemcpyDeviceToHost, st));
  if (count) CUDA_TRY(cudaMemcpyAsync(count, d_cnt.p, 4 * (size_t)n_rays, cudaMemcpyDeviceToHost, st));
  if (t_entry) CUDA_TRY(cudaMemcpyAsync(t_entry, d_te.p, 4 * (size_t)n_rays, cudaMemcpyDeviceToHost, st));
  if (t_exit) CUDA_TRY(cudaMemcpyAsync(t_exit, d_tx.p, 4 * (size_t)n_rays, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  for (size_t i = 0; i < N; ++i) {
    if (depths) depths[i] = hpd[i].w;
    if (positions) {
      positions[3 * i] = hpd[i].x;
      positions[3 * i + 1] = hpd[i].y;
      positions[3 * i + 2] = hpd[i].z;
    }
  }
  return PRENOM_OK;
}

prenom_status prenom_debug_batch_loss(prenom_ctx_t ctx, int n_rays, int S, const int* kind, const float* target_rgb,
                                      const float* target_depth, const int* count, const float* deltas,
                                      const float* depths, const float* sigma, const float* rgb,
                                      const float* bg_colors, float lambda_d, float lambda_sigma, double* terms,
                                      float* d_sigma, float* d_rgb, float* color_out, float* depth_out) {
  if (!ctx || !kind || !target_rgb || !target_depth || !count || !deltas || !depths || !sigma || !rgb || !bg_colors ||
      !terms || n_rays < 0 || S < 1 || S > 256)
    return fail(PRENOM_USAGE, "bad arguments");
  if (n_rays == 0) return fail(PRENOM_DATA, "batch_loss: no rays");
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const size_t N = (size_t)n_rays * S;
  std::vector<float4> hpd(N), hout(N), htgt(n_rays);
  for (size_t i = 0; i < N; ++i) {
    hpd[i] = make_float4(0.f, 0.f, 0.f, depths[i]);
    hout[i] = make_float4(sigma[i], rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]);
  }
  for (int r = 0; r < n_rays; ++r) {
    if (count[r] != 0 && count[r] != S) return fail(PRENOM_USAGE, "count must be 0 or S");
    htgt[r] = make_float4(target_rgb[3 * r], target_rgb[3 * r + 1], target_rgb[3 * r + 2], target_depth[r]);
  }
  DevBuf<float4> d_pd, d_out, d_dout, d_tgt;
  DevBuf<float> d_delta, d_bg, d_col, d_dep;
  DevBuf<int> d_kind, d_cnt, d_flag;
  DevBuf<StepStatsDev> d_stats;
  CUDA_TRY(d_pd.ensure(N));
  CUDA_TRY(d_out.ensure(N));
  CUDA_TRY(d_dout.ensure(N));
  CUDA_TRY(d_tgt.ensure(n_rays));
  CUDA_TRY(d_delta.ensure(N));
  CUDA_TRY(d_bg.ensure(3 * (size_t)n_rays));
  CUDA_TRY(d_col.ensure(3 * (size_t)n_rays));
  CUDA_TRY(d_dep.ensure(n_rays));
  CUDA_TRY(d_kind.ensure(n_rays));
  CUDA_TRY(d_cnt.ensure(n_rays));
  CUDA_TRY(d_flag.ensure(1));
  CUDA_TRY(d_stats.ensure(1));
  CUDA_TRY(cudaMemcpyAsync(d_pd.p, hpd.data(), N * sizeof(float4), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_out.p, hout.data(), N * sizeof(float4), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_tgt.p, htgt.data(), n_rays * sizeof(float4), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_delta.p, deltas, N * 4, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_bg.p, bg_colors, 12 * (size_t)n_rays, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_kind.p, kind, 4 * (size_t)n_rays, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_cnt.p, count, 4 * (size_t)n_rays, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemsetAsync(d_dout.p, 0, N * sizeof(float4), st));
  CUDA_TRY(cudaMemsetAsync(d_col.p, 0, 12 * (size_t)n_rays, st));
  CUDA_TRY(cudaMemsetAsync(d_dep.p, 0, 4 * (size_t)n_rays, st));
  CUDA_TRY(cudaMemsetAsync(d_flag.p, 0, 4, st));
  CUDA_TRY(cudaMemsetAsync(d_stats.p, 0, sizeof(StepStatsDev), st));
  CompositeArgs ca;
  std::memset(&ca, 0, sizeof ca);
  ca.B = n_rays;
  ca.S = S;
  ca.pos_depth = d_pd.p;
  ca.delta = d_delta.p;
  ca.target = d_tgt.p;
  ca.kind = d_kind.p;
  ca.count = d_cnt.p;
  ca.out = d_out.p;
  ca.bg_colors = d_bg.p;
  ca.lambda_d = lambda_d;
  ca.lambda_sigma = lambda_sigma;
  ca.dout = d_dout.p;
  ca.color_out = d_col.p;
  ca.depth_out = d_dep.p;
  ca.stats = d_stats.p;
  ca.flag = d_flag.p;
  CUDA_TRY(launch_composite(ca, st));
  ctx->launches += 2;
  StepStatsDev hs;
  std::vector<float4> hd(N);
  int hflag = 0;
  CUDA_TRY(cudaMemcpyAsync(&hs, d_stats.p, sizeof hs, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(hd.data(), d_dout.p, N * sizeof(float4), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(&hflag, d_flag.p, 4, cudaMemcpyDeviceToHost, st));
  if (color_out) CUDA_TRY(cudaMemcpyAsync(color_out, d_col.p, 12 * (size_t)n_rays, cudaMemcpyDeviceToHost, st));
  if (depth_out) CUDA_TRY(cudaMemcpyAsync(depth_out, d_dep.p, 4 * (size_t)n_rays, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  terms[0] = hs.total;
  terms[1] = hs.color;
  terms[2] = hs.depth;
  terms[3] = hs.sigma;
  for (size_t i = 0; i < N; ++i) {
    if (d_sigma) d_sigma[i] = hd[i].x;
    if (d_rgb) {
      d_rgb[3 * i] = hd[i].y;
      d_rgb[3 * i + 1] = hd[i].z;
      d_rgb[3 * i + 2] = hd[i].w;
    }
  }
  if (hflag) return fail(PRENOM_NUMERIC, "batch_loss: non-finite loss");
  return PRENOM_OK;
}

prenom_status prenom_debug_generate_rays(prenom_object_t o, int frame, int64_t step, float* origins, float* dirs,
                                         int* kind, float* target_rgb, float* target_depth, int* pick_px) {
  if (!o) return fail(PRENOM_USAGE, "NULL object");
  if (frame < 0 || frame >= (int)o->frames.size()) return fail(PRENOM_USAGE, "frame index out of range");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  const int B = o->cfg.rays_per_iter;
  STATUS_TRY(drop_prefetch(o));
  STATUS_TRY(ensure_scratch(o, B, o->cfg.samples_per_ray));
  const RaySource src = frame_source(o, frame);
  if (src.n_obj_px == 0) return fail(PRENOM_DATA, "generate_rays: no object pixels");
  cudaStream_t st = o->ctx->stream;
  DevBuf<float> d_o, d_d;
  DevBuf<int> d_pick;
  CUDA_TRY(d_o.ensure(3 * (size_t)B));
  CUDA_TRY(d_d.ensure(3 * (size_t)B));
  CUDA_TRY(d_pick.ensure(B));
  SampleBufs sb = bufs(o);
  sb.ray_o = d_o.p;
  sb.ray_d = d_d.p;
  sb.pick_px = d_pick.p;
  CUDA_TRY(launch_sample(src, sampler_cfg(o, B, 0, PRENOM_TAG_FINE, (uint32_t)step), sb, nullptr, st));
  o->ctx->launches += 1;
  std::vector<float4> tg(B);
  if (origins) CUDA_TRY(cudaMemcpyAsync(origins, d_o.p, 12 * (size_t)B, cudaMemcpyDeviceToHost, st));
  if (dirs) CUDA_TRY(cudaMemcpyAsync(dirs, d_d.p, 12 * (size_t)B, cudaMemcpyDeviceToHost, st));
  if (pick_px) CUDA_TRY(cudaMemcpyAsync(pick_px, d_pick.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, st));
  if (kind) CUDA_TRY(cudaMemcpyAsync(kind, sb.kind, 4 * (size_t)B, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(tg.data(), sb.target, sizeof(float4) * B, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  for (int r = 0; r < B; ++r) {
    if (target_rgb) {
      target_rgb[3 * r] = tg[r].x;
      target_rgb[3 * r + 1] = tg[r].y;
      target_rgb[3 * r + 2] = tg[r].z;
    }
    if (target_depth) target_depth[r] = tg[r].w;
  }
  return PRENOM_OK;
}

prenom_status prenom_debug_umma_gemm(prenom_ctx_t ctx, int M, int N, int K, int a_mn, int b_mn, const float* A,
                                     const float* B, float* D) {
  if (!ctx || !A || !B || !D) return fail(PRENOM_USAGE, "NULL argument");
  if ((M != 64 && M != 128) || N < 8 || N > 256 || N % 8 || K < 16 || K % 16 || K > 256 ||
      (M == 128 && N % 16))
    return fail(PRENOM_USAGE, "unsupported UMMA shape");
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  DevBuf<float> a, b, d;
  CUDA_TRY(a.ensure((size_t)M * K));
  CUDA_TRY(b.ensure((size_t)N * K));
  CUDA_TRY(d.ensure((size_t)M * N));
  CUDA_TRY(cudaMemcpyAsync(a.p, A, sizeof(float) * M * K, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(b.p, B, sizeof(float) * N * K, cudaMemcpyHostToDevice, st));
  CUDA_TRY(launch_umma_gemm(M, N, K, a_mn, b_mn, a.p, b.p, d.p, st));
  ctx->launches += 1;
  CUDA_TRY(cudaMemcpyAsync(D, d.p, sizeof(float) * M * N, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return PRENOM_OK;
}
prenom_status prenom_debug_bwd_trace(prenom_ctx_t ctx, int64_t* mlp, int64_t* scatter, int64_t* cta) {
  if (!ctx || !mlp || !scatter) return fail(PRENOM_USAGE, "NULL argument");
  CUDA_TRY(cudaSetDevice(ctx->device));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  CUDA_TRY(tc_bwd_trace(reinterpret_cast<long long*>(mlp), reinterpret_cast<long long*>(scatter),
                        reinterpret_cast<long long*>(cta)));
  return PRENOM_OK;
}
// L2 read bandwidth probe (the L2 peak is measured on the box): one launch
// re-reads an L2-resident buffer `reps` times (float4, grid-stride), timed with events.
prenom_status prenom_debug_l2_read(prenom_ctx_t ctx, int mbytes, int reps, double* gbs) {
  if (!ctx || !gbs || mbytes < 1 || reps < 1) return fail(PRENOM_USAGE, "bad arguments");
  CUDA_TRY(cudaSetDevice(ctx->device));
  const size_t n4 = (size_t)mbytes * (1 << 20) / 16;
  DevBuf<float4> buf;
  DevBuf<float> sink;
  CUDA_TRY(buf.ensure(n4));
  CUDA_TRY(sink.ensure(1 << 20));
  CUDA_TRY(cudaMemsetAsync(buf.p, 0, n4 * 16, ctx->stream));
  float ms = 0.f;
  CUDA_TRY(launch_l2_read(buf.p, n4, 1, sink.p, ctx->stream, nullptr));  // warm: lines into L2
  CUDA_TRY(launch_l2_read(buf.p, n4, reps, sink.p, ctx->stream, &ms));
  *gbs = (double)n4 * 16.0 * reps / (ms * 1e-3) / 1e9;
  return PRENOM_OK;
}
}  // extern "C"
