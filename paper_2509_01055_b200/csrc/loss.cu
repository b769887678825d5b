// K3 — masked clipped GRPO surrogate, its diagnostics and per-token gradient.
//
// fp64 parity mode (tl_loss_f64): the reference's exact operation sequence.
//   loss64_token_kernel   one CTA per trajectory, per-token ratio / clip /
//                         k3 / term in fp64 (no FMA contraction, correctly
//                         rounded exp) -> workspace
//   loss64_group_kernel   one thread per group walks its trajectories and
//                         tokens in reference order (loss.py:170-193) so the
//                         sums round exactly like the Python loop; skipping
//                         (not multiplying by) the mask keeps observation
//                         tokens bitwise invisible (loss.py:9-10).
//   report64_kernel       cli.loss aggregation (cli.py:317-345).
// fp32 performance mode (tl_loss_f32), also the back half of the fused
// LM-head step:
//   loss32_traj_kernel    one CTA per trajectory: fp32 terms + scaled
//                         gradient, fixed-shape tree into per-trajectory sums
//   traj_reduce_kernel    (LM-head step) per-trajectory tree over per-token
//                         terms written by the fused log-prob epilogue
//   group_reduce_kernel   one thread per group (fixed order)
//   report_kernel         one CTA, fixed order
// Every reduction has a fixed shape independent of scheduling, so results are
// run-to-run deterministic; masked tokens are selected, never multiplied.
#include "exact_fp64.cuh"
#include "grpo_token.cuh"
#include "loss_internal.cuh"
#include "tl_common.cuh"

namespace tl {
namespace {

constexpr double kClampD = 20.0;

// Python min(a, b) / max(a, b) on floats: first argument wins ties.
__device__ __forceinline__ double py_min(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double py_max(double a, double b) { return b > a ? b : a; }
__device__ __forceinline__ double clamp20(double d) {
  return d > kClampD ? kClampD : (d < -kClampD ? -kClampD : d);
}

__global__ void __launch_bounds__(256)
    loss64_token_kernel(const double* __restrict__ lnew, const double* __restrict__ lold,
                        const double* __restrict__ lref, const uint8_t* __restrict__ mask,
                        const int32_t* __restrict__ cu, const double* __restrict__ adv,
                        tl_loss_config cfg, double* __restrict__ term, double* __restrict__ k3o,
                        double* __restrict__ dterm, uint8_t* __restrict__ flags) {
  const int b = blockIdx.x;
  const int t0 = cu[b], t1 = cu[b + 1];
  const double a = adv[b];
  const double lo = __dadd_rn(1.0, -cfg.eps_low), hi = __dadd_rn(1.0, cfg.eps_high);
  for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
    double tm = 0.0, kk = 0.0, g = 0.0;
    uint8_t fl = 0;
    if (!cfg.use_mask || mask[t]) {
      const double nw = lnew[t];
      const double d = __dadd_rn(nw, -lold[t]);
      const bool clamped = d > kClampD || d < -kClampD;
      if (clamped) fl |= kFlagClamped;
      const double r = cr_exp(clamp20(d));
      const double ra = __dmul_rn(r, a);
      if (cfg.objective == 0) {
        const double ca = __dmul_rn(py_min(py_max(r, lo), hi), a);
        tm = py_min(ra, ca);
        if ((r > hi && a > 0.0) || (r < lo && a < 0.0)) fl |= kFlagClipped;
        g = (!clamped && ra <= ca) ? ra : 0.0;
      } else {
        tm = ra;
        g = clamped ? 0.0 : ra;
      }
      if (cfg.has_ref && lref[t] == lref[t]) {  // NaN = TokenRecord.logp_ref is None
        const double e = __dadd_rn(lref[t], -nw);
        const double ec = clamp20(e);
        const double ee = cr_exp(ec);
        kk = __dadd_rn(__dadd_rn(ee, -ec), -1.0);
        tm = __dadd_rn(tm, -__dmul_rn(cfg.kl_beta, kk));
        if (e >= -kClampD && e <= kClampD) g = __dadd_rn(g, __dmul_rn(cfg.kl_beta, __dadd_rn(ee, -1.0)));
      }
    }
    term[t] = tm;
    k3o[t] = kk;
    dterm[t] = g;
    flags[t] = fl;
  }
}

__global__ void loss64_group_kernel(const uint8_t* __restrict__ mask, const int32_t* __restrict__ cu,
                                    const int32_t* __restrict__ group_off, int n_groups,
                                    tl_loss_config cfg, const double* __restrict__ term,
                                    const double* __restrict__ k3o, const double* __restrict__ dterm,
                                    const uint8_t* __restrict__ flags, double* __restrict__ grad,
                                    double* __restrict__ group_out) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_groups) return;
  const int b0 = group_off[g], b1 = group_off[g + 1];
  const int G = b1 - b0;
  double total = 0.0, kl_sum = 0.0;
  long long masked = 0, total_tokens = 0, clipped = 0, clamps = 0;
  for (int b = b0; b < b1; ++b) {
    const int t0 = cu[b], t1 = cu[b + 1];
    total_tokens += t1 - t0;
    long long n_act = 0;
    if (cfg.use_mask) {
      for (int t = t0; t < t1; ++t) n_act += mask[t] ? 1 : 0;
    } else {
      n_act = t1 - t0;
    }
    if (n_act == 0) {
      if (grad)
        for (int t = t0; t < t1; ++t) grad[t] = 0.0;
      continue;
    }
    // scale = 1.0 / (n_actions * g)   (loss.py:255; integer product first)
    const double scale = __ddiv_rn(1.0, static_cast<double>(n_act * G));
    double acc = 0.0;
    for (int t = t0; t < t1; ++t) {
      if (cfg.use_mask && !mask[t]) {
        if (grad) grad[t] = 0.0;
        continue;
      }
      ++masked;
      const uint8_t f = flags[t];
      clamps += (f & kFlagClamped) ? 1 : 0;
      clipped += (f & kFlagClipped) ? 1 : 0;
      if (cfg.has_ref) kl_sum = __dadd_rn(kl_sum, k3o[t]);
      acc = __dadd_rn(acc, term[t]);
      if (grad) grad[t] = __dmul_rn(dterm[t], scale);
    }
    total = __dadd_rn(total, __ddiv_rn(acc, static_cast<double>(n_act)));
  }
  double* o = group_out + static_cast<long long>(g) * TL_GROUP_OUT_LEN;
  o[0] = __ddiv_rn(total, static_cast<double>(G));
  o[1] = static_cast<double>(masked);
  o[2] = static_cast<double>(total_tokens);
  o[3] = static_cast<double>(clipped);
  o[4] = static_cast<double>(clamps);
  o[5] = kl_sum;
  o[6] = masked ? __ddiv_rn(static_cast<double>(clipped), static_cast<double>(masked)) : 0.0;
  o[7] = masked ? __ddiv_rn(kl_sum, static_cast<double>(masked)) : 0.0;
}

__global__ void report64_kernel(const double* __restrict__ go, int n_groups, int n_traj,
                                double* __restrict__ rep) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double obj_sum = 0.0, clip_w = 0.0, kl_w = 0.0;
  long long masked_total = 0;
  double total_tokens = 0, clamps = 0, clipped = 0, kl_sum = 0;
  for (int g = 0; g < n_groups; ++g) {
    const double* o = go + static_cast<long long>(g) * TL_GROUP_OUT_LEN;
    obj_sum = __dadd_rn(obj_sum, o[0]);
    const long long m = static_cast<long long>(o[1]);
    masked_total += m;
    clip_w = __dadd_rn(clip_w, __dmul_rn(o[6], static_cast<double>(m)));
    kl_w = __dadd_rn(kl_w, __dmul_rn(o[7], static_cast<double>(m)));
    total_tokens += o[2];
    clipped += o[3];
    clamps += o[4];
    kl_sum += o[5];
  }
  const double mt = static_cast<double>(masked_total);
  rep[0] = n_groups ? __ddiv_rn(obj_sum, static_cast<double>(n_groups)) : 0.0;
  rep[1] = masked_total ? __ddiv_rn(clip_w, mt) : 0.0;
  rep[2] = mt;
  rep[3] = masked_total ? __ddiv_rn(kl_w, mt) : 0.0;
  rep[4] = n_groups;
  rep[5] = n_traj;
  rep[6] = total_tokens;
  rep[7] = clamps;
  rep[8] = clipped;
  rep[9] = kl_sum;
  rep[10] = 0.0;
  rep[11] = obj_sum;
}

__global__ void ratio64_kernel(const double* __restrict__ a, const double* __restrict__ b,
                               long long n, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = cr_exp(clamp20(__dadd_rn(a[i], -b[i])));
}

}  // namespace

// One CTA per trajectory: fixed-shape tree over the trajectory's packed
// range.  traj_out[b] = {sum term, n_act, clipped, clamps, sum k3, len,
// sum entropy, 0}.
__global__ void __launch_bounds__(256)
    traj_reduce_kernel(const float* __restrict__ term, const float* __restrict__ k3o,
                       const uint8_t* __restrict__ flags, const float* __restrict__ ent,
                       const uint8_t* __restrict__ mask, int use_mask,
                       const int32_t* __restrict__ cu, double* __restrict__ traj_out) {
  constexpr int kV = 6;
  __shared__ double sh[kV][256 / 32];
  const int b = blockIdx.x;
  const int t0 = cu[b], t1 = cu[b + 1];
  double v[kV] = {0, 0, 0, 0, 0, 0};  // term, k3, ent, n_act, clipped, clamps
  for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
    if (use_mask && !mask[t]) continue;
    v[0] += term[t];
    v[1] += k3o[t];
    if (ent) v[2] += ent[t];
    v[3] += 1.0;
    const uint8_t f = flags[t];
    v[4] += (f & kFlagClipped) ? 1.0 : 0.0;
    v[5] += (f & kFlagClamped) ? 1.0 : 0.0;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < kV; ++i) {
    double x = v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) sh[i][w] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double r[kV];
    for (int i = 0; i < kV; ++i) {
      double x = 0;
      for (int j = 0; j < (int)(blockDim.x / 32); ++j) x += sh[i][j];
      r[i] = x;
    }
    double* o = traj_out + static_cast<long long>(b) * 8;
    o[0] = r[0];
    o[1] = r[3];
    o[2] = r[4];
    o[3] = r[5];
    o[4] = r[1];
    o[5] = t1 - t0;
    o[6] = r[2];
    o[7] = 0;
  }
}

// One thread per group; group_out row as in tl_loss_f64.
__global__ void group_reduce_kernel(const double* __restrict__ traj_out,
                                    const int32_t* __restrict__ group_off, int n_groups,
                                    double* __restrict__ group_out) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_groups) return;
  const int b0 = group_off[g], b1 = group_off[g + 1];
  double total = 0, masked = 0, tokens = 0, clipped = 0, clamps = 0, kl = 0;
  for (int b = b0; b < b1; ++b) {
    const double* t = traj_out + static_cast<long long>(b) * 8;
    tokens += t[5];
    if (t[1] == 0) continue;
    total += t[0] / t[1];
    masked += t[1];
    clipped += t[2];
    clamps += t[3];
    kl += t[4];
  }
  double* o = group_out + static_cast<long long>(g) * TL_GROUP_OUT_LEN;
  o[0] = total / (b1 - b0);
  o[1] = masked;
  o[2] = tokens;
  o[3] = clipped;
  o[4] = clamps;
  o[5] = kl;
  o[6] = masked > 0 ? clipped / masked : 0.0;
  o[7] = masked > 0 ? kl / masked : 0.0;
}

// Batch report (one CTA, fixed-shape tree).  agg = 1 (token-mean):
// objective = sum(term) / sum(mask).
__global__ void __launch_bounds__(256)
    report_kernel(const double* __restrict__ group_out, const double* __restrict__ traj_out,
                  int n_groups, int n_traj, int agg, double* __restrict__ rep) {
  constexpr int kV = 8;
  __shared__ double sh[kV][256 / 32];
  double v[kV] = {0, 0, 0, 0, 0, 0, 0, 0};  // obj, masked, tokens, clipped, clamps, kl, term, ent
  for (int g = threadIdx.x; g < n_groups; g += blockDim.x) {
    const double* o = group_out + static_cast<long long>(g) * TL_GROUP_OUT_LEN;
    for (int i = 0; i < 6; ++i) v[i] += o[i];
  }
  for (int b = threadIdx.x; b < n_traj; b += blockDim.x) {
    v[6] += traj_out[static_cast<long long>(b) * 8 + 0];
    v[7] += traj_out[static_cast<long long>(b) * 8 + 6];
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < kV; ++i) {
    double x = v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) sh[i][w] = x;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double r[kV];
  for (int i = 0; i < kV; ++i) {
    double x = 0;
    for (int j = 0; j < (int)(blockDim.x / 32); ++j) x += sh[i][j];
    r[i] = x;
  }
  const double obj = r[0], masked = r[1], term = r[6];
  rep[0] = agg == 1 ? (masked > 0 ? term / masked : 0.0) : (n_groups ? obj / n_groups : 0.0);
  rep[1] = masked > 0 ? r[3] / masked : 0.0;
  rep[2] = masked;
  rep[3] = masked > 0 ? r[5] / masked : 0.0;
  rep[4] = n_groups;
  rep[5] = n_traj;
  rep[6] = r[2];
  rep[7] = r[4];
  rep[8] = r[3];
  rep[9] = r[5];
  rep[10] = r[7];
  rep[11] = agg == 1 ? term : obj;
}

// Fused standalone K3 (fp32): one CTA per trajectory computes the per-token
// terms and gradient and reduces them in a fixed-shape tree straight into
// traj_out — 13 B/token in (+4 with a reference), 4 B/token out.
__global__ void __launch_bounds__(256)
    loss32_traj_kernel(const float* __restrict__ lnew, const float* __restrict__ lold,
                       const float* __restrict__ lref, const uint8_t* __restrict__ mask,
                       const int32_t* __restrict__ cu, const float* __restrict__ adv,
                       const float* __restrict__ traj_w, tl_loss_config cfg,
                       float* __restrict__ grad, double* __restrict__ traj_out, int vec_ok) {
  constexpr int kV = 5;
  __shared__ double sh[kV][256 / 32];
  const int b = blockIdx.x;
  const int t0 = cu[b], t1 = cu[b + 1];
  const float a = adv[b];
  const float wt = traj_w ? traj_w[b] : 0.f;
  const float lo = static_cast<float>(1.0 - cfg.eps_low), hi = static_cast<float>(1.0 + cfg.eps_high);
  const float beta = static_cast<float>(cfg.kl_beta);
  double v[kV] = {0, 0, 0, 0, 0};  // term, k3, n_act, clipped, clamps
  auto one = [&](int t, float ln, float lf, float rf, bool act) -> float {
    if (!act) return 0.f;
    const TokTermF o = grpo_token_f32(ln, lf, rf, cfg.has_ref != 0 && rf == rf, a, lo, hi, beta,
                                      cfg.objective);
    v[0] += o.term;
    v[1] += o.k3;
    v[2] += 1.0;
    v[3] += (o.flags & kFlagClipped) ? 1.0 : 0.0;
    v[4] += (o.flags & kFlagClamped) ? 1.0 : 0.0;
    return o.dterm * wt;
  };
  auto scalar = [&](int t) {
    const bool act = !cfg.use_mask || mask[t];
    const float g = act ? one(t, lnew[t], lold[t], cfg.has_ref ? lref[t] : 0.f, true) : 0.f;
    if (grad) grad[t] = g;
  };
  // 16-byte vectors over the 4-aligned body (observation runs skip their
  // log-prob loads), scalar head / tail: trajectories start anywhere.
  const int b0 = (t0 + 3) & ~3, b1 = t1 & ~3;
  if (!vec_ok || b0 >= b1) {
    for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x) scalar(t);
  } else {
    if (t0 + static_cast<int>(threadIdx.x) < b0) scalar(t0 + threadIdx.x);
    if (b1 + static_cast<int>(threadIdx.x) < t1) scalar(b1 + threadIdx.x);
#pragma unroll 2
    for (int t = b0 + 4 * threadIdx.x; t < b1; t += 4 * blockDim.x) {
      const uchar4 m = cfg.use_mask ? *reinterpret_cast<const uchar4*>(mask + t)
                                    : make_uchar4(1, 1, 1, 1);
      float4 gr = make_float4(0.f, 0.f, 0.f, 0.f);
      if (m.x | m.y | m.z | m.w) {
        const float4 ln = *reinterpret_cast<const float4*>(lnew + t);
        const float4 lf = *reinterpret_cast<const float4*>(lold + t);
        const float4 rf = cfg.has_ref ? *reinterpret_cast<const float4*>(lref + t)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
        gr.x = one(t, ln.x, lf.x, rf.x, m.x);
        gr.y = one(t + 1, ln.y, lf.y, rf.y, m.y);
        gr.z = one(t + 2, ln.z, lf.z, rf.z, m.z);
        gr.w = one(t + 3, ln.w, lf.w, rf.w, m.w);
      }
      if (grad) *reinterpret_cast<float4*>(grad + t) = gr;
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < kV; ++i) {
    double x = v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) sh[i][w] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double r[kV];
    for (int i = 0; i < kV; ++i) {
      double x = 0;
      for (int j = 0; j < (int)(blockDim.x / 32); ++j) x += sh[i][j];
      r[i] = x;
    }
    double* o = traj_out + static_cast<long long>(b) * 8;
    o[0] = r[0];
    o[1] = r[2];
    o[2] = r[3];
    o[3] = r[4];
    o[4] = r[1];
    o[5] = t1 - t0;
    o[6] = 0;
    o[7] = 0;
  }
}

int launch_group_report(const double* traj_out, const int32_t* group_off, int n_traj,
                        int n_groups, int agg, double* group_out, double* report,
                        cudaStream_t st) {
  if (n_groups > 0) {
    group_reduce_kernel<<<(n_groups + 127) / 128, 128, 0, st>>>(traj_out, group_off, n_groups,
                                                                group_out);
    TL_LAUNCH_CHECK();
    count_launch();
  }
  report_kernel<<<1, 256, 0, st>>>(group_out, traj_out, n_groups, n_traj, agg, report);
  TL_LAUNCH_CHECK();
  count_launch();
  return TL_OK;
}

int launch_reductions(const float* term, const float* k3o, const uint8_t* flags, const float* ent,
                      const uint8_t* mask, int use_mask, const int32_t* cu, const int32_t* group_off,
                      int n_traj, int n_groups, int agg, double* traj_out, double* group_out,
                      double* report, cudaStream_t st) {
  ProfScope prof(PROF_REDUCE, st);
  if (n_traj > 0) {
    traj_reduce_kernel<<<n_traj, 256, 0, st>>>(term, k3o, flags, ent, mask, use_mask, cu, traj_out);
    TL_LAUNCH_CHECK();
    count_launch();
  }
  if (n_groups > 0) {
    group_reduce_kernel<<<(n_groups + 127) / 128, 128, 0, st>>>(traj_out, group_off, n_groups,
                                                                group_out);
    TL_LAUNCH_CHECK();
    count_launch();
  }
  report_kernel<<<1, 256, 0, st>>>(group_out, traj_out, n_groups, n_traj, agg, report);
  TL_LAUNCH_CHECK();
  count_launch();
  return TL_OK;
}

}  // namespace tl

static int check_cfg(const tl_loss_config* cfg) {
  TL_REQUIRE(cfg != nullptr, TL_ERR_INVALID_ARG, "cfg is NULL");
  TL_REQUIRE(cfg->eps_low > 0.0 && cfg->eps_low < 1.0, TL_ERR_INVALID_ARG,
             "epsilon_clip must lie in (0, 1)");
  TL_REQUIRE(cfg->eps_high > 0.0, TL_ERR_INVALID_ARG, "eps_high must be positive");
  TL_REQUIRE(cfg->kl_beta >= 0.0, TL_ERR_INVALID_ARG, "kl_beta must be non-negative");
  TL_REQUIRE(cfg->objective == 0 || cfg->objective == 1, TL_ERR_INVALID_ARG, "objective");
  TL_REQUIRE(cfg->agg == 0 || cfg->agg == 1, TL_ERR_INVALID_ARG, "agg");
  return TL_OK;
}

extern "C" size_t tl_loss_f64_workspace_bytes(int64_t n_tokens) {
  tl::Workspace w{nullptr, 0};
  w.take<double>(n_tokens);
  w.take<double>(n_tokens);
  w.take<double>(n_tokens);
  w.take<uint8_t>(n_tokens);
  return w.used + 256;
}

extern "C" int tl_loss_f64(const double* logp_new, const double* logp_old, const double* logp_ref,
                           const uint8_t* mask, const int32_t* cu_seqlens,
                           const int32_t* group_off, const double* adv, int32_t n_traj,
                           int32_t n_groups, int64_t n_tokens, const tl_loss_config* cfg,
                           double* grad, double* group_out, void* workspace,
                           size_t workspace_bytes, tl_stream_t stream) {
  if (int e = check_cfg(cfg)) return e;
  TL_REQUIRE(!cfg->has_ref || logp_ref, TL_ERR_INVALID_ARG, "has_ref without logp_ref");
  TL_REQUIRE(!cfg->use_mask || mask, TL_ERR_INVALID_ARG, "use_mask without mask");
  tl::Workspace w{static_cast<char*>(workspace), workspace_bytes};
  double* term = w.take<double>(n_tokens);
  double* k3o = w.take<double>(n_tokens);
  double* dterm = w.take<double>(n_tokens);
  uint8_t* flags = w.take<uint8_t>(n_tokens);
  TL_REQUIRE(w.ok(), TL_ERR_WORKSPACE, "loss_f64 workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  tl::ProfScope prof(tl::PROF_LOSS, st);
  if (n_traj > 0) {
    tl::loss64_token_kernel<<<n_traj, 256, 0, st>>>(logp_new, logp_old, logp_ref, mask, cu_seqlens,
                                                    adv, *cfg, term, k3o, dterm, flags);
    TL_LAUNCH_CHECK();
    tl::count_launch();
  }
  if (n_groups > 0) {
    tl::loss64_group_kernel<<<(n_groups + 63) / 64, 64, 0, st>>>(
        mask, cu_seqlens, group_off, n_groups, *cfg, term, k3o, dterm, flags, grad, group_out);
    TL_LAUNCH_CHECK();
    tl::count_launch();
  }
  return TL_OK;
}

extern "C" int tl_report_f64(const double* group_out, int32_t n_groups, int32_t n_traj,
                             double* report, tl_stream_t stream) {
  tl::report64_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(group_out, n_groups, n_traj,
                                                                      report);
  TL_LAUNCH_CHECK();
  tl::count_launch();
  return TL_OK;
}

extern "C" int tl_token_ratio_f64(const double* logp_new, const double* logp_old, int64_t n,
                                  double* ratio, tl_stream_t stream) {
  if (n <= 0) return TL_OK;
  const int grid = static_cast<int>((n + 255) / 256 > 1184 ? 1184 : (n + 255) / 256);
  tl::ratio64_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(logp_new, logp_old, n,
                                                                         ratio);
  TL_LAUNCH_CHECK();
  tl::count_launch();
  return TL_OK;
}

extern "C" size_t tl_loss_f32_workspace_bytes(int64_t n_tokens, int32_t n_traj, int32_t n_groups) {
  (void)n_tokens;
  tl::Workspace w{nullptr, 0};
  w.take<double>(static_cast<size_t>(n_traj) * 8);
  w.take<double>(static_cast<size_t>(n_groups) * TL_GROUP_OUT_LEN);
  return w.used + 256;
}

extern "C" int tl_loss_f32(const float* logp_new, const float* logp_old, const float* logp_ref,
                           const uint8_t* mask, const int32_t* traj_of_token,
                           const int32_t* cu_seqlens, const int32_t* group_off, const float* adv32,
                           const float* traj_w, int32_t n_traj, int32_t n_groups,
                           int64_t n_tokens, const tl_loss_config* cfg, float* grad,
                           double* report, void* workspace, size_t workspace_bytes,
                           tl_stream_t stream) {
  if (int e = check_cfg(cfg)) return e;
  TL_REQUIRE(!cfg->has_ref || logp_ref, TL_ERR_INVALID_ARG, "has_ref without logp_ref");
  TL_REQUIRE(!cfg->use_mask || mask, TL_ERR_INVALID_ARG, "use_mask without mask");
  TL_REQUIRE(!grad || traj_w, TL_ERR_INVALID_ARG, "grad requires traj_w");
  (void)traj_of_token;  // the fused kernel walks trajectories via cu_seqlens
  tl::Workspace w{static_cast<char*>(workspace), workspace_bytes};
  double* traj_out = w.take<double>(static_cast<size_t>(n_traj) * 8);
  double* group_out = w.take<double>(static_cast<size_t>(n_groups) * TL_GROUP_OUT_LEN);
  TL_REQUIRE(w.ok(), TL_ERR_WORKSPACE, "loss_f32 workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  tl::ProfScope prof(tl::PROF_LOSS, st);
  if (n_traj > 0) {
    auto al = [](const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; };
    const int vec_ok = al(logp_new, 16) && al(logp_old, 16) && al(logp_ref, 16) &&
                       al(grad, 16) && al(mask, 4);  // NULL pointers are aligned
    tl::loss32_traj_kernel<<<n_traj, 256, 0, st>>>(logp_new, logp_old, logp_ref, mask, cu_seqlens,
                                                   adv32, traj_w, *cfg, grad, traj_out, vec_ok);
    TL_LAUNCH_CHECK();
    tl::count_launch();
  }
  return tl::launch_group_report(traj_out, group_off, n_traj, n_groups, cfg->agg, group_out, report,
                                 st);
}
