// Per-token GRPO surrogate arithmetic shared by the standalone loss kernels
// (K3) and the fused LM-head epilogue (K4 combine).
//
// Reference: rl/loss.py
//   token_ratio  :119-126   r = exp(clamp(new - old, +-20))
//   _k3          :139-147   k3 = exp(d) - d - 1,  d = clamp(ref - new, +-20)
//   multi-turn   :176-191   term = min(r A, clip(r, lo, hi) A) - beta k3
//                           clipped iff (r > hi & A > 0) | (r < lo & A < 0)
//                           clamp counted iff |new - old| > 20
//   unclipped    :244-269   term = r A - beta k3;  grad = r A (0 if clamped)
//                           + beta (exp(d) - 1) inside the clamp window
// The clipped objective's gradient (build restatement, parity unpinned) takes
// the r A arm when r A <= clip(r) A, else 0.
#pragma once
#include <cstdint>

namespace tl {

constexpr float kClampF = 20.0f;
constexpr uint8_t kFlagClipped = 1, kFlagClamped = 2;

struct TokTermF {
  float term;   // contribution to the per-trajectory sum
  float k3;     // KL estimator (0 without reference)
  float dterm;  // d term / d logp_new (unscaled)
  uint8_t flags;
};

__device__ __forceinline__ TokTermF grpo_token_f32(float lnew, float lold, float lref, bool has_ref,
                                                   float adv, float lo, float hi, float beta,
                                                   int objective) {
  TokTermF o;
  const float d = lnew - lold;
  const bool clamped = d > kClampF || d < -kClampF;
  const float dc = fminf(fmaxf(d, -kClampF), kClampF);
  const float r = expf(dc);
  const float ra = r * adv;
  o.flags = clamped ? kFlagClamped : 0;
  if (objective == 0) {
    const float ca = fminf(fmaxf(r, lo), hi) * adv;
    o.term = ca < ra ? ca : ra;
    if ((r > hi && adv > 0.f) || (r < lo && adv < 0.f)) o.flags |= kFlagClipped;
    o.dterm = (!clamped && ra <= ca) ? ra : 0.f;
  } else {
    o.term = ra;
    o.dterm = clamped ? 0.f : ra;
  }
  o.k3 = 0.f;
  if (has_ref) {
    const float e = lref - lnew;
    const float ec = fminf(fmaxf(e, -kClampF), kClampF);
    const float ee = expf(ec);
    o.k3 = (ee - ec) - 1.f;
    o.term -= beta * o.k3;
    if (e >= -kClampF && e <= kClampF) o.dterm += beta * (ee - 1.f);
  }
  return o;
}

// The same arithmetic with the reference / objective choices as template
// parameters and the diagnostics as booleans (the standalone K3 streaming
// kernel: no per-token branches on the config, no flag-byte round trip).
// A NaN reference log-prob (TokenRecord.logp_ref is None) is selected out.
struct TokTermB {
  float term, k3, dterm;
  bool clipped, clamped;
};

template <bool kRef, int kObjective>
__device__ __forceinline__ TokTermB grpo_token_t(float lnew, float lold, float lref, float adv,
                                                 float lo, float hi, float beta) {
  TokTermB o;
  const float d = lnew - lold;
  o.clamped = d > kClampF || d < -kClampF;
  const float dc = fminf(fmaxf(d, -kClampF), kClampF);
  const float r = expf(dc);
  const float ra = r * adv;
  if constexpr (kObjective == 0) {
    const float ca = fminf(fmaxf(r, lo), hi) * adv;
    o.term = ca < ra ? ca : ra;
    o.clipped = (r > hi && adv > 0.f) || (r < lo && adv < 0.f);
    o.dterm = (!o.clamped && ra <= ca) ? ra : 0.f;
  } else {
    o.term = ra;
    o.clipped = false;
    o.dterm = o.clamped ? 0.f : ra;
  }
  o.k3 = 0.f;
  if constexpr (kRef) {
    const bool ok = lref == lref;
    const float e = lref - lnew;
    const float ec = fminf(fmaxf(e, -kClampF), kClampF);
    const float ee = expf(ec);
    const float k3 = (ee - ec) - 1.f;
    o.k3 = ok ? k3 : 0.f;
    o.term = ok ? o.term - beta * k3 : o.term;
    o.dterm = (ok && e >= -kClampF && e <= kClampF) ? o.dterm + beta * (ee - 1.f) : o.dterm;
  }
  return o;
}

}  // namespace tl
