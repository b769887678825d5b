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
// LM-head step — one kernel, loss_unit_kernel (see below):
//   <compute>  token-parallel 2,048-token units: fp32 terms + scaled gradient
//   <reduce>   (LM-head step) the same units over the per-token terms written
//              by the fused log-prob epilogue
//   and, in the same launch, unit -> trajectory -> group -> report by the
//   last-arriving CTA of each level.
// Every reduction has a fixed shape independent of scheduling, so results are
// run-to-run deterministic; masked tokens are selected, never multiplied.
#include <type_traits>

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

// ---------------------------------------------------------------------------
// fp32 mode: token-parallel work units + a last-arriver reduction tree.
//
// A trajectory of len tokens is cut into max(1, ceil(len / kUnit)) units of
// kUnit tokens counted from its own start.  Unit c of trajectory b gets the
// slot  key(b) + c,  key(b) = b + cu[b] / kUnit — injective, with at most
// n_traj + T / kUnit + 1 slots; the owner of a slot is the last b with
// key(b) <= slot (key is strictly increasing), so no scan is needed.
// A persistent grid (a few CTAs per SM) splits the slot range into equal
// contiguous pieces; a CTA finds the owner of its first slot with one
// block-wide search, then walks its slots in order, streaming each
// trajectory's part of the piece (one contiguous token range) through a
// strided vector loop and reducing it in a fixed-shape tree: the partial
// goes to the slot of the piece's first unit of that trajectory (the other
// units' slots get zeros).  The CTA that completes a trajectory (arrival
// counter per trajectory, counted in units) sums its slots in unit order into
// traj_out[b]; the one that completes a group sums the group's trajectories
// (fixed warp tree) into group_out[g]; the one that completes the last group
// writes the report.  Every sum has a fixed shape (a function of the sizes
// only), so results are bitwise run-to-run deterministic whichever CTA
// arrives last; masked-out tokens are selected, never multiplied.
constexpr int kUnit = 2048;
constexpr int kUnitThreads = 256;
constexpr int kUnitCtasPerSm = 4;  // resident CTAs per SM (<= 64 registers)
constexpr int kRedV = 6;  // term, k3, n_act, clipped, clamps, entropy

__device__ __forceinline__ int unit_key(const int32_t* cu, int b) { return b + cu[b] / kUnit; }
__device__ __forceinline__ int n_units_of(int len) { return len > kUnit ? (len + kUnit - 1) / kUnit : 1; }

long long unit_slots(long long n_tokens, int n_traj) { return n_traj + n_tokens / kUnit + 1; }

struct UnitArgs {
  // compute mode (standalone K3): per-token log-probs
  const float* lnew;
  const float* lold;
  const float* lref;
  const float* adv;
  const float* traj_w;
  float* grad;
  tl_loss_config cfg;
  // reduce mode (fused LM-head step): per-token terms from the epilogue
  const float* term;
  const float* k3o;
  const uint8_t* flags;
  const float* ent;
  // both
  const uint8_t* mask;
  int use_mask;
  int vec_ok;
  const int32_t* cu;
  const int32_t* group_off;
  int n_traj, n_groups, agg;
  long long n_slots;
  double* unit_out;   // [slots][8]
  double* traj_out;   // [n_traj][8]: term, n_act, clipped, clamps, k3, len, entropy, 0
  double* group_out;  // [n_groups][8]: obj, masked, tokens, clipped, clamps, kl, term, entropy
  double* report;     // [TL_REPORT_LEN]
  int* ctr;           // [1] finalize arrival counter (zeroed by the streaming kernel)
};

template <int N>
__device__ __forceinline__ void warp_sum(double (&v)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
}

// Block tree of N doubles per thread -> totals valid in thread 0.  Ends with
// a barrier, so `sh` can be reused right away.
template <int N>
__device__ __forceinline__ void block_sum(double (&v)[N], double (*sh)[kUnitThreads / 32]) {
  warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < N; ++i) sh[i][w] = v[i];
  __syncthreads();
  if (threadIdx.x == 0)
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double x = 0;
#pragma unroll
      for (int j = 0; j < kUnitThreads / 32; ++j) x += sh[i][j];
      v[i] = x;
    }
  __syncthreads();
}

// Last index in [0, n) whose key is <= target (key(0) <= target; key
// non-decreasing): 256-ary block-wide search.
template <class Key>
__device__ __forceinline__ int block_find_key(int n, long long target, Key key) {
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    const int step = (hi - lo + blockDim.x - 1) / blockDim.x;
    const int idx = lo + static_cast<int>(threadIdx.x) * step;
    const int cnt = __syncthreads_count(idx < hi && key(idx) <= target);
    lo += (cnt - 1) * step;
    hi = min(hi, lo + step);
  }
  return lo;
}

// Warp-wide: last g in [0, n) with arr[g] <= x (arr[0] <= x, non-decreasing).
__device__ __forceinline__ int warp_find_last_le(const int32_t* arr, int n, int x) {
  int lo = 0, hi = n;
  const int lane = threadIdx.x & 31;
  while (hi - lo > 1) {
    const int step = (hi - lo + 31) / 32;
    const int idx = lo + lane * step;
    const unsigned m = __ballot_sync(0xffffffffu, idx < hi && arr[idx] <= x);
    lo += (__popc(m) - 1) * step;
    hi = min(hi, lo + step);
  }
  return lo;
}

// Finalize (second kernel, launched with programmatic dependent launch so it
// is resident while the streaming kernel drains): warp w of CTA c owns group
// g = 8c + w; lane j sums trajectory j's unit slots in unit order into its
// trajectory row, the warp sums the group's trajectories in a fixed tree into
// the group row, and the CTA that completes the last group (one arrival
// counter, zeroed by the streaming kernel) writes the report.
constexpr int kFinGroupsPerCta = kUnitThreads / 32;

__global__ void __launch_bounds__(kUnitThreads) loss_finalize_kernel(const UnitArgs a) {
  __shared__ double sh[8][kUnitThreads / 32];
  __shared__ int sh_flag;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = blockIdx.x * kFinGroupsPerCta + w;
  if (g < a.n_groups) {
    const int gb0 = a.group_off[g], gb1 = a.group_off[g + 1];
    double gv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int j = gb0 + lane; j < gb1; j += 32) {
      const int t0 = a.cu[j], t1 = a.cu[j + 1];
      const int s0 = unit_key(a.cu, j), nu = n_units_of(t1 - t0);
      double tv[kRedV] = {0, 0, 0, 0, 0, 0};
      for (int u = 0; u < nu; ++u) {
        const double* uo = a.unit_out + static_cast<long long>(s0 + u) * 8;
#pragma unroll
        for (int i = 0; i < kRedV; ++i) tv[i] += uo[i];
      }
      double* o = a.traj_out + static_cast<long long>(j) * 8;
      o[0] = tv[0];
      o[1] = tv[2];
      o[2] = tv[3];
      o[3] = tv[4];
      o[4] = tv[1];
      o[5] = t1 - t0;
      o[6] = tv[5];
      o[7] = 0;
      // per-trajectory objective term / n_act, skipped when n = 0 (loss.py:173-174)
      gv[0] += tv[2] > 0 ? tv[0] / tv[2] : 0.0;
      gv[1] += tv[2];
      gv[2] += t1 - t0;
      gv[3] += tv[3];
      gv[4] += tv[4];
      gv[5] += tv[1];
      gv[6] += tv[0];
      gv[7] += tv[5];
    }
    warp_sum(gv);
    if (lane == 0) {
      double* o = a.group_out + static_cast<long long>(g) * 8;
      o[0] = gv[0] / (gb1 - gb0);
#pragma unroll
      for (int i = 1; i < 8; ++i) o[i] = gv[i];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    sh_flag = atomicAdd(a.ctr, 1) == static_cast<int>(gridDim.x) - 1;
  }
  __syncthreads();
  if (!sh_flag) return;
  // batch report over all groups (fixed order per thread, then the tree)
  __threadfence();
  double r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int gg = threadIdx.x; gg < a.n_groups; gg += kUnitThreads) {
    const double* o = a.group_out + static_cast<long long>(gg) * 8;
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] += __ldcg(o + i);
  }
  block_sum(r, sh);
  if (threadIdx.x != 0) return;
  const double obj = r[0], masked = r[1], term = r[6];
  double* rep = a.report;
  rep[0] = a.agg == 1 ? (masked > 0 ? term / masked : 0.0) : (a.n_groups ? obj / a.n_groups : 0.0);
  rep[1] = masked > 0 ? r[3] / masked : 0.0;
  rep[2] = masked;
  rep[3] = masked > 0 ? r[5] / masked : 0.0;
  rep[4] = a.n_groups;
  rep[5] = a.n_traj;
  rep[6] = r[2];
  rep[7] = r[4];
  rep[8] = r[3];
  rep[9] = r[5];
  rep[10] = r[7];
  rep[11] = a.agg == 1 ? term : obj;
  *a.ctr = 0;  // ready for the next launch
}

// Streaming kernel: per-token terms (and gradient) over the CTA's contiguous
// piece of the slot range, one fixed-shape block tree per (piece, trajectory)
// into the slot of the piece's first unit of that trajectory.
template <bool kCompute, bool kRef = false, int kObj = 0>
__global__ void __launch_bounds__(kUnitThreads, kUnitCtasPerSm) loss_unit_kernel(const UnitArgs a) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int kPark = 16;  // trajectory pieces parked before a block flush
  constexpr int kWarps = kUnitThreads / 32;
  __shared__ double park[kPark][kWarps][kRedV];
  __shared__ int park_slot[kPark], park_units[kPark];
  int n_park = 0;
  // sum the parked warp partials in warp order -> the slot of the piece's
  // first unit of each trajectory, zeros in the slots of the folded units
  auto flush = [&]() {
    __syncthreads();
    for (int j = threadIdx.x; j < n_park; j += kUnitThreads) {
      double* uo = a.unit_out + static_cast<long long>(park_slot[j]) * 8;
#pragma unroll
      for (int i = 0; i < kRedV; ++i) {
        double x = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) x += park[j][w][i];
        uo[i] = x;
      }
      for (int c = 1; c < park_units[j]; ++c)
#pragma unroll
        for (int i = 0; i < kRedV; ++i) uo[c * 8 + i] = 0.0;
    }
    __syncthreads();
    n_park = 0;
  };
  const int32_t* cu = a.cu;
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.ctr = 0;  // finalize's arrival counter
  // this CTA's contiguous piece of the slot range
  const long long s_begin = a.n_slots * blockIdx.x / gridDim.x;
  const long long s_end = a.n_slots * (blockIdx.x + 1) / gridDim.x;
  if (s_begin >= s_end) return;
  int b = block_find_key(a.n_traj, s_begin, [cu](int i) { return unit_key(cu, i); });
  long long s = s_begin;
  const float lo = static_cast<float>(1.0 - a.cfg.eps_low);
  const float hi = static_cast<float>(1.0 + a.cfg.eps_high);
  const float beta = static_cast<float>(a.cfg.kl_beta);
  constexpr bool has_ref = kCompute && kRef;
  while (s < s_end && b < a.n_traj) {
    const int t0 = cu[b], t1 = cu[b + 1];
    const int kb = b + t0 / kUnit, nb = n_units_of(t1 - t0);
    if (s >= kb + nb) {  // gap slot(s) after trajectory b
      ++b;
      continue;
    }
    if (s < kb) s = kb;
    if (s >= s_end) break;
    const int c0 = static_cast<int>(s - kb);
    const long long rem = s_end - kb;
    const int c1 = rem < nb ? static_cast<int>(rem) : nb;
    const int u0 = min(t1, t0 + c0 * kUnit), u1 = min(t1, t0 + c1 * kUnit);

    // per-thread partials: integer counts, and sums in fp64 for the fused
    // step's reductions (so its report is invariant, to ~1e-15, under
    // re-packing: data-parallel shards, micro-batches) or fp32 for the
    // standalone K3 (a few dozen same-sign terms per thread; its result is
    // deterministic for a given packing, fp32-exact to ~1e-9 across packings)
    using Acc = std::conditional_t<kCompute, float, double>;
    Acc f_term = 0, f_k3 = 0, f_ent = 0;
    int n_act = 0, n_clip = 0, n_clamp = 0;
    float adv = 0.f, wt = 0.f;
    if constexpr (kCompute) {
      adv = a.adv[b];
      wt = a.traj_w ? a.traj_w[b] : 0.f;
    }
    auto tok = [&](float x0, float x1, float x2, uint8_t fl, bool act) -> float {
      if (!act) return 0.f;
      if constexpr (kCompute) {
        const TokTermB o = grpo_token_t<kRef, kObj>(x0, x1, x2, adv, lo, hi, beta);
        f_term += o.term;
        f_k3 += o.k3;
        n_act += 1;
        n_clip += o.clipped;
        n_clamp += o.clamped;
        return o.dterm * wt;
      } else {
        f_term += x0;
        f_k3 += x1;
        n_act += 1;
        n_clip += (fl & kFlagClipped) ? 1 : 0;
        n_clamp += (fl & kFlagClamped) ? 1 : 0;
        f_ent += x2;
        return 0.f;
      }
    };
    auto scalar = [&](int t) {
      const bool act = !a.use_mask || a.mask[t];
      if constexpr (kCompute) {
        const float g = act ? tok(a.lnew[t], a.lold[t], has_ref ? a.lref[t] : 0.f, 0, true) : 0.f;
        if (a.grad) a.grad[t] = g;
      } else {
        if (act) tok(a.term[t], a.k3o[t], a.ent ? a.ent[t] : 0.f, a.flags[t], true);
      }
    };
    // 16-byte vectors over the 4-aligned body, scalar head / tail.  The body
    // runs in batches of kBatch quads per thread: every load of a batch
    // (masks, then the log-probs of quads with an action token) is issued
    // before any is consumed, so a thread keeps kBatch x 3 x 16 bytes in
    // flight instead of one dependent mask -> log-prob round trip per quad.
    const int b0 = (u0 + 3) & ~3, b1 = u1 & ~3;
    if (!a.vec_ok || b0 >= b1) {
      for (int t = u0 + threadIdx.x; t < u1; t += kUnitThreads) scalar(t);
    } else {
      if (u0 + static_cast<int>(threadIdx.x) < b0) scalar(u0 + threadIdx.x);
      if (b1 + static_cast<int>(threadIdx.x) < u1) scalar(b1 + threadIdx.x);
      constexpr int kBatch = 2;
      constexpr int kStride = 4 * kUnitThreads;
      for (int base = b0 + 4 * threadIdx.x; base < b1; base += kBatch * kStride) {
        uchar4 m[kBatch];
        float4 x0[kBatch], x1[kBatch], x2[kBatch];
        uchar4 fl[kBatch];
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
          const int t = base + j * kStride;
          m[j] = t >= b1 ? make_uchar4(0, 0, 0, 0)
                         : (a.use_mask ? __ldg(reinterpret_cast<const uchar4*>(a.mask + t))
                                       : make_uchar4(1, 1, 1, 1));
        }
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
          const int t = base + j * kStride;
          // a quad's values are loaded whatever its mask, so the batch's loads
          // do not wait on the mask loads (observation values are read and
          // ignored: the kernel is latency-, not bandwidth-bound; -1.5 % vs
          // loading only quads with an action token, gpu_s3f)
          const bool any = t < b1;
          const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
          if constexpr (kCompute) {
            x0[j] = any ? __ldg(reinterpret_cast<const float4*>(a.lnew + t)) : z;
            x1[j] = any ? __ldg(reinterpret_cast<const float4*>(a.lold + t)) : z;
            x2[j] = any && has_ref ? __ldg(reinterpret_cast<const float4*>(a.lref + t)) : z;
            fl[j] = make_uchar4(0, 0, 0, 0);
          } else {
            x0[j] = any ? __ldg(reinterpret_cast<const float4*>(a.term + t)) : z;
            x1[j] = any ? __ldg(reinterpret_cast<const float4*>(a.k3o + t)) : z;
            x2[j] = any && a.ent ? __ldg(reinterpret_cast<const float4*>(a.ent + t)) : z;
            fl[j] = any ? __ldg(reinterpret_cast<const uchar4*>(a.flags + t)) : make_uchar4(0, 0, 0, 0);
          }
        }
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
          const int t = base + j * kStride;
          float4 gr;
          gr.x = tok(x0[j].x, x1[j].x, x2[j].x, fl[j].x, m[j].x);
          gr.y = tok(x0[j].y, x1[j].y, x2[j].y, fl[j].y, m[j].y);
          gr.z = tok(x0[j].z, x1[j].z, x2[j].z, fl[j].z, m[j].z);
          gr.w = tok(x0[j].w, x1[j].w, x2[j].w, fl[j].w, m[j].w);
          if constexpr (kCompute) {
            if (t < b1 && a.grad) *reinterpret_cast<float4*>(a.grad + t) = gr;
          }
        }
      }
    }
    // warp partial (fixed shuffle tree) parked per (trajectory of the piece,
    // warp); no block barrier per trajectory — warps run through the piece
    // independently and the block combines the parked partials in warp order
    double v[kRedV] = {f_term, f_k3, static_cast<double>(n_act), static_cast<double>(n_clip),
                       static_cast<double>(n_clamp), f_ent};
    warp_sum(v);
    if ((threadIdx.x & 31) == 0)
#pragma unroll
      for (int i = 0; i < kRedV; ++i) park[n_park][threadIdx.x >> 5][i] = v[i];
    if (threadIdx.x == 0) {
      park_slot[n_park] = kb + c0;
      park_units[n_park] = c1 - c0;
    }
    if (++n_park == kPark) flush();
    s = kb + c1;
    ++b;
  }
  flush();
}

template <bool kCompute>
int launch_units(UnitArgs a, long long n_tokens, cudaStream_t st) {
  if (a.n_traj == 0) {  // empty batch: an all-zero report
    TL_CUDA_TRY(cudaMemsetAsync(a.report, 0, TL_REPORT_LEN * sizeof(double), st));
    return TL_OK;
  }
  TL_REQUIRE(a.n_groups > 0, TL_ERR_INVALID_ARG, "trajectories without groups");
  auto al = [](const void* p, uintptr_t n) { return (reinterpret_cast<uintptr_t>(p) & (n - 1)) == 0; };
  a.vec_ok = al(a.mask, 4) && al(a.lnew, 16) && al(a.lold, 16) && al(a.lref, 16) && al(a.grad, 16) &&
             al(a.term, 16) && al(a.k3o, 16) && al(a.flags, 4) && al(a.ent, 16);  // NULL is aligned
  a.n_slots = unit_slots(n_tokens, a.n_traj);
  const long long ctas = static_cast<long long>(num_sms()) * kUnitCtasPerSm;
  const unsigned grid = static_cast<unsigned>(a.n_slots < ctas ? a.n_slots : ctas);
  if constexpr (kCompute) {  // the config's reference / objective choices as template flags
    const int v = (a.cfg.has_ref ? 1 : 0) | (a.cfg.objective ? 2 : 0);
    if (v == 0) loss_unit_kernel<true, false, 0><<<grid, kUnitThreads, 0, st>>>(a);
    else if (v == 1) loss_unit_kernel<true, true, 0><<<grid, kUnitThreads, 0, st>>>(a);
    else if (v == 2) loss_unit_kernel<true, false, 1><<<grid, kUnitThreads, 0, st>>>(a);
    else loss_unit_kernel<true, true, 1><<<grid, kUnitThreads, 0, st>>>(a);
  } else {
    loss_unit_kernel<false><<<grid, kUnitThreads, 0, st>>>(a);
  }
  TL_LAUNCH_CHECK();
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3((a.n_groups + kFinGroupsPerCta - 1) / kFinGroupsPerCta);
  lc.blockDim = dim3(kUnitThreads);
  lc.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  TL_CUDA_TRY(cudaLaunchKernelEx(&lc, loss_finalize_kernel, a));
  count_launch(2);
  return TL_OK;
}

ReduceWs carve_reduce(Workspace& w, long long n_tokens, int n_traj, int n_groups) {
  ReduceWs r;
  r.unit_out = w.take<double>(static_cast<size_t>(unit_slots(n_tokens, n_traj)) * 8);
  r.traj_out = w.take<double>(static_cast<size_t>(n_traj) * 8);
  r.group_out = w.take<double>(static_cast<size_t>(n_groups) * 8);
  r.ctr = w.take<int>(1);
  return r;
}

int launch_reductions(const float* term, const float* k3o, const uint8_t* flags, const float* ent,
                      const uint8_t* mask, int use_mask, const int32_t* cu, const int32_t* group_off,
                      int n_traj, int n_groups, long long n_tokens, int agg, const ReduceWs& r,
                      double* report, cudaStream_t st) {
  ProfScope prof(PROF_REDUCE, st);
  UnitArgs a{};
  a.term = term;
  a.k3o = k3o;
  a.flags = flags;
  a.ent = ent;
  a.mask = mask;
  a.use_mask = use_mask;
  a.cu = cu;
  a.group_off = group_off;
  a.n_traj = n_traj;
  a.n_groups = n_groups;
  a.agg = agg;
  a.unit_out = r.unit_out;
  a.traj_out = r.traj_out;
  a.group_out = r.group_out;
  a.report = report;
  a.ctr = r.ctr;
  return launch_units<false>(a, n_tokens, st);
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
  tl::Workspace w{nullptr, 0};
  tl::carve_reduce(w, n_tokens, n_traj, n_groups);
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
  (void)traj_of_token;  // units walk trajectories via cu_seqlens
  tl::Workspace w{static_cast<char*>(workspace), workspace_bytes};
  const tl::ReduceWs r = tl::carve_reduce(w, n_tokens, n_traj, n_groups);
  TL_REQUIRE(w.ok(), TL_ERR_WORKSPACE, "loss_f32 workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  tl::ProfScope prof(tl::PROF_LOSS, st);
  tl::UnitArgs a{};
  a.lnew = logp_new;
  a.lold = logp_old;
  a.lref = cfg->has_ref ? logp_ref : nullptr;
  a.adv = adv32;
  a.traj_w = traj_w;
  a.grad = grad;
  a.cfg = *cfg;
  a.mask = mask;
  a.use_mask = cfg->use_mask;
  a.cu = cu_seqlens;
  a.group_off = group_off;
  a.n_traj = n_traj;
  a.n_groups = n_groups;
  a.agg = cfg->agg;
  a.unit_out = r.unit_out;
  a.traj_out = r.traj_out;
  a.group_out = r.group_out;
  a.report = report;
  a.ctr = r.ctr;
  return tl::launch_units<true>(a, n_tokens, st);
}
