// LM-head GEMM epilogues (included by lmhead.cu only; see its header for
// the per-chunk pipeline):
//   EpiLseStats   forward: per-row online log-sum-exp / E_p z / target logit
//                 over a vocab strip, logit stores for the backward (fp16 u,
//                 or bf16 q in the factored mode); the CTA finishing a
//                 128-row block's last strip merges the strips and runs the
//                 GRPO surrogate (combine_row).
//   EpiDSoftmax   recompute mode: dS = dLoss/dz straight from TMEM.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "gemm_sm100.cuh"
#include "grpo_token.cuh"

namespace tl {
namespace {

constexpr float kLog2e = 1.4426950408889634f;

// Packed fp32x2 (FFMA2 / FADD2 / FMUL2) in the forward epilogue and the dS
// pass; 0 = scalar A/B reference build (bitwise-identical results).
#ifndef TL_EPI_F32X2
#define TL_EPI_F32X2 1
#endif

// ------------------------------------------------------------- epilogues --
__device__ __forceinline__ uint32_t pack_f16x2_sat(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

struct CombineArgs {
  const float4* part;
  int n_strips, rows;
  const int32_t* idx;  // row -> packed position (nullable: identity)
  // forward-only outputs (indexed by row)
  float* logp_row;
  float* ent_row;
  float* lse_row;
  // fused loss (nullable block: forward-only when logp_old == nullptr)
  const int32_t* traj_of_token;
  const float* logp_old;
  const float* logp_ref;
  const float* adv;
  const float* traj_w;
  tl_loss_config cfg;
  float ent_grad;        // dLoss/dentropy per action token
  float* logp_out;       // [T]
  float* ent_out;        // [T]
  float* term;           // [T]
  float* k3o;            // [T]
  uint8_t* flags;        // [T]
  float* g_row;          // [C]
  float* c_row;          // [C]
  float* ez_row;         // [C]
  // factored store (EpiLseStatsT<true>; nullable anchor = off): per-row
  // scale alpha, the target column of q rewritten, out-of-range rows listed
  const float* anchor;         // [C] m0
  const int32_t* y_row;        // [C] target ids
  float* alpha_row;            // [C]
  __nv_bfloat16_raw* qout;     // [C, ldq]
  long long ldq;
  int* flagged;                // [1 + C]: count, then row ids
  int force_fixup;             // test hook (TL_LMHEAD_DEBUG_FIXUP): list every row with g != 0
};

// Factored backward (entropy_coef == 0).  dS = dLoss/dz = g (onehot(y) - p)
// is a per-row multiple of q = e^(z - m0) for any per-row anchor m0 fixed
// before the forward:  dS[r, v] = alpha_r * A[r, v]  with
//   alpha_r = -g_r e^(m0_r - lse_r),   A[r, v] = q[r, v]  (v != y_r),
//   A[r, y] = dS_y / alpha_r = expm1(logp_y) e^(lse_r - m0_r).
// So the forward stores bf16 q, the merge rewrites one element per row
// (the target) and computes alpha, and the backward needs no elementwise
// pass: dH = diag(alpha) (A W) (alpha in the dH epilogue) and
// dW = A^T (diag(alpha) h_c) (h_c scaled in place, a C x H pass).
// The anchor m0 = z~_y + clamp(-logp_old, 0, 40) (z~_y an fp32 dot product,
// gather_anchor_kernel) puts m0 near lse, so q ~ p.  d = lse - m0 must stay in
// [kQdMin, kQdMax]: above, q (<= e^d) and the dH accumulators (sum_v q W <=
// e^d max|W|) approach fp32 / bf16 range; below, tokens with p > e^(d - 87)
// would be lost to underflow.  Rows outside (only when the policy moved
// by e^40+ from logp_old, or logp_old is not a log-prob of this model) are
// listed and rewritten by fixup_rows_kernel with m0 = lse.
constexpr float kQdMin = -45.f, kQdMax = 80.f;

__device__ __forceinline__ void store_bf16(__nv_bfloat16_raw* p, float v) {
  uint32_t b;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(b) : "f"(0.f), "f"(v));
  p->x = static_cast<unsigned short>(b & 0xFFFFu);
}

// Merge a row's vocab-strip partials -> lse, logp, entropy; then the GRPO
// surrogate on logp_new (grpo_token.cuh) -> per-token term / k3 / flags and
// the row's dLoss/dlogp, dLoss/dent (K3 math fused into the log-prob
// epilogue).  Partials written by other CTAs are read with ld.global.cg.
__device__ void combine_row(const CombineArgs& a, int r) {
  float m = -INFINITY, s = 0.f, t = 0.f, zy = -INFINITY;
  for (int j = 0; j < a.n_strips; ++j) {
    const float4 q = __ldcg(a.part + static_cast<long long>(j) * a.rows + r);
    zy = fmaxf(zy, q.w);
    if (q.x == -INFINITY) continue;
    if (q.x > m) {
      const float f = expf(m - q.x);
      s = s * f + q.y;
      t = t * f + q.z;
      m = q.x;
    } else {
      const float f = expf(q.x - m);
      s += q.y * f;
      t += q.z * f;
    }
  }
  const float lse = m + logf(s);
  const float ez = t / s;
  const float logp = zy - lse;
  const float ent = lse - ez;
  if (a.logp_row) a.logp_row[r] = logp;
  if (a.ent_row) a.ent_row[r] = ent;
  if (a.lse_row) a.lse_row[r] = lse;
  if (a.logp_old) {
    const long long p = a.idx ? a.idx[r] : r;
    const int b = a.traj_of_token[p];
    const float lo = static_cast<float>(1.0 - a.cfg.eps_low);
    const float hi = static_cast<float>(1.0 + a.cfg.eps_high);
    const float rf = a.cfg.has_ref ? a.logp_ref[p] : 0.f;
    const TokTermF o = grpo_token_f32(logp, a.logp_old[p], rf, a.cfg.has_ref != 0 && rf == rf,
                                      a.adv[b], lo, hi, static_cast<float>(a.cfg.kl_beta),
                                      a.cfg.objective);
    a.logp_out[p] = logp;
    a.ent_out[p] = ent;
    a.term[p] = o.term;
    a.k3o[p] = o.k3;
    a.flags[p] = o.flags;
    const float g = -o.dterm * a.traj_w[b];  // loss = -objective
    a.g_row[r] = g;
    a.c_row[r] = a.ent_grad;
    a.ez_row[r] = ez;
    if (a.anchor) {
      const float d = lse - a.anchor[r];
      if (g == 0.f) {
        // no gradient: the row's q never matters (its dH row is written as
        // exact zeros, its h_c row scales to zero; q itself stays finite)
        a.alpha_row[r] = 0.f;
      } else if (d >= kQdMin && d <= kQdMax && !a.force_fixup) {
        a.alpha_row[r] = -g * expf(-d);
        // after every strip's q stores of this row (counter + fences)
        store_bf16(a.qout + static_cast<long long>(r) * a.ldq + a.y_row[r], expm1f(logp) * expf(d));
      } else {
        a.alpha_row[r] = 0.f;  // fixup_rows_kernel sets it
        const int k = atomicAdd(a.flagged, 1);
        a.flagged[1 + k] = r;
      }
    }
  }
}

// Online log-sum-exp over a vocab strip; one thread = one token row.
//
// Backward input (store mode): instead of the logits themselves, the
// epilogue keeps u = (z - m) log2e in fp16, where m is the row's running
// max, rounded UP to a multiple of 1/128, after the 32-column slice that
// holds z.  u <= 0 always, and the dS pass recovers p = 2^(u + (m - lse)
// log2e) and z = m + u ln2 with m read back exactly from a per-(row, slice)
// int16 offset (units of 1/128).  An fp16 error in u costs p an absolute
// error <= p |u| 2^-11 <= 2^-11 / e, and the row's top token sits within
// 1/128 of its offset (u > -0.012: fp16 spacing <= 2^-17), so the
// high-probability tokens, whose p cancels against onehot(y) in dS, keep
// ~fp32 precision.  Storing z in fp16 directly cost them up to 2^-7
// relative at |z| >= 16 (per-row dH errors up to 6.6x on p_y -> 1 rows,
// tests/test_lmhead_bwd_fullshape_gpu.py).  The quantised m also drives the
// log-sum-exp itself (any offset >= the max works).
//
// kFactored (entropy_coef == 0, see combine_row): the stores are bf16
// q = e^(z - m0) = 2^u * f with the row's fixed anchor m0 and the per-row
// factor f = 2^((m - m0) log2e), updated only when the running max m moves:
// one FMUL per logit, no offsets; the log-sum-exp itself is unchanged, so
// logp / entropy / the report are bitwise those of the fp16-u store.
constexpr float kOffScale = 128.f;             // offset units: 1/128
constexpr float kMaxOff = 32767.f / kOffScale;  // |m| cap (|z| beyond ~256: unsupported)

template <bool kFactored>
struct EpiLseStatsT {
  static constexpr bool kSplitTail = false;
  struct Params {
    const int32_t* targets;  // [C] target id of each chunk row
    float4* part;            // [n_strips, C]: (max, sum e, sum e z, z_target)
    int rows;                // C (partials row stride)
    void* zout;              // optional backward input [C, ldz]: fp16 u = (z - m) log2e, or
                             // (kFactored) bf16 q = e^(z - m0)
    long long ldz;
    int16_t* zoff;           // [C, ldo] slice offsets m (8 per 256-column tile), with zout
    long long ldo;
    int* tile_ctr;           // [ceil(C/128)] strips finished per 128-row block (zeroed)
    CombineArgs ca;          // last-strip fixup: merge + surrogate for the block's rows
    int z_policy;            // make_policy() kind of the fp16 stores
    const float* anchor;     // kFactored: [C] m0 per row
  };
  struct State {
    float m, s, t, zy;
    int y;
    uint64_t zpol;
    uint64_t olo, ohi;  // the tile's 8 slice offsets (int16), shifted in slice by slice
    float a, f;         // kFactored: m0 log2e, 2^(m log2e - a)
  };
  __device__ static void begin_unit(const Params& p, const GemmShape& sh, State& st, int row,
                                    const UnitCoord&) {
    st.m = -INFINITY;
    st.s = 0.f;
    st.t = 0.f;
    st.zy = -INFINITY;
    st.y = row < sh.M ? p.targets[row] : -1;
    st.zpol = make_policy(p.z_policy);
    st.olo = st.ohi = 0;
    st.a = kFactored && row < sh.M ? p.anchor[row] * kLog2e : 0.f;
    st.f = 0.f;
  }
  // One 32-column slice of the row: running max rescale, then sum e and
  // sum e*z with e = 2^u, u = z*log2e - m*log2e, and (store mode) fp16 u.
  // Full slices (all but the vocab tail) take a branch-free path: 3-input
  // max, one SFU op per logit, split accumulators; the target column is
  // looked up only in the one slice that holds it.
  __device__ static __forceinline__ void slice(const Params& p, const GemmShape& sh, State& st,
                                               int row, int cb, const uint32_t (&r)[32]) {
    const int nvalid = sh.N - cb;  // columns >= N are padding
    const int yl = st.y - cb;
    if (static_cast<unsigned>(yl) < 32u) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j == yl) st.zy = __uint_as_float(r[j]);
    }
    float cm;
    if (nvalid >= 32) {
      float m4[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float* v = reinterpret_cast<const float*>(r) + 8 * q;
        m4[q] = fmax3(fmax3(v[0], v[1], v[2]), fmax3(v[3], v[4], v[5]), fmaxf(v[6], v[7]));
      }
      cm = fmax3(m4[0], m4[1], fmaxf(m4[2], m4[3]));
    } else {
      cm = -INFINITY;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nvalid) cm = fmaxf(cm, __uint_as_float(r[j]));
    }
    if (cm > st.m) {
      const float mq = fminf(ceilf(cm * kOffScale) * (1.f / kOffScale), kMaxOff);
      const float f = ex2_ftz((st.m - mq) * kLog2e);
      st.s *= f;
      st.t *= f;
      st.m = mq;
      // exponent capped: rows that far above their anchor are rewritten by
      // the fixup (combine_row), the cap only keeps q finite meanwhile
      if constexpr (kFactored) st.f = ex2_ftz(fminf(fmaf(mq, kLog2e, -st.a), 126.f));
    }
    const float mb = st.m * kLog2e;
    const bool keep = p.zout != nullptr && row < sh.M;
    uint16_t* dst = keep ? static_cast<uint16_t*>(p.zout) + static_cast<long long>(row) * p.ldz + cb
                         : nullptr;
    float s0 = 0.f, s1 = 0.f, t0 = 0.f, t1 = 0.f;
    if (nvalid >= 32) {
#if TL_EPI_F32X2
      // even / odd columns as the two lanes of packed fp32 pairs (FFMA2 /
      // FADD2: same bits as the scalar split accumulators, half the issues)
      uint32_t hq[16];
      const float2 l2 = make_float2(kLog2e, kLog2e), nmb = make_float2(-mb, -mb);
      float2 s2 = make_float2(0.f, 0.f), t2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const float2 v = make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1]));
        const float2 u = ffma2(v, l2, nmb);
        const float2 e = make_float2(ex2_ftz(u.x), ex2_ftz(u.y));
        s2 = fadd2(s2, e);
        t2 = ffma2(e, v, t2);
        if constexpr (kFactored) {
          const float2 q = fmul2(e, make_float2(st.f, st.f));
          hq[j / 2] = pack_bf16x2(q.x, q.y);
        } else {
          hq[j / 2] = pack_f16x2_sat(u.x, u.y);
        }
      }
      s0 = s2.x;
      s1 = s2.y;
      t0 = t2.x;
      t1 = t2.y;
#else
      uint32_t hq[16];
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const float v0 = __uint_as_float(r[j]), v1 = __uint_as_float(r[j + 1]);
        const float u0 = fmaf(v0, kLog2e, -mb), u1 = fmaf(v1, kLog2e, -mb);
        const float e0 = ex2_ftz(u0), e1 = ex2_ftz(u1);
        s0 += e0;
        s1 += e1;
        t0 = fmaf(e0, v0, t0);
        t1 = fmaf(e1, v1, t1);
        if constexpr (kFactored) hq[j / 2] = pack_bf16x2(e0 * st.f, e1 * st.f);
        else hq[j / 2] = pack_f16x2_sat(u0, u1);
      }
#endif
      if (keep) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          st_v4_hint(dst + 8 * q, make_uint4(hq[4 * q], hq[4 * q + 1], hq[4 * q + 2], hq[4 * q + 3]),
                     st.zpol);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float v = __uint_as_float(r[j]);
        const float u = fmaf(v, kLog2e, -mb);
        const float e = j < nvalid ? ex2_ftz(u) : 0.f;
        s0 += e;
        t0 = fmaf(e, v, t0);
        if (keep && j < nvalid)
          dst[j] = static_cast<unsigned short>(
              (kFactored ? pack_bf16x2(e * st.f, 0.f) : pack_f16x2_sat(u, 0.f)) & 0xFFFFu);
      }
    }
    st.s += s0 + s1;
    st.t += t0 + t1;
    if (!kFactored && p.zout) {  // this slice's offset m into the tile's 8-slot shift register
      const uint64_t m16 =
          static_cast<uint16_t>(static_cast<int16_t>(fmaxf(st.m, -kMaxOff) * kOffScale));
      st.olo = (st.olo >> 16) | (st.ohi << 48);
      st.ohi = (st.ohi >> 16) | (m16 << 48);
    }
  }
  // TMEM loads are double-buffered: slice c+1 is in flight while slice c is
  // reduced (tcgen05.wait::ld waits for all outstanding loads).
  template <int BN>
  __device__ static void tile(const Params& p, const GemmShape& sh, State& st, int row, int col0,
                              uint32_t taddr) {
    static_assert(BN == 256, "slice offsets are stored 8 (16 bytes) per 256-column tile");
    uint32_t ra[32], rb[32];
    tmem_ld32(taddr, ra);
    tmem_ld_wait_regs(ra);
#pragma unroll 1
    for (int c = 0; c < BN; c += 64) {
      tmem_ld32(taddr + c + 32, rb);
      slice(p, sh, st, row, col0 + c, ra);
      tmem_ld_wait_regs(rb);
      const bool more = c + 64 < BN;
      if (more) tmem_ld32(taddr + c + 64, ra);
      slice(p, sh, st, row, col0 + c + 32, rb);
      if (more) tmem_ld_wait_regs(ra);
    }
    if (!kFactored && p.zout && row < sh.M)
      st_v4_hint(p.zoff + static_cast<long long>(row) * p.ldo + col0 / 32,
                 make_uint4(static_cast<uint32_t>(st.olo), static_cast<uint32_t>(st.olo >> 32),
                            static_cast<uint32_t>(st.ohi), static_cast<uint32_t>(st.ohi >> 32)),
                 st.zpol);
  }
  // Publish this strip's row stats; the CTA that finishes the LAST strip of a
  // 128-row block (stream-K style fixup, counter per block) merges all strips
  // and runs the GRPO surrogate for those rows inside this epilogue.
  __device__ static void end_unit(const Params& p, const GemmShape& sh, State& st, int row,
                                  const UnitCoord& uc) {
    if (row < sh.M)
      p.part[static_cast<long long>(uc.strip_idx) * p.rows + row] = make_float4(st.m, st.s, st.t, st.zy);
    if (sh.n_strips == 1) {  // no other strip: merge straight away (own writes)
      if (row < sh.M) combine_row(p.ca, row);
      return;
    }
    __shared__ int s_last;
    __threadfence();                                                   // release partials
    asm volatile("bar.sync 1, %0;" ::"n"(4 * 32) : "memory");         // 4 epilogue warps
    if ((threadIdx.x & 127) == 0) {
      const int blk = row / kBM;
      const int prev = atomicAdd(p.tile_ctr + blk, 1);
      s_last = prev == sh.n_strips - 1;
      if (s_last) p.tile_ctr[blk] = 0;  // re-arm for the next launch
    }
    asm volatile("bar.sync 1, %0;" ::"n"(4 * 32) : "memory");
    if (s_last) {
      __threadfence();  // acquire the other strips' partials
      if (row < sh.M) combine_row(p.ca, row);
    }
  }
};
using EpiLseStats = EpiLseStatsT<false>;

// dS = dLoss/dz (bf16) from recomputed logits.
struct EpiDSoftmax {
  static constexpr bool kSplitTail = false;
  struct Params {
    const int32_t* targets;
    const float* lse;
    const float* g;   // dLoss/dlogp
    const float* c;   // dLoss/dentropy
    const float* ez;  // E_p[z]
    __nv_bfloat16_raw* ds;
    long long ldd;
  };
  struct State {
    float lse2, g, c, ez;
    int y;
  };
  __device__ static void begin_unit(const Params& p, const GemmShape& sh, State& st, int row,
                                    const UnitCoord&) {
    if (row < sh.M) {
      st.lse2 = p.lse[row] * kLog2e;
      st.g = p.g[row];
      st.c = p.c[row];
      st.ez = p.ez[row];
      st.y = p.targets[row];
    } else {
      st.lse2 = 0.f;
      st.g = st.c = st.ez = 0.f;
      st.y = -1;
    }
  }
  template <int BN>
  __device__ static void tile(const Params& p, const GemmShape& sh, State& st, int row, int col0,
                              uint32_t taddr) {
    const bool row_ok = row < sh.M;
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t r[32];
      tmem_ld32(taddr + c, r);
      tmem_ld_wait();
      if (!row_ok) continue;
      const int cb = col0 + c;
      float d[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float z = __uint_as_float(r[j]);
        const float pr = exp2f(fmaf(z, kLog2e, -st.lse2));
        float v = -st.g * pr - st.c * pr * (z - st.ez);
        if (cb + j == st.y) v += st.g;
        d[j] = v;
      }
      __nv_bfloat16_raw* dst = p.ds + static_cast<long long>(row) * p.ldd + cb;
      if (cb + 32 <= sh.N) {
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          uint4 v;
          v.x = pack_bf16x2(d[j + 0], d[j + 1]);
          v.y = pack_bf16x2(d[j + 2], d[j + 3]);
          v.z = pack_bf16x2(d[j + 4], d[j + 5]);
          v.w = pack_bf16x2(d[j + 6], d[j + 7]);
          *reinterpret_cast<uint4*>(dst + j) = v;
        }
      } else {
        for (int j = 0; j < 32; ++j)
          if (cb + j < sh.N) dst[j].x = static_cast<unsigned short>(pack_bf16x2(d[j], 0.f) & 0xFFFFu);
      }
    }
  }
  __device__ static void end_unit(const Params&, const GemmShape&, State&, int, const UnitCoord&) {}
};

}  // namespace
}  // namespace tl
