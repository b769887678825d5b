// K4/K5 — fused LM-head log-prob / entropy with the GRPO surrogate epilogue,
// and its backward, on tcgen05 (gemm_sm100.cuh).
//
// No reference implementation: the contract is PolicyAction.token_logprobs
// (rollout/policy.py:25-28) consumed as TokenRecord.logp_new (rl/loss.py:30).
// Per chunk of C action rows (act_idx[c0 .. c0+C)):
//   gather      h_c[C, H]  <- hidden[act_idx[c0 + r]]                 (HBM copy)
//   fwd GEMM    z = h_c W^T tile by tile (128 x 256, K = H) in TMEM; the
//               epilogue keeps, per row and per vocab strip, the online
//               log-sum-exp state (max, sum e^(z-max), sum e^(z-max) z) and
//               the target logit -> partials [n_strips, C]; the CTA that
//               finishes the last strip of a 128-row block merges the strips
//               (lse, logp = z_y - lse, entropy) and runs the GRPO surrogate
//               (grpo_token.cuh) on logp_new in the same epilogue: per-token
//               term / k3 / flags and dLoss/dlogp, dLoss/dent.  In store mode
//               the epilogue also writes the chunk's logits as fp16
//               u = (z - m) log2e <= 0 with an int16 offset m per 32 columns
//               (lmhead_epilogue.cuh) — or, factored (entropy_coef == 0),
//               bf16 q = e^(z - m0) with a per-row anchor m0 fixed by the
//               gather, and the merge turns dS into alpha_r * q.
//   dsoftmax    (store mode) fp16 u -> bf16 dS in place, HBM-bound
//   rescale     (factored) h_c *= alpha (dW's B operand); rows outside the
//               anchor's range rewritten on CUDA cores (never in practice)
//   recompute   (recompute mode) same GEMM, epilogue writes dS (bf16, [C, V])
//               dS = g (onehot(y) - p) - c p (z - E_p z),  p = e^(z - lse)
//   dH GEMM     dhidden[act_idx] = dS W          (A K-major, B = W MN-major;
//                                                  factored: alpha (q W))
//   dW GEMM     dW (+)= dS^T h_c                 (A, B MN-major; fp32 store,
//               then red.add accumulation across chunks / micro-batches)
// after all chunks: deterministic trajectory -> group -> batch reductions.
// Epilogues live in lmhead_epilogue.cuh; this file holds the TMA maps, the
// launch wrapper, the small kernels and the host drivers (serial or
// pipelined chunk schedule).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <mutex>

#include "gemm_sm100.cuh"
#include "grpo_token.cuh"
#include "loss_internal.cuh"
#include "tl_common.cuh"

namespace tl {
namespace {

constexpr int kBN = 256;
constexpr int kCG = 2;  // 2-CTA (cta_group::2) tiles of 256 x 256
// dH / dW (long K, light epilogue): 256 x 512 pair tiles (two N=256 UMMAs per
// k-step, TMEM single-buffered) halve the dS re-reads across N tiles.
constexpr int kBNWide = 512;
#ifndef TL_STAGES256
#define TL_STAGES256 7
#endif
constexpr int kStages = TL_STAGES256;  // ring depth of the 256-wide tiles (32 KB stages;
                                       // 7 = 224 KB, -0.2 % vs 6 at C2, gpu_r48)
constexpr int kStripsFwd = 6;  // even: a wave covers 2 strips of one M group
constexpr int kGroupM = 16;

// ------------------------------------------------------------------ TMA maps --
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// bf16 matrix stored row-major as [outer, inner] with row stride ld elements;
// box = {box_inner, box_outer}, SWIZZLE_128B (box_inner * 2 == 128 bytes).
int make_map(CUtensorMap* m, const void* ptr, long long inner, long long outer, long long ld,
             int box_inner, int box_outer) {
  EncodeFn enc = get_encode();
  TL_REQUIRE(enc, TL_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  TL_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & 15) == 0, TL_ERR_INVALID_ARG,
             "TMA base pointer must be 16-byte aligned");
  TL_REQUIRE((ld * 2) % 16 == 0, TL_ERR_INVALID_ARG, "row stride must be a multiple of 16 bytes");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  TL_REQUIRE(r == CUDA_SUCCESS, TL_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return TL_OK;
}

// Operand map: K-major [rows, K] -> box {64, box_rows}; MN-major [K, MN] -> box {64, 64}.
int make_operand_map(CUtensorMap* m, const void* ptr, bool mn_major, long long mn, long long k,
                     long long ld, int box_rows) {
  if (!mn_major) return make_map(m, ptr, k, mn, ld, 64, box_rows);
  return make_map(m, ptr, mn, k, ld, 64, 64);
}

// Operand maps for a GEMM run with CTA group `cg`: A tiles are 128 rows per
// CTA, B tiles BN/cg rows per CTA (K-major); MN-major boxes are 64 x 64.
int make_ab_maps(CUtensorMap* ma, CUtensorMap* mb, const void* A, bool a_mn, long long M,
                 long long lda, const void* B, bool b_mn, long long N, long long ldb, long long K,
                 int cg) {
  if (int e = make_operand_map(ma, A, a_mn, M, K, lda, kBM)) return e;
  return make_operand_map(mb, B, b_mn, N, K, ldb, kBN / cg);
}

#if TL_GEMM_STATS
unsigned long long* h_stats_base = nullptr;  // [PROF categories][160 CTAs][8]
#endif

// split-K tail slice buffer: tile halves of 128 rows x 512 fp32 columns
constexpr int kTailSlots = 160;
constexpr int kMaxDevices = 64;

template <int CG, bool A_MN, bool B_MN, class Epi, int BN = kBN>
int launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, const GemmShape& s,
                const typename Epi::Params& ep, cudaStream_t st, int prof_cat = PROF_GEMM_OTHER,
                int reserve_sms = 0) {
  ProfScope prof(prof_cat, st);
  constexpr int kSt = BN <= 256 ? kStages : 4;  // 48 KB stages at BN = 512
  using Smem = GemmSmem<BN, kSt, CG>;
  auto kern = gemm_sm100_kernel<BN, kSt, CG, A_MN, B_MN, Epi>;
  cudaLaunchConfig_t lc{};
  lc.blockDim = dim3(kGemmThreads);
  lc.dynamicSmemBytes = Smem::kBytes;
  lc.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  // Persistent grid: never more CTA groups than can be co-resident (the
  // wave lockstep and the static unit schedule assume every group is live).
  // The smem attribute and the occupancy are per device: cached per device
  // id (a process may drive several GPUs, or GPUs with other SM counts).
  static std::mutex mu;
  static int cached[kMaxDevices] = {};
  int dev = 0;
  TL_CUDA_TRY(cudaGetDevice(&dev));
  TL_REQUIRE(dev >= 0 && dev < kMaxDevices, TL_ERR_UNSUPPORTED, "device %d", dev);
  int max_groups;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (cached[dev] == 0) {
      TL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       Smem::kBytes));
      lc.gridDim = dim3(num_sms());
      int active = 0;
      if (cudaOccupancyMaxActiveClusters(&active, kern, &lc) != cudaSuccess || active <= 0) {
        cudaGetLastError();
        active = num_sms() / CG;
      }
      cached[dev] = active < num_sms() / CG ? active : num_sms() / CG;
    }
    max_groups = cached[dev];
  }
  if (s.n_units == 0 || s.k_blocks == 0) return TL_OK;
  TL_REQUIRE(s.cg == CG, TL_ERR_INVALID_ARG, "shape built for cg=%d, kernel cg=%d", s.cg, CG);
  // reserve_sms: leave whole CTA groups free for a concurrent kernel (a
  // collective on another stream, tl_grpo_lmhead_step_overlap)
  if (reserve_sms > 0) max_groups = max(1, max_groups - (reserve_sms + CG - 1) / CG);
  const int groups = s.n_units < max_groups ? s.n_units : max_groups;
  lc.gridDim = dim3(groups * CG);
  GemmShape sh = s;
  if constexpr (Epi::kSplitTail) {
    // split-K tail: cut the partial last wave's units into K-slices that fill
    // the idle pairs (slice buffer holds one wave: kTailSlots tile halves)
    const int rem = sh.n_units % groups;
    if (sh.tail_part && sh.strip == 1 && rem > 0 && sh.n_units > groups) {
      int split = groups / rem;
      split = split < sh.k_blocks ? split : sh.k_blocks;
      if (rem * split * CG > kTailSlots) split = kTailSlots / (rem * CG);
      if (split >= 2) {
        sh.tail_begin = sh.n_units - rem;
        sh.tail_split = split;
        TL_CUDA_TRY(cudaMemsetAsync(sh.tail_ctr, 0, rem * CG * sizeof(int), st));
      }
    }
  }
#if TL_GEMM_STATS
  if (h_stats_base) {  // stream-ordered: this launch's counters go to its category's block
    unsigned long long* p = h_stats_base + static_cast<size_t>(prof_cat) * 160 * 8;
    TL_CUDA_TRY(cudaMemcpyToSymbolAsync(g_gemm_stats, &p, sizeof(p), 0, cudaMemcpyHostToDevice, st));
  }
#endif
  TL_CUDA_TRY(cudaLaunchKernelEx(&lc, kern, ma, mb, sh, ep));
  count_launch();
  return TL_OK;
}

}  // namespace
}  // namespace tl

#include "lmhead_epilogue.cuh"

namespace tl {
namespace {

// ----------------------------------------------------------- small kernels --
__global__ void gather_rows_kernel(const uint4* __restrict__ src, const int32_t* __restrict__ idx,
                                   long long n_rows, int row_vec, uint4* __restrict__ dst) {
  const long long total = n_rows * row_vec;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / row_vec;
    const int c = static_cast<int>(i - r * row_vec);
    const long long s = idx ? idx[r] : r;
    dst[i] = __ldg(src + s * row_vec + c);
  }
}

__device__ __forceinline__ float dot8_bf16(uint4 a, uint4 b) {
  const uint32_t x[4] = {a.x, a.y, a.z, a.w}, w[4] = {b.x, b.y, b.z, b.w};
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    s = fmaf(__uint_as_float(x[k] << 16), __uint_as_float(w[k] << 16), s);
    s = fmaf(__uint_as_float(x[k] & 0xFFFF0000u), __uint_as_float(w[k] & 0xFFFF0000u), s);
  }
  return s;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Factored store: gather the chunk's action rows (h_c[r] = hidden[idx[r]],
// y[r] = ids[idx[r]]) and fix each row's anchor m0 before the forward —
// one warp per row also reads W[y] and takes the fp32 dot product
// z~_y = h . W[y]; m0 = z~_y + clamp(-logp_old, 0, 40) (20 if logp_old is
// NaN), i.e. m0 ~ lse when the policy is near the one that sampled the token
// (lmhead_epilogue.cuh: kQdMin / kQdMax).  z~_y only places the anchor; any
// value works as long as the row's forward and merge use the same one.
__global__ void __launch_bounds__(256)
    gather_anchor_kernel(const uint4* __restrict__ hidden, const uint4* __restrict__ weight,
                         const int32_t* __restrict__ idx, const int32_t* __restrict__ ids,
                         const float* __restrict__ logp_old, int rows, int row_vec, int V,
                         uint4* __restrict__ h_c, int32_t* __restrict__ y_out,
                         float* __restrict__ anchor) {
  const int lane = threadIdx.x & 31;
  const int n_warps = gridDim.x * (blockDim.x / 32);
  for (int r = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; r < rows; r += n_warps) {
    const long long p = idx[r];
    const int y = ids[p];
    const bool y_ok = static_cast<unsigned>(y) < static_cast<unsigned>(V);
    const uint4* src = hidden + p * row_vec;
    const uint4* wy = weight + static_cast<long long>(y_ok ? y : 0) * row_vec;
    uint4* dst = h_c + static_cast<long long>(r) * row_vec;
    float acc = 0.f;
#pragma unroll 2
    for (int c = lane; c < row_vec; c += 32) {
      const uint4 h = __ldg(src + c);
      dst[c] = h;
      if (y_ok) acc += dot8_bf16(h, __ldg(wy + c));
    }
    acc = warp_sum(acc);
    if (lane == 0) {
      y_out[r] = y;
      const float lo = logp_old[p];
      anchor[r] = acc + (lo == lo ? fminf(fmaxf(-lo, 0.f), 40.f) : 20.f);
    }
  }
}

// Factored store, rows combine_row listed (lse - m0 outside [kQdMin,
// kQdMax] with a nonzero gradient; none in practice): recompute the row's
// logits on CUDA cores (fp32 dot products of the bf16 rows, one warp per
// vocab entry) and rewrite the row with the anchor m0 = lse: q = p,
// alpha = -g, A[y] = expm1(logp_y).  Work item = (listed row, 1,024-column
// block); the list is read on the device, so an empty list costs one launch.
__global__ void __launch_bounds__(256)
    fixup_rows_kernel(const int* __restrict__ flagged, const uint4* __restrict__ h_c,
                      const uint4* __restrict__ weight, int row_vec, int V,
                      const int32_t* __restrict__ y, const float* __restrict__ lse,
                      const float* __restrict__ g, float* __restrict__ alpha,
                      __nv_bfloat16_raw* __restrict__ q, long long ldq) {
  const int n = flagged[0];
  if (n == 0) return;
  constexpr int kCols = 1024;
  const int nb = (V + kCols - 1) / kCols;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  for (long long it = blockIdx.x; it < static_cast<long long>(n) * nb; it += gridDim.x) {
    const int r = flagged[1 + it / nb];
    const int v0 = static_cast<int>(it % nb) * kCols;
    const int v1 = min(v0 + kCols, V);
    const uint4* h = h_c + static_cast<long long>(r) * row_vec;
    const float l = lse[r];
    const int yr = y[r];
    if (v0 == 0 && threadIdx.x == 0) alpha[r] = -g[r];
    for (int v = v0 + warp; v < v1; v += blockDim.x / 32) {
      const uint4* w = weight + static_cast<long long>(v) * row_vec;
      float acc = 0.f;
      for (int c = lane; c < row_vec; c += 32) acc += dot8_bf16(__ldg(h + c), __ldg(w + c));
      acc = warp_sum(acc);
      if (lane == 0) store_bf16(q + static_cast<long long>(r) * ldq + v, v == yr ? expm1f(acc - l) : expf(acc - l));
    }
  }
}

// Factored store: dW's B operand h_c[r] *= alpha_r (bf16, in place).
__global__ void scale_rows_kernel(uint4* __restrict__ h_c, const float* __restrict__ alpha,
                                  long long rows, int row_vec) {
  const long long total = rows * row_vec;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const float a = alpha[i / row_vec];
    uint4 v = h_c[i];
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k)
      w[k] = pack_bf16x2(__uint_as_float(w[k] << 16) * a, __uint_as_float(w[k] & 0xFFFF0000u) * a);
    h_c[i] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

__global__ void gather_i32_kernel(const int32_t* __restrict__ src, const int32_t* __restrict__ idx,
                                  long long n, int32_t* __restrict__ dst) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[idx ? idx[i] : i];
}


// In place: fp16 u = (z - m) log2e (written by the forward epilogue, m =
// the int16 offset of the 32-column slice, units of 1/128) -> bf16
// dS = g (onehot(y) - p) - c p (z - E_p z).  With z = m + u ln2:
//   p = 2^(u + K),  K = m log2e - lse log2e              (one FADD + one SFU op)
//   dS = p (A' + B' u),  A' = c E_p z - g - c m,  B' = -c ln2   (one FFMA, one FMUL)
// plus g at the target column (the one word that holds it).  K and A' are
// per slice: one thread owns a whole slice (four 16-byte words), so the
// offset is loaded and turned into (K, A') once per 32 logits.
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ uint4 dsoftmax8(uint4 q, int col0, float K, float A, float B, int yy,
                                           float gg) {
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
  float d[8];
#if TL_EPI_F32X2
  const float2 K2 = make_float2(K, K), A2 = make_float2(A, A), B2 = make_float2(B, B);
#pragma unroll
  for (int k = 0; k < 4; ++k) {  // packed fp32 pairs: bitwise the scalar math
    const float2 u = __half22float2(*reinterpret_cast<const __half2*>(&w[k]));
    const float2 x = fadd2(u, K2);
    const float2 pd = fmul2(make_float2(ex2_ftz(x.x), ex2_ftz(x.y)), ffma2(B2, u, A2));
    d[2 * k] = pd.x;
    d[2 * k + 1] = pd.y;
  }
#else
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 u = __half22float2(*reinterpret_cast<const __half2*>(&w[k]));
    d[2 * k] = ex2_ftz(u.x + K) * fmaf(B, u.x, A);
    d[2 * k + 1] = ex2_ftz(u.y + K) * fmaf(B, u.y, A);
  }
#endif
  const int yl = yy - col0;
  if (static_cast<unsigned>(yl) < 8u) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j == yl) d[j] += gg;
  }
  return make_uint4(pack_bf16x2(d[0], d[1]), pack_bf16x2(d[2], d[3]), pack_bf16x2(d[4], d[5]),
                    pack_bf16x2(d[6], d[7]));
}

// Rows are grid-strided: one CTA per row when launched alone, or a small
// persistent grid when it runs beside the next chunk's forward GEMM
// (pipelined mode) and should trickle at low HBM intensity.  A thread
// streams one 32-logit slice (64 bytes: four 16-byte words in flight, read
// through the non-coherent path so the warp's interleaved 16-byte requests
// share L1 sectors) per step; the pass is HBM-bound and, at the power-capped
// SM clock of the step, kept short in instructions.
__global__ void __launch_bounds__(256)
    dsoftmax_inplace_kernel(uint4* __restrict__ buf, long long ld_vec,
                            const int16_t* __restrict__ zoff, long long ldo, int V, int rows,
                            const int32_t* __restrict__ y, const float* __restrict__ lse,
                            const float* __restrict__ g, const float* __restrict__ c,
                            const float* __restrict__ ez) {
  const int nvec = (V + 7) / 8;
  const int nsl = (nvec + 3) / 4;
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const float l2 = lse[r] * kLog2e, gg = g[r], cc = c[r];
    const float A = cc * ez[r] - gg, B = -cc, Bu = -cc * kLn2;
    const int yy = y[r];
    uint4* row = buf + static_cast<long long>(r) * ld_vec;
    const int16_t* off = zoff + static_cast<long long>(r) * ldo;
    for (int sl = threadIdx.x; sl < nsl; sl += blockDim.x) {
      const float m = static_cast<float>(__ldg(off + sl)) * (1.f / 128.f);
      const float K = fmaf(m, kLog2e, -l2), Aw = fmaf(B, m, A);
      const int v0 = sl * 4;
      if (v0 + 4 <= nvec) {
        uint4 q[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) q[j] = __ldg(row + v0 + j);
#pragma unroll
        for (int j = 0; j < 4; ++j) row[v0 + j] = dsoftmax8(q[j], (v0 + j) * 8, K, Aw, Bu, yy, gg);
      } else {
        for (int v = v0; v < nvec; ++v) row[v] = dsoftmax8(row[v], v * 8, K, Aw, Bu, yy, gg);
      }
    }
  }
}

__global__ void zero_obs_rows_kernel(const uint8_t* __restrict__ mask, long long n_tokens,
                                     int row_vec, uint4* __restrict__ dh) {
  const long long total = n_tokens * row_vec;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long p = i / row_vec;
    if (!mask[p]) dh[i] = make_uint4(0, 0, 0, 0);
  }
}

__global__ void fill_f32_kernel(float* __restrict__ x, long long n, float v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    x[i] = v;
}

int grid_for(long long n, int block) {
  long long g = (n + block - 1) / block;
  const long long cap = static_cast<long long>(num_sms()) * 16;
  return static_cast<int>(g < 1 ? 1 : (g > cap ? cap : g));
}

// --------------------------------------------------------------- workspace --
struct ChunkWs {
  uint16_t* h;      // [C, H]
  float4* part;     // [kStripsFwd, C]
  int32_t* y;       // [C]
  float* lse;       // [C]
  float* g;         // [C]
  float* c;         // [C]
  float* ez;        // [C]
  float* logp;      // [C]
  float* ent;       // [C]
  uint16_t* ds;     // [C, Vld]  fp16 u = (z - m) log2e, then bf16 dS in place
  int16_t* zoff;    // [C, ldo]  int16 slice offsets m of the fp16 u (store mode)
  float* anc;       // [C]  factored store: anchor m0 per row
  float* alpha;     // [C]  factored store: dS row scale
  int* flagged;     // [1 + C] factored store: rows for fixup_rows_kernel
  // step-level
  float* term;      // [T]  (written at action positions only)
  float* k3o;       // [T]
  uint8_t* flags;   // [T]
  ReduceWs red;     // trajectory / group / report reductions
  int* sync;        // [3 * kSyncWaves] wave-lockstep counters (fwd / dH / dW)
  float* tail_part; // [kTailSlots][128][512] split-K tail slices of the dW GEMM
  int* tail_ctr;    // [kTailSlots] slice arrival counters
};

constexpr int kSyncWaves = 4096;

// Schedule parameters, measured at C2 on power-capped B200s (
// the A/B runs that chose them are in the git history of tools/experiments).
namespace tune {
// L2 eviction priority of TMA operand loads / stores (make_policy kinds)
constexpr int kNormal = 0, kEvictFirst = 1, kEvictLast = 2;
// forward: h_c rows reused by every W tile of the strip (evict_last), W tiles
// consumed within one lockstep window (evict_first): fwd -4.9 % (gpu_r51)
constexpr int kFwdPolA = kEvictLast, kFwdPolB = kEvictFirst;
constexpr int kFwdZStorePolicy = kEvictFirst;  // fp16 u stores: read once, by the dS pass
// forward lockstep: steps of 4 tiles, window 1, per (M group, strip): 1 -> 2
// -> 4-tile steps -0.5 / -0.4 %, 4 beats 8 by 0.3 % (gpu_r25, r30-r32, r57)
constexpr int kFwdSyncTiles = 4, kFwdSyncWindow = 1, kFwdSyncSplit = 1;
// dH / dW: dS streams (evict_first); W (dH) and h_c (dW) are re-read by every
// wave (evict_last): dH -1.1 %, dW -2.8 % (gpu_r50)
constexpr int kDhPolA = kEvictFirst, kDhPolB = kEvictLast;
constexpr int kDwPolA = kEvictFirst, kDwPolB = kEvictLast;
// dH / dW lockstep: 64-k-block steps, window 1 (without: step +7.8 %, gpu_r21)
constexpr int kBwdSyncBlocks = 64, kBwdSyncWindow = 1;
// pipelined mode: CTAs per SM of the dS pass running beside the forward
constexpr int kDsOverlapCtasPerSm = 2;
}  // namespace tune

// Attach wave-lockstep counters to a shape (see GemmShape::sync_ctr) and
// turn on the serpentine K order.
GemmShape with_sync(GemmShape s, int* ctr, int every, int window, int split = 0,
                    int reserve_sms = 0) {
  s.serpentine = 1;
  const int n_pairs = max(1, num_sms() / s.cg - (reserve_sms + s.cg - 1) / s.cg);
  const int waves = (s.n_units + n_pairs - 1) / n_pairs;
  if (ctr && waves * (split ? 8 : 1) <= kSyncWaves && every > 0) {
    s.sync_ctr = ctr;
    s.sync_every = every;
    s.sync_window = window;
    s.sync_split = split;
  }
  return s;
}

long long vld_of(int vocab) { return (vocab + 7) / 8 * 8; }
// int16 slice offsets per row: 8 per 256-column forward tile (16-byte stores)
long long ldo_of(int vocab) { return (vocab + kBN - 1) / kBN * 8; }

// Chunk buffers (h_c, partials, per-row stats, dS, lockstep counters) once,
// or twice when `second` is given (pipelined mode); step-level buffers once.
void carve_chunk(Workspace& w, ChunkWs& c, int C, int H, int V, bool with_bwd) {
  c.h = w.take<uint16_t>(static_cast<size_t>(C) * H);
  c.part = w.take<float4>(static_cast<size_t>(kStripsFwd) * C);
  c.y = w.take<int32_t>(C);
  c.lse = w.take<float>(C);
  c.g = w.take<float>(C);
  c.c = w.take<float>(C);
  c.ez = w.take<float>(C);
  c.logp = w.take<float>(C);
  c.ent = w.take<float>(C);
  c.ds = with_bwd ? w.take<uint16_t>(static_cast<size_t>(C) * vld_of(V)) : nullptr;
  c.zoff = with_bwd ? w.take<int16_t>(static_cast<size_t>(C) * ldo_of(V)) : nullptr;
  c.anc = with_bwd ? w.take<float>(C) : nullptr;
  c.alpha = with_bwd ? w.take<float>(C) : nullptr;
  c.flagged = with_bwd ? w.take<int>(C + 1) : nullptr;
  c.sync = w.take<int>(5 * kSyncWaves);
  if (with_bwd) {
    c.tail_part = w.take<float>(static_cast<size_t>(kTailSlots) * kBM * kBNWide);
    c.tail_ctr = w.take<int>(kTailSlots);
  }
}

ChunkWs carve(Workspace& w, int C, int H, int V, long long T, int B, int G, bool with_bwd,
              ChunkWs* second = nullptr) {
  ChunkWs c{};
  carve_chunk(w, c, C, H, V, with_bwd);
  if (second) carve_chunk(w, *second, C, H, V, with_bwd);
  c.term = w.take<float>(T);
  c.k3o = w.take<float>(T);
  c.flags = w.take<uint8_t>(T);
  c.red = carve_reduce(w, T, B, G);
  if (second) {
    second->term = c.term;
    second->k3o = c.k3o;
    second->flags = c.flags;
    second->red = c.red;
  }
  return c;
}

// A side stream + two events for one pipelined step (created per call so
// concurrent callers never share them; destroyed asynchronously).
struct StreamPair {
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fwd = nullptr, ev_ds = nullptr;
  int err = TL_OK;
  StreamPair() {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, lo) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_fwd, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_ds, cudaEventDisableTiming) != cudaSuccess)
      err = TL_ERR_CUDA;
  }
  ~StreamPair() {
    if (ev_fwd) cudaEventDestroy(ev_fwd);
    if (ev_ds) cudaEventDestroy(ev_ds);
    if (side) cudaStreamDestroy(side);
  }
};

// Forward LM-head GEMM shape: A-stationary strips.  A wave of n_pairs units
// is 2 strips x (n_pairs / 2) M-tiles, so the wave's h_c rows (37 x 256 x H
// bf16 = 67 MB at C2) stay in L2 (evict_last) across the strip while every
// W tile is fetched once per wave and shared by the n_pairs / 2 pairs of its
// strip, kept close by the wave lockstep: sync steps of four tiles, window
// 1 (a producer may not start step s before every CTA of its strip group has
// issued step s-1).  Measured at C2 (tools/experiments/gpu_r17, r25, r30-r32,
// r57): one-tile window 2 -> 1 cut the forward's DRAM reads 33 -> 14 GB per
// chunk (before serpentine K); per-strip instead of whole-wave groups -0.5 %;
// 1 -> 2 -> 4-tile steps -0.5 / -0.4 %; with W tiles evict_first the
// forward depends on the lockstep more (none: +10.6 %) and 4 beats 8 by 0.3 %.
GemmShape fwd_shape(int rows, int V, int H, int* sync = nullptr) {
  const int n_tiles = (V + kBN - 1) / kBN;
  const int strip = (n_tiles + kStripsFwd - 1) / kStripsFwd;
  const int group_m = num_sms() / kCG / 2;  // a wave = 2 strips x (pairs / 2) M tiles
  GemmShape s = make_shape(rows, V, H, kBN, strip, group_m, kCG, tune::kFwdPolA, tune::kFwdPolB);
  // per-strip lockstep: a strip's pairs (sharing its W tiles) wait on each
  // other only, not on the other strip of the wave
  s = with_sync(s, sync, tune::kFwdSyncTiles * s.k_blocks, tune::kFwdSyncWindow,
                tune::kFwdSyncSplit);
  // K order by vocab tile: a row's logits (and logp / entropy / dS) are
  // bitwise the same whatever chunk, M tile or rank it is processed in
  s.serpentine = 2;
  return s;
}

// z = h_c W^T with the online-LSE epilogue, then merge strips.  zout: also
// keep the chunk's logits for the backward (store mode): fp16 u with int16
// offsets, or (factored) bf16 q against the anchors c.anc.
int lmhead_forward_chunk(const ChunkWs& c, const uint16_t* weight, int rows, int H, int V,
                         CombineArgs ca, cudaStream_t st, void* zout = nullptr,
                         long long ldz = 0, int16_t* zoff = nullptr, bool factored = false) {
  CUtensorMap ma, mb;
  if (int e = make_ab_maps(&ma, &mb, c.h, false, rows, H, weight, false, V, H, H, kCG)) return e;
  // fresh wave-lockstep counters for this chunk's GEMMs (fwd / dS / dH / dW)
  // and the per-128-row strip counters of the fused merge + surrogate
  TL_CUDA_TRY(cudaMemsetAsync(c.sync, 0, 5 * kSyncWaves * sizeof(int), st));
  TL_REQUIRE((rows + kBM - 1) / kBM <= kSyncWaves, TL_ERR_UNSUPPORTED, "chunk_rows too large");
  const GemmShape s = fwd_shape(rows, V, H, c.sync);
  ca.part = c.part;
  ca.n_strips = s.n_strips;
  ca.rows = rows;
  if (factored) {
    TL_CUDA_TRY(cudaMemsetAsync(c.flagged, 0, sizeof(int), st));
    ca.anchor = c.anc;
    ca.y_row = c.y;
    ca.alpha_row = c.alpha;
    ca.qout = static_cast<__nv_bfloat16_raw*>(zout);
    ca.ldq = ldz;
    ca.flagged = c.flagged;
    EpiLseStatsT<true>::Params ep{c.y, c.part, rows, zout, ldz, nullptr, ldo_of(V),
                                  c.sync + 4 * kSyncWaves, ca, tune::kFwdZStorePolicy, c.anc};
    return launch_gemm<kCG, false, false, EpiLseStatsT<true>>(ma, mb, s, ep, st, PROF_GEMM_FWD);
  }
  EpiLseStats::Params ep{c.y, c.part, rows, zout, ldz, zoff, ldo_of(V), c.sync + 4 * kSyncWaves, ca,
                         tune::kFwdZStorePolicy};
  return launch_gemm<kCG, false, false, EpiLseStats>(ma, mb, s, ep, st, PROF_GEMM_FWD);
}

}  // namespace
}  // namespace tl

using namespace tl;

// Profiling builds only (not in the public header): point the GEMM stall
// counters at a device buffer of [grid * 8] u64 (NULL = off).
extern "C" int tl_debug_gemm_stats(void* buf) {
#if TL_GEMM_STATS
  h_stats_base = static_cast<unsigned long long*>(buf);
  return TL_OK;
#else
  (void)buf;
  return TL_ERR_UNSUPPORTED;
#endif
}

extern "C" size_t tl_lmhead_workspace_bytes(int32_t chunk_rows, int32_t hidden, int32_t vocab,
                                            int64_t n_tokens, int32_t n_traj, int32_t n_groups) {
  Workspace w{nullptr, 0};
  carve(w, chunk_rows, hidden, vocab, n_tokens, n_traj, n_groups, true);
  return w.used + 1024;
}

extern "C" size_t tl_lmhead_logprobs_workspace_bytes(int32_t chunk_rows, int32_t hidden,
                                                     int32_t vocab) {
  Workspace w{nullptr, 0};
  carve(w, chunk_rows, hidden, vocab, 0, 0, 0, false);
  return w.used + 1024;
}

extern "C" size_t tl_lmhead_step_workspace_bytes(int32_t chunk_rows, int32_t hidden,
                                                 int32_t vocab, int64_t n_tokens, int32_t n_traj,
                                                 int32_t n_groups, int32_t mode) {
  Workspace w{nullptr, 0};
  ChunkWs second{};
  carve(w, chunk_rows, hidden, vocab, n_tokens, n_traj, n_groups, true,
        (mode & 0xFF) == TL_LMHEAD_STORE_LOGITS_PIPELINED ? &second : nullptr);
  return w.used + 1024;
}

extern "C" int tl_gemm_bf16(const uint16_t* A, int32_t a_mn_major, int64_t lda, const uint16_t* B,
                            int32_t b_mn_major, int64_t ldb, int32_t M, int32_t N, int32_t K,
                            void* C, int32_t c_fp32, int64_t ldc, int32_t accumulate,
                            tl_stream_t stream) {
  TL_REQUIRE(M >= 0 && N >= 0 && K >= 0, TL_ERR_INVALID_ARG, "negative sizes");
  if (M == 0 || N == 0) return TL_OK;
  TL_REQUIRE(K > 0, TL_ERR_UNSUPPORTED, "K must be positive");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CUtensorMap ma, mb;
  if (int e = make_ab_maps(&ma, &mb, A, a_mn_major != 0, M, lda, B, b_mn_major != 0, N, ldb, K,
                           kCG))
    return e;
  const int sel = (a_mn_major ? 2 : 0) | (b_mn_major ? 1 : 0);
  if (c_fp32 && N >= 1024) {  // wide 256 x 512 pair tiles (as the dH / dW GEMMs)
    const GemmShape s = make_shape(M, N, K, kBNWide, 1, kGroupM, kCG);
    EpiStoreF32::Params ep{static_cast<float*>(C), ldc, accumulate};
    switch (sel) {
      case 0: return launch_gemm<kCG, false, false, EpiStoreF32, kBNWide>(ma, mb, s, ep, st);
      case 1: return launch_gemm<kCG, false, true, EpiStoreF32, kBNWide>(ma, mb, s, ep, st);
      case 2: return launch_gemm<kCG, true, false, EpiStoreF32, kBNWide>(ma, mb, s, ep, st);
      default: return launch_gemm<kCG, true, true, EpiStoreF32, kBNWide>(ma, mb, s, ep, st);
    }
  }
  const GemmShape s = make_shape(M, N, K, kBN, 1, kGroupM, kCG);
  if (c_fp32) {
    EpiStoreF32::Params ep{static_cast<float*>(C), ldc, accumulate};
    switch (sel) {
      case 0: return launch_gemm<kCG, false, false, EpiStoreF32>(ma, mb, s, ep, st);
      case 1: return launch_gemm<kCG, false, true, EpiStoreF32>(ma, mb, s, ep, st);
      case 2: return launch_gemm<kCG, true, false, EpiStoreF32>(ma, mb, s, ep, st);
      default: return launch_gemm<kCG, true, true, EpiStoreF32>(ma, mb, s, ep, st);
    }
  }
  TL_REQUIRE(!accumulate, TL_ERR_UNSUPPORTED, "accumulate needs fp32 C");
  EpiStoreBF16::Params ep{static_cast<__nv_bfloat16_raw*>(C), ldc, nullptr, nullptr};
  switch (sel) {
    case 0: return launch_gemm<kCG, false, false, EpiStoreBF16>(ma, mb, s, ep, st);
    case 1: return launch_gemm<kCG, false, true, EpiStoreBF16>(ma, mb, s, ep, st);
    case 2: return launch_gemm<kCG, true, false, EpiStoreBF16>(ma, mb, s, ep, st);
    default: return launch_gemm<kCG, true, true, EpiStoreBF16>(ma, mb, s, ep, st);
  }
}

extern "C" int tl_lmhead_logprobs(const uint16_t* hidden, const uint16_t* weight,
                                  const int32_t* targets, const int32_t* idx, int64_t n_rows,
                                  int32_t H, int32_t V, float* logp, float* entropy, float* lse,
                                  int32_t chunk_rows, void* workspace, size_t workspace_bytes,
                                  tl_stream_t stream) {
  TL_REQUIRE(H > 0 && V > 0 && n_rows >= 0 && chunk_rows > 0, TL_ERR_INVALID_ARG, "bad sizes");
  TL_REQUIRE(H % 8 == 0, TL_ERR_UNSUPPORTED, "hidden must be a multiple of 8");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Workspace w{static_cast<char*>(workspace), workspace_bytes};
  ChunkWs c = carve(w, chunk_rows, H, V, 0, 0, 0, false);
  TL_REQUIRE(w.ok(), TL_ERR_WORKSPACE, "lmhead workspace too small");
  for (long long c0 = 0; c0 < n_rows; c0 += chunk_rows) {
    const int rows = static_cast<int>(n_rows - c0 < chunk_rows ? n_rows - c0 : chunk_rows);
    const int32_t* ci = idx ? idx + c0 : nullptr;
    gather_rows_kernel<<<grid_for((long long)rows * H / 8, 256), 256, 0, st>>>(
        reinterpret_cast<const uint4*>(hidden) + (idx ? 0 : c0 * H / 8), ci, rows, H / 8,
        reinterpret_cast<uint4*>(c.h));
    TL_LAUNCH_CHECK();
    gather_i32_kernel<<<grid_for(rows, 256), 256, 0, st>>>(targets + (idx ? 0 : c0), ci, rows, c.y);
    TL_LAUNCH_CHECK();
    count_launch(2);
    CombineArgs ca{};
    ca.logp_row = logp + c0;
    ca.ent_row = entropy ? entropy + c0 : nullptr;
    ca.lse_row = lse ? lse + c0 : nullptr;
    if (int e = lmhead_forward_chunk(c, weight, rows, H, V, ca, st)) return e;
  }
  return TL_OK;
}

extern "C" int tl_grpo_lmhead_step_overlap(
    const uint16_t* hidden, const uint16_t* weight, const int32_t* input_ids,
    const uint8_t* loss_mask, const int32_t* act_idx, int64_t n_act, const int32_t* traj_of_token,
    const int32_t* cu_seqlens, const int32_t* group_off, const float* logp_old,
    const float* logp_ref, const float* adv32, const float* traj_w, int64_t n_tokens, int32_t H,
    int32_t V, int32_t n_traj, int32_t n_groups, const tl_loss_config* cfg, float* logp_out,
    float* entropy_out, uint16_t* dhidden, float* dweight, double* report, int32_t chunk_rows,
    int32_t mode_flags, void* workspace, size_t workspace_bytes, tl_stream_t stream,
    const tl_step_overlap* overlap) {
  TL_REQUIRE(cfg, TL_ERR_INVALID_ARG, "cfg is NULL");
  TL_REQUIRE(!overlap || overlap->reserve_sms >= 0, TL_ERR_INVALID_ARG, "reserve_sms < 0");
  // N2 overlap: the last chunk runs dW before dH and announces the final dW
  cudaEvent_t dw_ready = overlap ? static_cast<cudaEvent_t>(overlap->dw_ready_event) : nullptr;
  const int reserve = overlap ? overlap->reserve_sms : 0;
  const int mode =
      mode_flags & ~(TL_LMHEAD_ACCUMULATE_DW | TL_LMHEAD_NO_SPLIT_TAIL | TL_LMHEAD_NO_FACTORED |
                     TL_LMHEAD_DEBUG_FIXUP);
  const bool acc_dw = (mode_flags & TL_LMHEAD_ACCUMULATE_DW) != 0;
  const bool no_split_tail = (mode_flags & TL_LMHEAD_NO_SPLIT_TAIL) != 0;
  TL_REQUIRE(mode == TL_LMHEAD_STORE_LOGITS || mode == TL_LMHEAD_RECOMPUTE ||
                 mode == TL_LMHEAD_STORE_LOGITS_PIPELINED,
             TL_ERR_INVALID_ARG, "unknown lmhead mode %d", mode_flags);
  TL_REQUIRE(cfg->use_mask == 1, TL_ERR_UNSUPPORTED, "LM-head step computes action rows only");
  TL_REQUIRE(!cfg->has_ref || logp_ref, TL_ERR_INVALID_ARG, "has_ref without logp_ref");
  TL_REQUIRE(H > 0 && V > 0 && chunk_rows > 0 && n_act >= 0, TL_ERR_INVALID_ARG, "bad sizes");
  TL_REQUIRE(H % 64 == 0, TL_ERR_UNSUPPORTED, "hidden must be a multiple of 64");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // backward if either gradient is wanted: dweight NULL = frozen LM head
  // (dH only), dhidden NULL = detached hidden states (dW only)
  const bool bwd = dhidden != nullptr || dweight != nullptr;
  Workspace w{static_cast<char*>(workspace), workspace_bytes};
  ChunkWs c2{};
  ChunkWs c = carve(w, chunk_rows, H, V, n_tokens, n_traj, n_groups, bwd,
                    mode == TL_LMHEAD_STORE_LOGITS_PIPELINED && bwd ? &c2 : nullptr);
  TL_REQUIRE(w.ok(), TL_ERR_WORKSPACE, "lmhead workspace too small (%zu < %zu)", workspace_bytes,
             w.used);
  const long long Vld = vld_of(V);
  // dLoss/dentropy per action token: the bonus is a mean over the step's
  // global action tokens (entropy_norm), not this micro-batch's / rank's
  const double ent_norm = cfg->entropy_norm > 0 ? cfg->entropy_norm : double(n_act);
  const float ent_grad = n_act > 0 ? static_cast<float>(-cfg->entropy_coef / ent_norm) : 0.f;

  // observation rows: logp / entropy 0 and (if training) zero dH rows; their
  // term / k3 / flags slots are never read (the reductions select by mask)
  if (n_tokens > 0) {
    // observation positions report logp 0.0 like cli._flat_logps (cli.py:251)
    cudaMemsetAsync(logp_out, 0, n_tokens * sizeof(float), st);
    cudaMemsetAsync(entropy_out, 0, n_tokens * sizeof(float), st);
    if (dhidden) {
      zero_obs_rows_kernel<<<grid_for(n_tokens * H / 8, 256), 256, 0, st>>>(
          loss_mask, n_tokens, H / 8, reinterpret_cast<uint4*>(dhidden));
      TL_LAUNCH_CHECK();
      count_launch();
    }
  }
  if (dweight && n_act == 0 && !acc_dw) {
    cudaMemsetAsync(dweight, 0, static_cast<size_t>(V) * H * sizeof(float), st);
  }

  const bool store = bwd && mode != TL_LMHEAD_RECOMPUTE;
  // factored store: dS = alpha_r q, no elementwise pass (lmhead_epilogue.cuh)
  // — exact for dLoss/dz without the entropy term
  const bool factored = store && ent_grad == 0.f && !(mode_flags & TL_LMHEAD_NO_FACTORED);
  // the pipelined schedule overlaps the dS pass, which the factored store has not
  const bool pipelined = bwd && mode == TL_LMHEAD_STORE_LOGITS_PIPELINED && !factored;
  const long long n_chunks = (n_act + chunk_rows - 1) / chunk_rows;
  auto rows_of = [&](long long i) {
    const long long c0 = i * chunk_rows;
    return static_cast<int>(n_act - c0 < chunk_rows ? n_act - c0 : chunk_rows);
  };
  const ChunkWs* bufs[2] = {&c, pipelined ? &c2 : &c};

  // stage F: gather the chunk's action rows, fused forward (+ surrogate, + fp16 logits)
  auto stage_fwd = [&](long long i) -> int {
    const ChunkWs& b = *bufs[i & 1];
    const int rows = rows_of(i);
    const int32_t* ci = act_idx + i * chunk_rows;
    if (factored) {
      ProfScope prof(PROF_GATHER, st);
      gather_anchor_kernel<<<grid_for(static_cast<long long>(rows) * 32, 256), 256, 0, st>>>(
          reinterpret_cast<const uint4*>(hidden), reinterpret_cast<const uint4*>(weight), ci,
          input_ids, logp_old, rows, H / 8, V, reinterpret_cast<uint4*>(b.h), b.y, b.anc);
      TL_LAUNCH_CHECK();
      count_launch();
    } else {
      ProfScope prof(PROF_GATHER, st);
      gather_rows_kernel<<<grid_for((long long)rows * H / 8, 256), 256, 0, st>>>(
          reinterpret_cast<const uint4*>(hidden), ci, rows, H / 8, reinterpret_cast<uint4*>(b.h));
      TL_LAUNCH_CHECK();
      gather_i32_kernel<<<grid_for(rows, 256), 256, 0, st>>>(input_ids, ci, rows, b.y);
      TL_LAUNCH_CHECK();
      count_launch(2);
    }
    CombineArgs ca{};
    ca.idx = ci;
    ca.traj_of_token = traj_of_token;
    ca.logp_old = logp_old;
    ca.logp_ref = logp_ref;
    ca.adv = adv32;
    ca.traj_w = traj_w;
    ca.cfg = *cfg;
    ca.ent_grad = ent_grad;
    ca.logp_out = logp_out;
    ca.ent_out = entropy_out;
    ca.term = b.term;
    ca.k3o = b.k3o;
    ca.flags = b.flags;
    ca.g_row = b.g;
    ca.c_row = b.c;
    ca.ez_row = b.ez;
    ca.lse_row = b.lse;
    ca.force_fixup = (mode_flags & TL_LMHEAD_DEBUG_FIXUP) != 0;
    return lmhead_forward_chunk(b, weight, rows, H, V, ca, st, store ? b.ds : nullptr, Vld,
                                store ? b.zoff : nullptr, factored);
  };
  // stage S: dS for the chunk (in place over its fp16 logits, or recomputed)
  auto stage_ds = [&](long long i, cudaStream_t s_ds, int grid) -> int {
    const ChunkWs& b = *bufs[i & 1];
    const int rows = rows_of(i);
    if (factored) {
      ProfScope prof(PROF_RESCALE, s_ds);
      fixup_rows_kernel<<<4 * num_sms(), 256, 0, s_ds>>>(
          b.flagged, reinterpret_cast<const uint4*>(b.h), reinterpret_cast<const uint4*>(weight),
          H / 8, V, b.y, b.lse, b.g, b.alpha, reinterpret_cast<__nv_bfloat16_raw*>(b.ds), Vld);
      TL_LAUNCH_CHECK();
      count_launch();
      if (dweight) {
        scale_rows_kernel<<<grid_for(static_cast<long long>(rows) * H / 8, 256), 256, 0, s_ds>>>(
            reinterpret_cast<uint4*>(b.h), b.alpha, rows, H / 8);
        TL_LAUNCH_CHECK();
        count_launch();
      }
      return TL_OK;
    }
    if (store) {
      ProfScope prof(PROF_DSOFTMAX, s_ds);
      dsoftmax_inplace_kernel<<<grid < rows ? grid : rows, 256, 0, s_ds>>>(
          reinterpret_cast<uint4*>(b.ds), Vld / 8, b.zoff, ldo_of(V), V, rows, b.y, b.lse, b.g,
          b.c, b.ez);
      TL_LAUNCH_CHECK();
      count_launch();
      return TL_OK;
    }
    CUtensorMap ma, mb;
    if (int e = make_ab_maps(&ma, &mb, b.h, false, rows, H, weight, false, V, H, H, kCG)) return e;
    const GemmShape sh = fwd_shape(rows, V, H, b.sync + kSyncWaves);
    EpiDSoftmax::Params ep{b.y, b.lse, b.g, b.c, b.ez,
                           reinterpret_cast<__nv_bfloat16_raw*>(b.ds), Vld};
    return launch_gemm<kCG, false, false, EpiDSoftmax>(ma, mb, sh, ep, s_ds, PROF_GEMM_DS);
  };
  // stage B: dH rows = dS W (scattered to packed positions), dW (+)= dS^T h_c.
  // The last chunk with a dw_ready event: dW first, the event, then dH with
  // `reserve` SMs left free, so the caller's dW collective (issued on another
  // stream after the event) runs beside the dH GEMM.  Either order gives the
  // same bits (dH does not read dW; each dH tile is one pair's full-K sum).
  auto stage_dh = [&](long long i, int reserve_sms) -> int {
    const ChunkWs& b = *bufs[i & 1];
    const int rows = rows_of(i);
    const int32_t* ci = act_idx + i * chunk_rows;
    if (dhidden) {
      CUtensorMap ma, mb;
      if (int e = make_ab_maps(&ma, &mb, b.ds, false, rows, Vld, weight, true, H, H, V, kCG))
        return e;
      // N-complete raster (group_m = 1): all H tiles of an M tile run together
      // so each dS k-block is fetched from HBM once; dS streams (evict first).
      // dS streams (evict_first); W is re-read by every wave and the
      // serpentine order starts each wave on what the last one read
      // (evict_last): -1.1 % dH (gpu_r50)
      const GemmShape sh = with_sync(
          make_shape(rows, H, V, kBNWide, 1, 1, kCG, tune::kDhPolA, tune::kDhPolB),
          b.sync + 2 * kSyncWaves, tune::kBwdSyncBlocks, tune::kBwdSyncWindow, 0, reserve_sms);
      // dhidden rows are written once and not read again in the step
      EpiStoreBF16::Params ep{reinterpret_cast<__nv_bfloat16_raw*>(dhidden), H, ci,
                              factored ? b.alpha : nullptr};
      if (int e = launch_gemm<kCG, false, true, EpiStoreBF16, kBNWide>(ma, mb, sh, ep, st,
                                                                       PROF_GEMM_DH, reserve_sms))
        return e;
    }
    return TL_OK;
  };
  auto stage_dw = [&](long long i) -> int {
    const ChunkWs& b = *bufs[i & 1];
    const int rows = rows_of(i);
    if (!dweight) return TL_OK;
    CUtensorMap ma, mb;
    if (int e = make_ab_maps(&ma, &mb, b.ds, true, V, Vld, b.h, true, H, H, rows, kCG)) return e;
    GemmShape sh = with_sync(
        make_shape(V, H, rows, kBNWide, 1, 1, kCG, tune::kDwPolA, tune::kDwPolB),
        b.sync + 3 * kSyncWaves, tune::kBwdSyncBlocks, tune::kBwdSyncWindow);
    if (!no_split_tail) {  // split-K tail for the partial last wave
      sh.tail_part = b.tail_part;
      sh.tail_ctr = b.tail_ctr;
    }
    EpiStoreF32::Params ep{dweight, H, (i > 0 || acc_dw) ? 1 : 0};
    return launch_gemm<kCG, true, true, EpiStoreF32, kBNWide>(ma, mb, sh, ep, st, PROF_GEMM_DW);
  };
  auto stage_bwd = [&](long long i) -> int {
    if (dw_ready && i == n_chunks - 1) {
      if (int e = stage_dw(i)) return e;
      TL_CUDA_TRY(cudaEventRecord(dw_ready, st));
      return stage_dh(i, reserve);
    }
    if (int e = stage_dh(i, 0)) return e;
    return stage_dw(i);
  };

  if (!pipelined) {
    for (long long i = 0; i < n_chunks; ++i) {
      if (int e = stage_fwd(i)) return e;
      if (!bwd) continue;
      if (int e = stage_ds(i, st, 1 << 30)) return e;
      if (int e = stage_bwd(i)) return e;
    }
  } else if (n_chunks > 0) {
    // Two chunk buffers; chunk i's dS pass runs on a side stream beside chunk
    // i+1's forward GEMM (the GEMM is tensor-bound and leaves HBM idle):
    //   main: F0 F1 . B0 F2 . B1 F3 . B2 ...      side: S0 (|| F1)  S1 (|| F2) ...
    // S_i is submitted after F_{i+1} so the GEMM's persistent CTAs are placed
    // first and the pass (a small grid-strided grid) fills the remaining slots.
    StreamPair sp;
    if (sp.err) return sp.err;
    const int ds_grid = tune::kDsOverlapCtasPerSm * num_sms();
    if (int e = stage_fwd(0)) return e;
    for (long long i = 0; i < n_chunks; ++i) {
      TL_CUDA_TRY(cudaEventRecord(sp.ev_fwd, st));  // F_i done
      if (i + 1 < n_chunks)
        if (int e = stage_fwd(i + 1)) return e;     // buffer (i+1)&1, freed by B_{i-1}
      TL_CUDA_TRY(cudaStreamWaitEvent(sp.side, sp.ev_fwd, 0));
      if (int e = stage_ds(i, sp.side, ds_grid)) return e;
      TL_CUDA_TRY(cudaEventRecord(sp.ev_ds, sp.side));
      TL_CUDA_TRY(cudaStreamWaitEvent(st, sp.ev_ds, 0));
      if (int e = stage_bwd(i)) return e;
    }
  }
  // no chunk (or no backward): dW is final now
  if (dw_ready && (n_chunks == 0 || !bwd)) TL_CUDA_TRY(cudaEventRecord(dw_ready, st));
  return launch_reductions(c.term, c.k3o, c.flags, entropy_out, loss_mask, 1, cu_seqlens,
                           group_off, n_traj, n_groups, n_tokens, cfg->agg, c.red, report, st);
}

extern "C" int tl_grpo_lmhead_step(const uint16_t* hidden, const uint16_t* weight,
                                   const int32_t* input_ids, const uint8_t* loss_mask,
                                   const int32_t* act_idx, int64_t n_act,
                                   const int32_t* traj_of_token, const int32_t* cu_seqlens,
                                   const int32_t* group_off, const float* logp_old,
                                   const float* logp_ref, const float* adv32, const float* traj_w,
                                   int64_t n_tokens, int32_t H, int32_t V, int32_t n_traj,
                                   int32_t n_groups, const tl_loss_config* cfg, float* logp_out,
                                   float* entropy_out, uint16_t* dhidden, float* dweight,
                                   double* report, int32_t chunk_rows, int32_t mode_flags,
                                   void* workspace, size_t workspace_bytes, tl_stream_t stream) {
  return tl_grpo_lmhead_step_overlap(hidden, weight, input_ids, loss_mask, act_idx, n_act,
                                     traj_of_token, cu_seqlens, group_off, logp_old, logp_ref,
                                     adv32, traj_w, n_tokens, H, V, n_traj, n_groups, cfg,
                                     logp_out, entropy_out, dhidden, dweight, report, chunk_rows,
                                     mode_flags, workspace, workspace_bytes, stream, nullptr);
}
