// Persistent, warp-specialised tcgen05 GEMM for sm_100a:
//   D[M, N] = A[M, K] * B[N, K]^T     (bf16 operands, fp32 accumulate in TMEM)
// with a pluggable epilogue that consumes the fp32 accumulator straight from
// TMEM.  Both operands may be K-major or MN-major in global memory; TMA
// (SWIZZLE_128B) stages them into a STAGES-deep shared-memory ring, one
// elected thread issues tcgen05.mma (K=16), accumulators are double-buffered
// in TMEM (2 x BN columns, BN <= 256) so the epilogue of tile i overlaps the
// MMAs of tile i+1; BN = 512 tiles (dH / dW) use all 512 columns once.
//
// CG = 1: one CTA per tile, UMMA 128 x BN.
// CG = 2: a 2-CTA cluster (one TPC) per tile, UMMA 256 x BN issued by the
//   leader (tcgen05.mma.cta_group::2): each CTA stages its own 128 A rows and
//   HALF of the B tile, so per-SM shared-memory fill and L2 reads per FLOP
//   drop by a third versus CG = 1 (the step is power-capped, so bytes moved per
//   FLOP set the clock).  TMA completion is counted on the leader's barrier,
//   MMA completion is multicast to both CTAs' barriers, the peer's epilogue
//   signals the leader's TMEM-empty barrier remotely.
//
// Warp roles (256 threads per CTA):
//   warp 0      TMA producer (one lane)            [both CTAs]
//   warp 1      MMA issuer (one lane)              [leader only]
//   warp 2      TMEM allocator / deallocator
//   warp 3      idle
//   warps 4..7  epilogue: warp (4+q) owns TMEM lanes [32q, 32q+32) = tile rows
//
// Work decomposition: a "unit" is (m_tile of 128*CG rows, a strip of `strip`
// consecutive n_tiles).  Units are rasterised in groups of `group_m` M-tiles
// (all strips of the group before the next group) so the concurrently running
// units share A and B tiles in L2; unit u runs on CTA(-pair) u % n_pairs.  The
// epilogue sees begin_unit / tile / end_unit so row-wise reductions over a
// strip (the online log-sum-exp of the LM head) stay in registers.
//
// L2 reuse across CTAs (the step is energy-bound):
//   wave lockstep  the i-th units of all CTA pairs form wave i; producers
//                  publish progress on a per-wave (or per-(wave, strip)
//                  group) counter and may run at most `sync_window` sync
//                  steps ahead of the slowest member, so tiles that share an
//                  operand load it while it is still in L2;
//   serpentine K   tiles of odd (wave + tile) parity stream their k-blocks
//                  last-to-first, starting on what the previous tile (and
//                  the wave) read last.
#pragma once
#include <cuda_bf16.h>

#include "sm100_ptx.cuh"

// Optional stall accounting (profiling builds only: TL_GEMM_STATS=1, see
// tools/gemm_stats.py): per CTA, clock64 cycles spent in each wait of the
// three roles, accumulated into tl::g_gemm_stats[blockIdx.x * 8 + slot].
#ifndef TL_GEMM_STATS
#define TL_GEMM_STATS 0
#endif

namespace tl {

#if TL_GEMM_STATS
__device__ unsigned long long* g_gemm_stats = nullptr;  // one TU (lmhead.cu) includes this
enum { ST_PROD_SYNC = 0, ST_PROD_EMPTY, ST_MMA_FULL, ST_MMA_TEMPTY, ST_MMA_TOTAL, ST_EPI_TFULL,
       ST_EPI_TILE, ST_EPI_END };
// accumulated in registers, flushed once per thread at kernel exit
#define TL_STAT_DECL long long tl_stat[8] = {0, 0, 0, 0, 0, 0, 0, 0}
#define TL_STAT_BEGIN(v) const long long v = clock64()
#define TL_STAT_END(v, slot) (tl_stat[(slot)] += clock64() - (v))
#define TL_STAT_FLUSH()                                                                  \
  do {                                                                                   \
    unsigned long long* gs = g_gemm_stats;                                               \
    if (gs)                                                                              \
      for (int i_ = 0; i_ < 8; ++i_)                                                     \
        if (tl_stat[i_]) atomicAdd(gs + blockIdx.x * 8 + i_,                            \
                                   static_cast<unsigned long long>(tl_stat[i_]));         \
  } while (0)
#else
#define TL_STAT_DECL
#define TL_STAT_BEGIN(v)
#define TL_STAT_END(v, slot)
#define TL_STAT_FLUSH()
#endif

constexpr int kBM = 128;  // rows per CTA
constexpr int kBK = 64;
constexpr int kGemmThreads = 256;
constexpr int kEpiWarp0 = 4;

struct GemmShape {
  int M, N, K;
  int m_tiles, n_tiles, k_blocks;
  int strip;      // n-tiles per unit
  int n_strips;   // ceil(n_tiles / strip)
  int group_m;    // M-tiles per raster group
  int n_units;
  int cg;         // CTAs per tile (M rows per tile = 128 * cg)
  int pol_a, pol_b;  // L2 eviction policy of the A / B TMA loads (make_policy)
  // Wave lockstep (optional): the i-th unit of every CTA(-pair) forms wave i;
  // within a wave every CTA bumps sync_ctr[i] after each `sync_every`
  // k-blocks it has issued, and may not start sync step s before all CTAs of
  // the wave finished step s - sync_window.  Keeps the CTAs that share A / B
  // tiles within a few k-blocks of each other so the sharing hits L2
  // (unsynchronised they drift apart and re-read operands from HBM 10-18x).
  int* sync_ctr;  // [n_waves] (or [n_waves * 8] split), zeroed before launch (NULL = off)
  int sync_every, sync_window;
  // sync_split: lockstep only among the CTAs of a wave that run the same
  // (M group, strip) — the ones sharing B tiles — instead of the whole wave.
  int sync_split;
  // Serpentine K order: tiles with odd (wave + tile-in-unit) parity stream
  // their k-blocks last-to-first, so each tile starts on the operand blocks
  // the previous tile (of this CTA and, in lockstep, of its whole wave) read
  // last — still in L2 when the operand is too large to stay resident.  Only
  // the producer's block order changes (fixed per tile: deterministic).
  // serpentine == 2: parity of the global N tile instead (strip shapes: a
  // CTA still alternates along its strip), so an output element's K order —
  // and its fp32 bits — do not depend on which M tile / wave / chunk its row
  // landed in (the LM-head forward: per-row outputs invariant under
  // chunking and data-parallel sharding).
  int serpentine;
  // Split-K tail (strip == 1 shapes, epilogues with Epi::kSplitTail; set by
  // the launcher once it knows the number of co-resident pairs): the units of
  // a partial last wave [tail_begin, n_units) are cut into tail_split
  // K-slices that run as separate work items on the otherwise idle pairs.
  // Each slice writes its fp32 partial tile to tail_part; the slice that
  // arrives last for a tile half (counter tail_ctr) sums all slices in slice
  // order and hands the sum to the epilogue's final write: deterministic.
  int tail_begin;    // == n_units: off
  int tail_split;
  float* tail_part;  // [(n_units - tail_begin) * tail_split][cg][kBM][BN]
  int* tail_ctr;     // [(n_units - tail_begin) * cg], zeroed before launch
};

struct UnitCoord {
  int m_tile, n_begin, n_count, strip_idx;
};

__host__ __device__ inline UnitCoord unit_coord(const GemmShape& s, int u) {
  const int per_full_group = s.group_m * s.n_strips;
  const int full_groups = s.m_tiles / s.group_m;
  int mg, rem, rows;
  if (u < full_groups * per_full_group) {
    mg = u / per_full_group;
    rem = u - mg * per_full_group;
    rows = s.group_m;
  } else {
    mg = full_groups;
    rem = u - full_groups * per_full_group;
    rows = s.m_tiles - full_groups * s.group_m;
  }
  const int strip_idx = rem / rows;
  const int mi = rem - strip_idx * rows;
  UnitCoord c;
  c.m_tile = mg * s.group_m + mi;
  c.strip_idx = strip_idx;
  c.n_begin = strip_idx * s.strip;
  c.n_count = min(s.strip, s.n_tiles - c.n_begin);
  return c;
}

// Work item i of the persistent schedule: a whole unit, or (tail) one
// K-slice [kb_begin, kb_end) of a unit; piece = slice index among all tail
// slices, -1 for a whole unit.
struct WorkItem {
  int unit, kb_begin, kb_end, piece;
};

__host__ __device__ inline int n_work_items(const GemmShape& s) {
  return s.tail_begin + (s.n_units - s.tail_begin) * s.tail_split;
}

__host__ __device__ inline WorkItem work_item(const GemmShape& s, int i) {
  WorkItem w;
  if (i < s.tail_begin) {
    w.unit = i;
    w.kb_begin = 0;
    w.kb_end = s.k_blocks;
    w.piece = -1;
    return w;
  }
  const int q = i - s.tail_begin;
  const int t = q / s.tail_split, sl = q - t * s.tail_split;
  w.unit = s.tail_begin + t;
  w.kb_begin = static_cast<int>(static_cast<long long>(s.k_blocks) * sl / s.tail_split);
  w.kb_end = static_cast<int>(static_cast<long long>(s.k_blocks) * (sl + 1) / s.tail_split);
  w.piece = q;
  return w;
}

inline GemmShape make_shape(int M, int N, int K, int BN, int strip, int group_m, int cg = 1,
                            int pol_a = 0, int pol_b = 0) {
  GemmShape s;
  s.M = M;
  s.N = N;
  s.K = K;
  s.cg = cg;
  s.pol_a = pol_a;
  s.pol_b = pol_b;
  s.sync_ctr = nullptr;
  s.sync_every = 0;
  s.sync_window = 0;
  s.sync_split = 0;
  s.serpentine = 0;
  s.tail_split = 1;
  s.tail_part = nullptr;
  s.tail_ctr = nullptr;
  s.m_tiles = (M + kBM * cg - 1) / (kBM * cg);
  s.n_tiles = (N + BN - 1) / BN;
  s.k_blocks = (K + kBK - 1) / kBK;
  s.strip = strip < 1 ? 1 : (strip > s.n_tiles ? s.n_tiles : strip);
  s.n_strips = (s.n_tiles + s.strip - 1) / s.strip;
  s.group_m = group_m < 1 ? 1 : (group_m > s.m_tiles ? s.m_tiles : group_m);
  s.n_units = s.m_tiles * s.n_strips;
  s.tail_begin = s.n_units;
  return s;
}

// BN = tile width; UMMA instructions are N = min(BN, 256) wide, NSUB of them
// per k-step side by side in TMEM; accumulators are double-buffered when two
// tiles fit in TMEM's 512 columns (BN <= 256), single-buffered for BN = 512.
template <int BN, int STAGES, int CG>
struct GemmSmem {
  static constexpr int kUmmaN = BN < 256 ? BN : 256;
  static constexpr int kNSub = BN / kUmmaN;
  static constexpr int kNAcc = 2 * BN <= 512 ? 2 : 1;
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBRows = kUmmaN / CG;  // B rows staged by each CTA per sub-MMA
  static constexpr int kBSubBytes = kBRows * kBK * 2;
  static constexpr int kBBytes = kNSub * kBSubBytes;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kBarOffset = STAGES * kStageBytes;
  // full[S], empty[S], tmem_full[2], tmem_empty[2], tmem base slot
  static constexpr int kBytes = kBarOffset + (2 * STAGES + 4) * 8 + 16 + 1024;  // +1 KB align
};

// Walk a thread's BN-wide accumulator row in 32-column slices, the next
// slice's tcgen05.ld in flight while the current one is consumed by f(col,
// regs) (the ld is warp-collective: every lane calls this, in-range or not).
#ifndef TL_EPI_PIPELINE
#define TL_EPI_PIPELINE 1
#endif
template <int BN, class F>
__device__ __forceinline__ void tmem_row_slices(uint32_t taddr, F&& f) {
  static_assert(BN % 64 == 0, "slices are processed in pairs");
  if constexpr (!TL_EPI_PIPELINE) {  // A/B reference: one slice at a time
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t r[32];
      tmem_ld32(taddr + c, r);
      tmem_ld_wait_regs(r);
      f(c, r);
    }
    return;
  }
  uint32_t ra[32], rb[32];
  tmem_ld32(taddr, ra);
  tmem_ld_wait_regs(ra);
#pragma unroll 1
  for (int c = 0; c < BN; c += 64) {
    tmem_ld32(taddr + c + 32, rb);
    f(c, ra);
    tmem_ld_wait_regs(rb);
    const bool more = c + 64 < BN;
    if (more) tmem_ld32(taddr + c + 64, ra);
    f(c + 32, rb);
    if (more) tmem_ld_wait_regs(ra);
  }
}

template <int BN, int STAGES, int CG, bool A_MN, bool B_MN, class Epi>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_sm100_kernel(const __grid_constant__ CUtensorMap map_a,
                      const __grid_constant__ CUtensorMap map_b, const GemmShape shape,
                      const typename Epi::Params ep) {
  using Smem = GemmSmem<BN, STAGES, CG>;
  static_assert(BN % 64 == 0 && BN >= 64 && BN <= 512 && (BN <= 256 || BN % 256 == 0), "BN");
  static_assert(CG == 1 || CG == 2, "CG");
  static_assert(Smem::kBRows % 64 == 0, "B half tile must be a multiple of 64 rows");
  constexpr int kNAcc = Smem::kNAcc;
  constexpr int kUmmaN = Smem::kUmmaN;
  constexpr uint32_t kCols = kNAcc * BN;
  constexpr uint32_t kTmemCols = kCols <= 32 ? 32 : (kCols <= 64 ? 64 : (kCols <= 128 ? 128 : (kCols <= 256 ? 256 : 512)));
  constexpr uint32_t kIdesc = idesc_bf16(kBM * CG, kUmmaN, A_MN ? 1u : 0u, B_MN ? 1u : 0u);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Smem::kBarOffset);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x / 32;
  const uint32_t lane = threadIdx.x % 32;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
  const int pair = CG == 2 ? static_cast<int>(cluster_id_x()) : static_cast<int>(blockIdx.x);
  const int n_pairs = CG == 2 ? static_cast<int>(nclusters_x()) : static_cast<int>(gridDim.x);

  if (warp == 0 && lane == 0) {
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 4 * CG);  // one arrive per epilogue warp of the pair
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (CG == 2) tmem_alloc_cg2<kTmemCols>(tmem_slot);
    else tmem_alloc<kTmemCols>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  TL_STAT_DECL;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer --
    if (lane == 0) {
      const uint64_t pol_a = make_policy(shape.pol_a);
      const uint64_t pol_b = make_policy(shape.pol_b);
      int stage = 0;
      uint32_t phase = 0;
      int wave = 0;
      const int n_items = n_work_items(shape);
      for (int it = pair; it < n_items; it += n_pairs, ++wave) {
        const WorkItem wi = work_item(shape, it);
        const int u = wi.unit;
        const int nkb = wi.kb_end - wi.kb_begin;
        const UnitCoord uc = unit_coord(shape, u);
        const int m0 = uc.m_tile * kBM * CG + static_cast<int>(rank) * kBM;
        int* ctr = nullptr;
        int wave_ctas = 0;
        if (shape.sync_ctr) {
          const int w0 = wave * n_pairs;
          const int wn = min(n_pairs, n_items - w0);
          if (shape.sync_split) {
            auto key = [&](int ii) {
              const UnitCoord c = unit_coord(shape, work_item(shape, ii).unit);
              return (c.m_tile / shape.group_m) * shape.n_strips + c.strip_idx;
            };
            const int km = key(it);
            int cnt = 0;
            for (int j = 0; j < wn; ++j) cnt += key(w0 + j) == km;
            const int slot = km - key(w0);  // keys ascend within a wave
            // slots >= 8 share the last counter: extra arrivals only loosen the wait
            ctr = shape.sync_ctr + wave * 8 + (slot < 8 ? slot : 7);
            wave_ctas = CG * cnt;
          } else {
            ctr = shape.sync_ctr + wave;
            wave_ctas = CG * wn;
          }
        }
        int sstep = 0, in_step = 0;
        bool do_wait = true;
        for (int t = 0; t < uc.n_count; ++t) {
          // sub-MMA j covers tile columns [j*kUmmaN, (j+1)*kUmmaN); this CTA
          // stages rows rank*kBRows.. of each (the pair MMA splits B in half)
          const int n0 = (uc.n_begin + t) * BN + static_cast<int>(rank) * Smem::kBRows;
          const bool rev = shape.serpentine == 2 ? ((uc.n_begin + t) & 1)
                                                 : (shape.serpentine && ((wave + t) & 1));
          for (int kb = 0; kb < nkb; ++kb) {
            if (ctr && do_wait && in_step == 0 && sstep >= shape.sync_window) {
              // The lockstep only shapes L2 reuse, never correctness: a wait that
              // exceeds ~50 ms (co-residency lost, preemption) stops waiting for
              // the rest of this wave instead of hanging (progress is still
              // published so the other CTAs are not held up either).
              const int need = wave_ctas * (sstep - shape.sync_window + 1);
              int spins = 0;
              TL_STAT_BEGIN(t_sync);
              while (ld_acquire_gpu(ctr) < need) {
                __nanosleep(64);
                if (++spins > (1 << 19)) {
                  do_wait = false;
                  break;
                }
              }
              TL_STAT_END(t_sync, ST_PROD_SYNC);
            }
            {
              TL_STAT_BEGIN(t_e);
              mbar_wait(&empty_bar[stage], phase ^ 1);
              TL_STAT_END(t_e, ST_PROD_EMPTY);
            }
            uint8_t* sa = smem + stage * Smem::kStageBytes;
            uint8_t* sb = sa + Smem::kABytes;
            if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], CG * Smem::kStageBytes);
            const int k0 = (rev ? wi.kb_end - 1 - kb : wi.kb_begin + kb) * kBK;
            auto load = [&](const CUtensorMap* m, void* dst, int c0, int c1, uint64_t pol) {
              if constexpr (CG == 2) tma_load_2d_cg2(m, &full_bar[stage], dst, c0, c1, pol);
              else tma_load_2d(m, &full_bar[stage], dst, c0, c1, pol);
            };
            if constexpr (!A_MN) {
              load(&map_a, sa, k0, m0, pol_a);
            } else {
#pragma unroll
              for (int j = 0; j < kBM / 64; ++j) load(&map_a, sa + j * 8192, m0 + 64 * j, k0, pol_a);
            }
#pragma unroll
            for (int js = 0; js < Smem::kNSub; ++js) {
              uint8_t* sbj = sb + js * Smem::kBSubBytes;
              const int nj = n0 + js * kUmmaN;
              if constexpr (!B_MN) {
                load(&map_b, sbj, k0, nj, pol_b);
              } else {
#pragma unroll
                for (int j = 0; j < Smem::kBRows / 64; ++j)
                  load(&map_b, sbj + j * 8192, nj + 64 * j, k0, pol_b);
              }
            }
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
            if (ctr && ++in_step == shape.sync_every) {
              red_release_gpu_add(ctr, 1);
              in_step = 0;
              ++sstep;
            }
          }
        }
        if (ctr) {
          // a unit shorter than the wave's longest counts as finished for
          // every step a longer unit can still wait on
          const int max_steps = (shape.strip * shape.k_blocks + shape.sync_every - 1) / shape.sync_every;
          if (max_steps > sstep) red_release_gpu_add(ctr, max_steps - sstep);
        }
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------- MMA issuer --
    if (lane == 0 && rank == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      TL_STAT_BEGIN(t_all);
      const int n_items = n_work_items(shape);
      for (int it = pair; it < n_items; it += n_pairs) {
        const WorkItem wi = work_item(shape, it);
        const int nkb = wi.kb_end - wi.kb_begin;
        const UnitCoord uc = unit_coord(shape, wi.unit);
        for (int t = 0; t < uc.n_count; ++t) {
          {
            TL_STAT_BEGIN(t_te);
            mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
            TL_STAT_END(t_te, ST_MMA_TEMPTY);
          }
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * BN;
          for (int kb = 0; kb < nkb; ++kb) {
            {
              TL_STAT_BEGIN(t_f);
              mbar_wait(&full_bar[stage], phase);
              TL_STAT_END(t_f, ST_MMA_FULL);
            }
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + stage * Smem::kStageBytes);
            const uint32_t sb = sa + Smem::kABytes;
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk) {
              const uint64_t da = A_MN ? sw128_desc(sa + kk * 2048, 8192, 1024)
                                       : sw128_desc(sa + kk * 32, 16, 1024);
#pragma unroll
              for (int js = 0; js < Smem::kNSub; ++js) {
                const uint32_t sbj = sb + js * Smem::kBSubBytes;
                const uint64_t db = B_MN ? sw128_desc(sbj + kk * 2048, 8192, 1024)
                                         : sw128_desc(sbj + kk * 32, 16, 1024);
                const uint32_t dj = d_tmem + js * kUmmaN;
                if constexpr (CG == 2) umma_bf16_cg2(dj, da, db, kIdesc, (kb | kk) != 0 ? 1u : 0u);
                else umma_bf16(dj, da, db, kIdesc, (kb | kk) != 0 ? 1u : 0u);
              }
            }
            if constexpr (CG == 2) umma_commit_cg2_mc(&empty_bar[stage]);
            else umma_commit(&empty_bar[stage]);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          if constexpr (CG == 2) umma_commit_cg2_mc(&tfull_bar[acc]);
          else umma_commit(&tfull_bar[acc]);
          if (++acc == kNAcc) {
            acc = 0;
            acc_phase ^= 1;
          }
        }
      }
      TL_STAT_END(t_all, ST_MMA_TOTAL);
    }
  } else if (warp >= kEpiWarp0) {
    // ---------------------------------------------------------- epilogue --
    const int q = warp - kEpiWarp0;  // TMEM lane quarter
    const int row_in_tile = q * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    typename Epi::State st;
    const int n_items = n_work_items(shape);
    for (int it = pair; it < n_items; it += n_pairs) {
      const WorkItem wi = work_item(shape, it);
      const UnitCoord uc = unit_coord(shape, wi.unit);
      const int row = uc.m_tile * kBM * CG + static_cast<int>(rank) * kBM + row_in_tile;
      Epi::begin_unit(ep, shape, st, row, uc);
      for (int t = 0; t < uc.n_count; ++t) {
        {
          TL_STAT_BEGIN(t_tf);
          mbar_wait(&tfull_bar[acc], acc_phase);
          if (lane == 0 && q == 0) TL_STAT_END(t_tf, ST_EPI_TFULL);
        }
        tc_fence_after();
        const uint32_t taddr = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
        TL_STAT_BEGIN(t_tile);
        if constexpr (Epi::kSplitTail) {
          if (wi.piece >= 0) {
            // tail slice: park this slice's fp32 partial tile (this CTA's rows)
            float* part = shape.tail_part +
                          ((static_cast<long long>(wi.piece) * CG + rank) * kBM + row_in_tile) * BN;
            tmem_row_slices<BN>(taddr, [&](int c, const uint32_t (&r)[32]) {
#pragma unroll
              for (int j = 0; j < 32; j += 4)
                __stcg(reinterpret_cast<float4*>(part + c + j),
                       make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                   __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3])));
            });
          } else {
            Epi::template tile<BN>(ep, shape, st, row, (uc.n_begin + t) * BN, taddr);
          }
        } else {
          Epi::template tile<BN>(ep, shape, st, row, (uc.n_begin + t) * BN, taddr);
        }
        if (lane == 0 && q == 0) TL_STAT_END(t_tile, ST_EPI_TILE);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2) mbar_arrive_cluster(&tempty_bar[acc], 0);
          else mbar_arrive(&tempty_bar[acc]);
        }
        if (++acc == kNAcc) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      TL_STAT_BEGIN(t_end);
      if constexpr (Epi::kSplitTail) {
        if (wi.piece >= 0) {
          // the last slice to arrive for this tile half sums all slices in
          // slice order (deterministic) and performs the epilogue's write
          __shared__ int s_last;
          __threadfence();                                            // release the partial
          asm volatile("bar.sync 1, %0;" ::"n"(4 * 32) : "memory");  // 4 epilogue warps
          const int t_local = wi.unit - shape.tail_begin;
          if (q == 0 && lane == 0) {
            int* c = shape.tail_ctr + t_local * CG + rank;
            const int prev = atomicAdd(c, 1);
            s_last = prev == shape.tail_split - 1;
          }
          asm volatile("bar.sync 1, %0;" ::"n"(4 * 32) : "memory");
          if (s_last) {
            __threadfence();  // acquire the other slices' partials
            const float* p0 = shape.tail_part +
                              ((static_cast<long long>(t_local) * shape.tail_split * CG + rank) * kBM +
                               row_in_tile) * BN;
            const long long slice_stride = static_cast<long long>(CG) * kBM * BN;
            for (int c = 0; c < BN; c += 4) {
              float4 v = __ldcg(reinterpret_cast<const float4*>(p0 + c));
              for (int sl = 1; sl < shape.tail_split; ++sl) {
                const float4 w = __ldcg(reinterpret_cast<const float4*>(p0 + sl * slice_stride + c));
                v.x += w.x;
                v.y += w.y;
                v.z += w.z;
                v.w += w.w;
              }
              Epi::store4(ep, shape, row, uc.n_begin * BN + c, v);
            }
          }
        } else {
          Epi::end_unit(ep, shape, st, row, uc);
        }
      } else {
        Epi::end_unit(ep, shape, st, row, uc);
      }
      if (lane == 0 && q == 0) TL_STAT_END(t_end, ST_EPI_END);
    }
  }

  TL_STAT_FLUSH();
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();
  else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (CG == 2) tmem_dealloc_cg2<kTmemCols>(tmem_base);
    else tmem_dealloc<kTmemCols>(tmem_base);
  }
}

// ------------------------------------------------------- epilogue helpers --
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// Plain store of the fp32 accumulator as bf16 (optionally with a row remap
// and a per-row fp32 scale), used for the dH GEMM (rows scattered back to
// packed positions; the factored backward's alpha_r) and tests.
struct EpiStoreBF16 {
  static constexpr bool kSplitTail = false;
  struct Params {
    __nv_bfloat16_raw* out;
    long long ldo;            // elements
    const int32_t* row_map;   // nullable: out row = row_map[row]
    const float* row_scale;   // nullable: out = row_scale[row] * acc
  };
  struct State {};
  __device__ static void begin_unit(const Params&, const GemmShape&, State&, int, const UnitCoord&) {}
  __device__ static void end_unit(const Params&, const GemmShape&, State&, int, const UnitCoord&) {}
  template <int BN>
  __device__ static void tile(const Params& p, const GemmShape& s, State&, int row, int col0,
                              uint32_t taddr) {
    const bool row_ok = row < s.M;
    long long orow = row;
    if (row_ok && p.row_map) orow = p.row_map[row];
    const bool scaled = p.row_scale != nullptr;
    const float sc = row_ok && scaled ? p.row_scale[row] : 1.f;
    tmem_row_slices<BN>(taddr, [&](int c, const uint32_t (&r)[32]) {
      if (!row_ok) return;
      const int cb = col0 + c;
      __nv_bfloat16_raw* dst = p.out + orow * p.ldo + cb;
      // a zero scale writes exact zeros whatever the accumulator holds (the
      // factored backward's rows without gradient may sum far-off-anchor q
      // past the fp32 range: 0 * inf must not become NaN)
      auto val = [&](int j) {
        return scaled ? (sc != 0.f ? __uint_as_float(r[j]) * sc : 0.f) : __uint_as_float(r[j]);
      };
      if (cb + 32 <= s.N) {
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          uint4 v;
          v.x = pack_bf16x2(val(j + 0), val(j + 1));
          v.y = pack_bf16x2(val(j + 2), val(j + 3));
          v.z = pack_bf16x2(val(j + 4), val(j + 5));
          v.w = pack_bf16x2(val(j + 6), val(j + 7));
          *reinterpret_cast<uint4*>(dst + j) = v;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (cb + j < s.N) {
            const uint32_t b = pack_bf16x2(val(j), 0.f);
            dst[j].x = static_cast<unsigned short>(b & 0xFFFFu);
          }
        }
      }
    });
  }
};

// fp32 store or accumulate (out += acc), used for dW across token chunks.
// Accumulation is a fire-and-forget vector reduction at L2 (red.add.v4.f32):
// the dW tile is BN = 512 wide and single-buffered in TMEM, so an epilogue
// waiting on 512 loads per row (load + add + store) would stall the next
// tile's MMAs (dW -7 % per chunk).  Each element has one writer per launch,
// so the result is deterministic.
struct EpiStoreF32 {
  static constexpr bool kSplitTail = true;
  struct Params {
    float* out;
    long long ldo;
    int accumulate;
  };
  struct State {};
  __device__ static void begin_unit(const Params&, const GemmShape&, State&, int, const UnitCoord&) {}
  __device__ static void end_unit(const Params&, const GemmShape&, State&, int, const UnitCoord&) {}
  // out[row, col .. col+3] (+)= v  (also the final write of a split-K tail tile)
  __device__ static __forceinline__ void store4(const Params& p, const GemmShape& s, int row,
                                                int col, float4 v) {
    if (row >= s.M) return;
    float* dst = p.out + static_cast<long long>(row) * p.ldo + col;
    if (col + 4 <= s.N) {
      if (p.accumulate)
        red_add_v4_f32(dst, v);
      else
        *reinterpret_cast<float4*>(dst) = v;
    } else {
      const float e[4] = {v.x, v.y, v.z, v.w};
      for (int j = 0; j < 4; ++j)
        if (col + j < s.N) dst[j] = (p.accumulate ? dst[j] : 0.f) + e[j];
    }
  }
  template <int BN>
  __device__ static void tile(const Params& p, const GemmShape& s, State&, int row, int col0,
                              uint32_t taddr) {
    tmem_row_slices<BN>(taddr, [&](int c, const uint32_t (&r)[32]) {
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        store4(p, s, row, col0 + c + j,
               make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                           __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3])));
    });
  }
};

}  // namespace tl
