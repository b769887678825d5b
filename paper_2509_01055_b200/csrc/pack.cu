// K1 — trajectory packer.
//
// Reference semantics: trajectory.flatten (trajectory.py:154-159) concatenates
// the per-segment token lists without re-tokenising; trajectory.action_mask
// (trajectory.py:162-167) is 1 on action tokens, 0 on observation tokens;
// rl.loss.token_records (loss.py:76-100) zips them per token.  Here the whole
// batch is packed at once into varlen (cu_seqlens) form plus the action-row
// index the LM head runs on.
//
//  pack_scan_kernel    one CTA: block-wide exclusive scans over the segment
//                      table (packed offset and action offset of every
//                      segment), segment->trajectory map, cu_seqlens, act_off.
//  pack_scatter_kernel token-parallel: every thread owns 4 consecutive packed
//                      positions (16-byte vector stores of ids / positions /
//                      trajectory ids, 4-byte mask stores), finds its segment
//                      by binary search over the segment offsets, and copies
//                      from the (arbitrarily ordered) token pool.
#include "tl_common.cuh"

namespace tl {
namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;

struct ScanPair {
  int a, b;
};

__device__ __forceinline__ ScanPair warp_incl_scan(ScanPair v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int xa = __shfl_up_sync(0xffffffffu, v.a, o);
    const int xb = __shfl_up_sync(0xffffffffu, v.b, o);
    if (lane >= o) {
      v.a += xa;
      v.b += xb;
    }
  }
  return v;
}

__global__ void __launch_bounds__(kScanThreads)
    pack_scan_kernel(const int32_t* __restrict__ seg_len, const uint8_t* __restrict__ seg_is_action,
                     const int32_t* __restrict__ traj_seg_off, int n_traj, int n_seg,
                     int32_t* __restrict__ seg_dst, int32_t* __restrict__ seg_act_dst,
                     int32_t* __restrict__ seg_traj, int32_t* __restrict__ seg_tstart,
                     int32_t* __restrict__ cu_seqlens, int32_t* __restrict__ act_off) {
  __shared__ ScanPair warp_tot[kScanThreads / 32];
  __shared__ ScanPair carry_sh;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  ScanPair carry{0, 0};
  for (int base = 0; base < n_seg; base += kScanThreads * kScanItems) {
    int la[kScanItems], lb[kScanItems];
    ScanPair tot{0, 0};
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      const int s = base + tid * kScanItems + i;
      const int len = s < n_seg ? seg_len[s] : 0;
      const int act = (s < n_seg && seg_is_action[s]) ? len : 0;
      la[i] = tot.a;  // exclusive within thread
      lb[i] = tot.b;
      tot.a += len;
      tot.b += act;
    }
    ScanPair incl = warp_incl_scan(tot);
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      ScanPair w = warp_tot[lane];
      ScanPair wi = warp_incl_scan(w);
      warp_tot[lane] = ScanPair{wi.a - w.a, wi.b - w.b};  // exclusive over warps
      if (lane == 31) carry_sh = ScanPair{carry.a + wi.a, carry.b + wi.b};
    }
    __syncthreads();
    const ScanPair wex = warp_tot[warp];
    const int ta = carry.a + wex.a + incl.a - tot.a;
    const int tb = carry.b + wex.b + incl.b - tot.b;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      const int s = base + tid * kScanItems + i;
      if (s < n_seg) {
        seg_dst[s] = ta + la[i];
        seg_act_dst[s] = tb + lb[i];
      }
    }
    carry = carry_sh;
    __syncthreads();
  }
  __syncthreads();
  const int total = carry.a, total_act = carry.b;
  for (int b = tid; b < n_traj; b += kScanThreads) {
    const int s0 = traj_seg_off[b], s1 = traj_seg_off[b + 1];
    const int start = s0 < n_seg ? seg_dst[s0] : total;
    for (int s = s0; s < s1; ++s) {
      seg_traj[s] = b;
      seg_tstart[s] = start;
    }
    cu_seqlens[b] = start;
    act_off[b] = s0 < n_seg ? seg_act_dst[s0] : total_act;
  }
  if (tid == 0) {
    cu_seqlens[n_traj] = total;
    act_off[n_traj] = total_act;
  }
}

// Last segment whose packed start <= p (== the segment containing p, see
// empty segments are skipped because a later segment shares the
// same start).
__device__ __forceinline__ int find_segment(const int32_t* __restrict__ seg_dst, int n_seg, int p) {
  int lo = 0, hi = n_seg;  // first index with seg_dst > p
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(seg_dst + mid) <= p) lo = mid + 1;
    else hi = mid;
  }
  return lo - 1;
}

// Block-wide version of find_segment: every round each thread probes one of
// blockDim.x evenly spaced segments of the current bracket; the probes with
// seg_dst <= p form a prefix (seg_dst is non-decreasing), so its length
// (__syncthreads_count) narrows the bracket blockDim.x-fold.
__device__ __forceinline__ int block_find_segment(const int32_t* __restrict__ seg_dst, int n_seg,
                                                  int p) {
  int lo = 0, hi = n_seg;  // answer in [lo, hi); seg_dst[0] = 0 <= p
  while (hi - lo > 1) {
    const int step = (hi - lo + blockDim.x - 1) / blockDim.x;
    const int idx = lo + static_cast<int>(threadIdx.x) * step;
    const int cnt = __syncthreads_count(idx < hi && __ldg(seg_dst + idx) <= p);
    lo += (cnt - 1) * step;
    hi = min(hi, lo + step);
  }
  return lo;
}

constexpr int kScatterThreads = 256;
constexpr int kScatterRounds = 4;
constexpr int kTilePos = kScatterThreads * 4 * kScatterRounds;  // packed positions per CTA
constexpr int kSegCap = 1024;                                    // staged segments per CTA

// Per-segment metadata, staged in shared memory for the segments a CTA's tile
// overlaps (global fallback when a tile spans more than kSegCap segments).
struct SegView {
  const int32_t* dst;
  const int32_t* len;
  const int32_t* src;
  const int32_t* act;
  const int32_t* tstart;  // cu_seqlens of the segment's trajectory
  const int32_t* traj;
  const uint8_t* is_act;
};

template <bool kShared>
__device__ __forceinline__ void scatter_rounds(const SegView v, int s_lo, int n_local,
                                               long long tile_begin, long long tile_end,
                                               const int32_t* __restrict__ pool, int32_t* ids,
                                               uint8_t* mask, int32_t* pos, int32_t* tot,
                                               int32_t* act_idx) {
#pragma unroll 1
  for (int r = 0; r < kScatterRounds; ++r) {
    const long long p0 = tile_begin + (static_cast<long long>(r) * kScatterThreads + threadIdx.x) * 4;
    if (p0 >= tile_end) return;
    // segment of p0: last local segment with dst <= p0
    int lo = 0, hi = n_local;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (v.dst[mid] <= p0) lo = mid + 1;
      else hi = mid;
    }
    int s = lo - 1;
    int o_ids[4], o_pos[4], o_tot[4];
    uint8_t o_m[4];
    const int cnt = tile_end - p0 >= 4 ? 4 : static_cast<int>(tile_end - p0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j >= cnt) break;
      const int p = static_cast<int>(p0) + j;
      while (p >= v.dst[s] + v.len[s]) ++s;
      const int off = p - v.dst[s];
      const uint8_t a = v.is_act[s];
      o_ids[j] = __ldg(pool + v.src[s] + off);
      o_m[j] = a;
      o_tot[j] = v.traj[s];
      o_pos[j] = p - v.tstart[s];
      if (a) act_idx[v.act[s] + off] = p;
    }
    if (cnt == 4) {
      *reinterpret_cast<int4*>(ids + p0) = make_int4(o_ids[0], o_ids[1], o_ids[2], o_ids[3]);
      *reinterpret_cast<int4*>(pos + p0) = make_int4(o_pos[0], o_pos[1], o_pos[2], o_pos[3]);
      *reinterpret_cast<int4*>(tot + p0) = make_int4(o_tot[0], o_tot[1], o_tot[2], o_tot[3]);
      *reinterpret_cast<uchar4*>(mask + p0) = make_uchar4(o_m[0], o_m[1], o_m[2], o_m[3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {  // static indices keep o_*[] in registers
        if (j < cnt) {
          ids[p0 + j] = o_ids[j];
          pos[p0 + j] = o_pos[j];
          tot[p0 + j] = o_tot[j];
          mask[p0 + j] = o_m[j];
        }
      }
    }
  }
  (void)s_lo;
}

__global__ void __launch_bounds__(kScatterThreads)
    pack_scatter_kernel(const int32_t* __restrict__ pool, const int32_t* __restrict__ seg_src_off,
                        const int32_t* __restrict__ seg_len, const uint8_t* __restrict__ seg_is_action,
                        const int32_t* __restrict__ seg_dst, const int32_t* __restrict__ seg_act_dst,
                        const int32_t* __restrict__ seg_traj, const int32_t* __restrict__ seg_tstart,
                        int n_seg, long long n_tokens, int32_t* __restrict__ ids,
                        uint8_t* __restrict__ mask, int32_t* __restrict__ pos,
                        int32_t* __restrict__ tot, int32_t* __restrict__ act_idx) {
  __shared__ int32_t sh_dst[kSegCap], sh_len[kSegCap], sh_src[kSegCap], sh_act[kSegCap],
      sh_ts[kSegCap], sh_traj[kSegCap];
  __shared__ uint8_t sh_isa[kSegCap];
  __shared__ int sh_range[2];
  const long long tile_begin = static_cast<long long>(blockIdx.x) * kTilePos;
  const long long tile_end = min(n_tokens, tile_begin + kTilePos);
  // Segments holding the tile's first and last position: a block-wide
  // 256-ary search (one probe per thread per round, 2 rounds up to 65 k
  // segments) instead of one thread's 14 dependent loads.
  const int s_first = block_find_segment(seg_dst, n_seg, static_cast<int>(tile_begin));
  const int s_last = block_find_segment(seg_dst, n_seg, static_cast<int>(tile_end - 1));
  (void)sh_range;
  const int s_lo = s_first, n_local = s_last - s_lo + 1;
  if (n_local <= kSegCap) {
    for (int i = threadIdx.x; i < n_local; i += kScatterThreads) {
      const int s = s_lo + i;
      sh_dst[i] = seg_dst[s];
      sh_len[i] = seg_len[s];
      sh_src[i] = seg_src_off[s];
      sh_act[i] = seg_act_dst[s];
      sh_ts[i] = seg_tstart[s];
      sh_traj[i] = seg_traj[s];
      sh_isa[i] = seg_is_action[s];
    }
    __syncthreads();
    const SegView v{sh_dst, sh_len, sh_src, sh_act, sh_ts, sh_traj, sh_isa};
    scatter_rounds<true>(v, s_lo, n_local, tile_begin, tile_end, pool, ids, mask, pos, tot,
                         act_idx);
  } else {
    const SegView v{seg_dst, seg_len, seg_src_off, seg_act_dst, seg_tstart, seg_traj, seg_is_action};
    scatter_rounds<false>(v, 0, n_seg, tile_begin, tile_end, pool, ids, mask, pos, tot, act_idx);
  }
}

__global__ void pack_padded_kernel(const int32_t* __restrict__ ids, const uint8_t* __restrict__ mask,
                                   const int32_t* __restrict__ cu, int n_traj, int lmax, int pad_id,
                                   int32_t* __restrict__ ids_out, uint8_t* __restrict__ mask_out,
                                   int32_t* __restrict__ pos_out) {
  const int b = blockIdx.y;
  const int start = cu[b], len = cu[b + 1] - start;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < lmax; j += gridDim.x * blockDim.x) {
    const long long o = static_cast<long long>(b) * lmax + j;
    const bool in = j < len;
    ids_out[o] = in ? ids[start + j] : pad_id;
    mask_out[o] = in ? mask[start + j] : 0;
    pos_out[o] = in ? j : 0;
  }
}

}  // namespace
}  // namespace tl

extern "C" size_t tl_pack_workspace_bytes(int32_t n_traj, int32_t n_seg) {
  (void)n_traj;
  tl::Workspace w{nullptr, 0};
  for (int i = 0; i < 4; ++i) w.take<int32_t>(n_seg);
  return w.used + 256;
}

extern "C" int tl_pack_varlen(const int32_t* token_pool, const int32_t* seg_src_off,
                              const int32_t* seg_len, const uint8_t* seg_is_action,
                              const int32_t* traj_seg_off, int32_t n_traj, int32_t n_seg,
                              int64_t n_tokens, int32_t* input_ids, uint8_t* loss_mask,
                              int32_t* position_ids, int32_t* traj_of_token, int32_t* cu_seqlens,
                              int32_t* act_off, int32_t* act_idx, void* workspace,
                              size_t workspace_bytes, tl_stream_t stream) {
  TL_REQUIRE(n_traj >= 0 && n_seg >= 0 && n_tokens >= 0, TL_ERR_INVALID_ARG, "negative sizes");
  TL_REQUIRE(n_tokens < (1LL << 31), TL_ERR_UNSUPPORTED, "n_tokens must fit int32");
  tl::Workspace w{static_cast<char*>(workspace), workspace_bytes};
  int32_t* seg_dst = w.take<int32_t>(n_seg);
  int32_t* seg_act = w.take<int32_t>(n_seg);
  int32_t* seg_traj = w.take<int32_t>(n_seg);
  int32_t* seg_tstart = w.take<int32_t>(n_seg);
  TL_REQUIRE(w.ok(), TL_ERR_WORKSPACE, "pack workspace too small (%zu < %zu)", workspace_bytes,
             w.used);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  tl::ProfScope prof(tl::PROF_PACK, st);
  tl::pack_scan_kernel<<<1, tl::kScanThreads, 0, st>>>(seg_len, seg_is_action, traj_seg_off, n_traj,
                                                       n_seg, seg_dst, seg_act, seg_traj,
                                                       seg_tstart, cu_seqlens, act_off);
  TL_LAUNCH_CHECK();
  tl::count_launch();
  if (n_tokens > 0) {
    const int grid = static_cast<int>((n_tokens + tl::kTilePos - 1) / tl::kTilePos);
    tl::pack_scatter_kernel<<<grid, tl::kScatterThreads, 0, st>>>(
        token_pool, seg_src_off, seg_len, seg_is_action, seg_dst, seg_act, seg_traj, seg_tstart,
        n_seg, n_tokens, input_ids, loss_mask, position_ids, traj_of_token, act_idx);
    TL_LAUNCH_CHECK();
    tl::count_launch();
  }
  return TL_OK;
}

extern "C" int tl_pack_padded(const int32_t* input_ids, const uint8_t* loss_mask,
                              const int32_t* cu_seqlens, int32_t n_traj, int32_t lmax,
                              int32_t pad_id, int32_t* ids_out, uint8_t* mask_out,
                              int32_t* pos_out, tl_stream_t stream) {
  TL_REQUIRE(n_traj >= 0 && lmax >= 0, TL_ERR_INVALID_ARG, "negative sizes");
  if (n_traj == 0 || lmax == 0) return TL_OK;
  TL_REQUIRE(n_traj <= 65535, TL_ERR_UNSUPPORTED, "n_traj > 65535");
  dim3 grid((lmax + 255) / 256 > 64 ? 64 : (lmax + 255) / 256, n_traj);
  tl::pack_padded_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      input_ids, loss_mask, cu_seqlens, n_traj, lmax, pad_id, ids_out, mask_out, pos_out);
  TL_LAUNCH_CHECK();
  tl::count_launch();
  return TL_OK;
}
