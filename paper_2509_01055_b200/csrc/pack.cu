// K1 — trajectory packer.
//
// Reference semantics: trajectory.flatten (trajectory.py:154-159) concatenates
// the per-segment token lists without re-tokenising; trajectory.action_mask
// (trajectory.py:162-167) is 1 on action tokens, 0 on observation tokens;
// rl.loss.token_records (loss.py:76-100) zips them per token.  Here the whole
// batch is packed at once into varlen (cu_seqlens) form plus the action-row
// index the LM head runs on.
//
//  pack_scan_kernel    single-pass decoupled look-back scan over the segment
//                      table: 512 segments per CTA (tiles taken in order
//                      from a ticket counter), exclusive prefix sums of the
//                      (token, action-token) lengths -> packed offset and
//                      action offset of every segment.
//  pack_scatter_kernel token-parallel: every thread owns 4 consecutive packed
//                      positions (16-byte vector stores of ids / positions /
//                      trajectory ids, 4-byte mask stores), finds its segment
//                      in the CTA's staged segment window, and copies from the
//                      (arbitrarily ordered) token pool.  Launched with
//                      programmatic dependent launch so its CTAs are resident
//                      and waiting while the scan runs; the first CTAs also
//                      write cu_seqlens / act_off.
// Optional per-trajectory drop bits (error / timed-out episodes whose
// gradients the paper masks): a dropped trajectory keeps its
// tokens but all of them get loss_mask 0, so it has no action rows (no LM-head
// work, zero gradient) and counts as an all-observation trajectory in the loss
// (skipped, still counted in its group: loss.py:173-174, :193).
#include <cuda/atomic>

#include "tl_common.cuh"

namespace tl {
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 2;  // 512-segment tiles: scan 9.7 -> 5.1 us at C2 vs 2,048 (gpu_s3n)
constexpr int kScanTile = kScanThreads * kScanItems;  // segments per CTA

// Look-back status word of a scan tile: flag (2 bits: 0 not ready,
// 1 aggregate, 2 inclusive prefix) | token sum (31 bits) | action sum (31).
// Both sums are < 2^31 (n_tokens < 2^31 is checked on the host side).
constexpr unsigned long long kFlagAgg = 1ull, kFlagIncl = 2ull;
__device__ __forceinline__ unsigned long long status_word(unsigned long long flag, int a, int b) {
  return (flag << 62) | (static_cast<unsigned long long>(a) << 31) | static_cast<unsigned long long>(b);
}

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

// Last index i in [0, n) with arr[i] <= key (arr non-decreasing, arr[0] <=
// key): every round each thread of the block probes one of blockDim.x evenly
// spaced entries of the bracket; the probes <= key form a prefix whose length
// (__syncthreads_count) narrows the bracket blockDim.x-fold (2 rounds up to
// 65 k entries).  All threads must call it.
__device__ __forceinline__ int block_find_last_le(const int32_t* __restrict__ arr, int n, int key) {
  int lo = 0, hi = n;  // answer in [lo, hi)
  while (hi - lo > 1) {
    const int step = (hi - lo + blockDim.x - 1) / blockDim.x;
    const int idx = lo + static_cast<int>(threadIdx.x) * step;
    const int cnt = __syncthreads_count(idx < hi && __ldg(arr + idx) <= key);
    lo += (cnt - 1) * step;
    hi = min(hi, lo + step);
  }
  return lo;
}

// block_find_last_le for two keys k0 <= k1 at once (one probe pass per round
// serves both brackets): returns {last <= k0, last <= k1}.
__device__ __forceinline__ int2 block_find_last_le2(const int32_t* __restrict__ arr, int n, int k0,
                                                    int k1) {
  int lo0 = 0, hi0 = n, lo1 = 0, hi1 = n;
  while (hi0 - lo0 > 1 || hi1 - lo1 > 1) {
    const int st0 = (hi0 - lo0 + blockDim.x - 1) / blockDim.x;
    const int st1 = (hi1 - lo1 + blockDim.x - 1) / blockDim.x;
    const int i0 = lo0 + static_cast<int>(threadIdx.x) * st0;
    const int i1 = lo1 + static_cast<int>(threadIdx.x) * st1;
    const bool p0 = hi0 - lo0 > 1 && i0 < hi0 && __ldg(arr + i0) <= k0;
    const bool p1 = hi1 - lo1 > 1 && i1 < hi1 && __ldg(arr + i1) <= k1;
    const int c0 = __syncthreads_count(p0);
    const int c1 = __syncthreads_count(p1);
    if (hi0 - lo0 > 1) {
      lo0 += (c0 - 1) * st0;
      hi0 = min(hi0, lo0 + st0);
    }
    if (hi1 - lo1 > 1) {
      lo1 += (c1 - 1) * st1;
      hi1 = min(hi1, lo1 + st1);
    }
  }
  return make_int2(lo0, lo1);
}

// Trajectory owning segment s: last b in [0, n_traj) with traj_seg_off[b] <= s.
__device__ __forceinline__ int traj_of_segment(const int32_t* __restrict__ tso, int n_traj, int s) {
  int lo = 0, hi = n_traj;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(tso + mid) <= s) lo = mid;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(kScanThreads)
    pack_scan_kernel(const int32_t* __restrict__ seg_len, const uint8_t* __restrict__ seg_is_action,
                     const int32_t* __restrict__ traj_seg_off, const uint8_t* __restrict__ traj_drop,
                     int n_traj, int n_seg, int32_t* __restrict__ seg_dst,
                     int32_t* __restrict__ seg_act_dst, unsigned long long* __restrict__ status,
                     int* __restrict__ ticket, int32_t* __restrict__ cu_seqlens,
                     int32_t* __restrict__ act_off) {
  // let the scatter grid get resident (it waits in griddepcontrol.wait)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ int sh_len[kScanTile];
  __shared__ ScanPair warp_tot[kScanThreads / 32];
  __shared__ int sh_tile;
  __shared__ ScanPair sh_prefix;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // tiles in dispatch order (a ticket) unless every tile is co-resident
  if (tid == 0) sh_tile = ticket ? atomicAdd(ticket, 1) : static_cast<int>(blockIdx.x);
  __syncthreads();
  const int tile = sh_tile;
  const int base = tile * kScanTile;
  // coalesced staging: token length and action length (bit 31 = action)
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int s = base + i * kScanThreads + tid;
    int v = 0;
    if (s < n_seg) {
      const int len = seg_len[s];
      bool act = seg_is_action[s] != 0;
      if (act && traj_drop) act = traj_drop[traj_of_segment(traj_seg_off, n_traj, s)] == 0;
      v = act ? (len | static_cast<int>(0x80000000u)) : len;
    }
    sh_len[i * kScanThreads + tid] = v;
  }
  __syncthreads();
  int la[kScanItems], lb[kScanItems];
  ScanPair tot{0, 0};
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int v = sh_len[tid * kScanItems + i];
    const int len = v & 0x7fffffff;
    la[i] = tot.a;  // exclusive within the thread
    lb[i] = tot.b;
    tot.a += len;
    tot.b += v < 0 ? len : 0;
  }
  const ScanPair incl = warp_incl_scan(tot);
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const ScanPair w = lane < kScanThreads / 32 ? warp_tot[lane] : ScanPair{0, 0};
    const ScanPair wi = warp_incl_scan(w);
    if (lane < kScanThreads / 32) warp_tot[lane] = ScanPair{wi.a - w.a, wi.b - w.b};
    // this tile's aggregate, broadcast from the last warp-total lane
    const int agg_a = __shfl_sync(0xffffffffu, wi.a, kScanThreads / 32 - 1);
    const int agg_b = __shfl_sync(0xffffffffu, wi.b, kScanThreads / 32 - 1);
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> me(status[tile]);
    if (lane == 0)
      me.store(status_word(tile == 0 ? kFlagIncl : kFlagAgg, agg_a, agg_b),
               cuda::memory_order_release);
    // warp-parallel look-back: lane l waits on tile (j - l) of a 32-tile
    // window; the nearest inclusive prefix ends the walk
    ScanPair pre{0, 0};
    for (int j = tile - 1; j >= 0; j -= 32) {
      const int t = j - lane;
      unsigned long long sw = status_word(kFlagAgg, 0, 0);
      if (t >= 0) {
        cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> st(status[t]);
        while (((sw = st.load(cuda::memory_order_acquire)) >> 62) == 0) {
        }
      }
      const unsigned incl_mask = __ballot_sync(0xffffffffu, t >= 0 && (sw >> 62) == kFlagIncl);
      const int stop = incl_mask ? __ffs(incl_mask) - 1 : 31;  // nearest inclusive lane
      int va = lane <= stop && t >= 0 ? static_cast<int>((sw >> 31) & 0x7fffffffull) : 0;
      int vb = lane <= stop && t >= 0 ? static_cast<int>(sw & 0x7fffffffull) : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        va += __shfl_xor_sync(0xffffffffu, va, o);
        vb += __shfl_xor_sync(0xffffffffu, vb, o);
      }
      pre.a += va;
      pre.b += vb;
      if (incl_mask) break;
    }
    if (lane == 0) {
      if (tile > 0)
        me.store(status_word(kFlagIncl, pre.a + agg_a, pre.b + agg_b), cuda::memory_order_release);
      sh_prefix = pre;
      if (base + kScanTile >= n_seg) {  // last tile: the batch totals
        cu_seqlens[n_traj] = pre.a + agg_a;
        act_off[n_traj] = pre.b + agg_b;
      }
    }
  }
  __syncthreads();
  const ScanPair wex = warp_tot[warp];
  const ScanPair pre = sh_prefix;
  const int ta = pre.a + wex.a + incl.a - tot.a;
  const int tb = pre.b + wex.b + incl.b - tot.b;
  // back through shared memory for coalesced stores
  int* sh_b = reinterpret_cast<int*>(sh_len);  // reuse: a first, then b
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) sh_b[tid * kScanItems + i] = ta + la[i];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int s = base + i * kScanThreads + tid;
    if (s < n_seg) seg_dst[s] = sh_b[i * kScanThreads + tid];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) sh_b[tid * kScanItems + i] = tb + lb[i];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int s = base + i * kScanThreads + tid;
    if (s < n_seg) seg_act_dst[s] = sh_b[i * kScanThreads + tid];
  }
}

constexpr int kScatterThreads = 256;  // 128 x 8 rounds: same; 512 x 2: +28 % (gpu_s3o)
constexpr int kScatterRounds = 4;  // 2: +9 %, 8: +9 %, 16: same (gpu_s3f, s3o)
constexpr int kTilePos = kScatterThreads * 4 * kScatterRounds;  // packed positions per CTA
constexpr int kSegCap = 1024;                                    // staged segments per CTA
constexpr int kTrajCap = 512;                                    // staged trajectories per CTA

// Segment metadata of the CTA's tile window, staged in shared memory.
struct SegWindow {
  int32_t dst[kSegCap], len[kSegCap], src[kSegCap], act[kSegCap], traj[kSegCap], tstart[kSegCap];
  uint8_t is_act[kSegCap];
};

__global__ void __launch_bounds__(kScatterThreads)
    pack_scatter_kernel(const int32_t* __restrict__ pool, const int32_t* __restrict__ seg_src_off,
                        const int32_t* __restrict__ seg_len, const uint8_t* __restrict__ seg_is_action,
                        const int32_t* __restrict__ traj_seg_off, const uint8_t* __restrict__ traj_drop,
                        const int32_t* seg_dst, const int32_t* seg_act_dst, int n_traj, int n_seg,
                        long long n_tokens, int32_t* __restrict__ ids, uint8_t* __restrict__ mask,
                        int32_t* __restrict__ pos, int32_t* __restrict__ tot,
                        int32_t* __restrict__ act_idx, int32_t* cu_seqlens,
                        int32_t* __restrict__ act_off) {
  __shared__ SegWindow w;
  __shared__ int32_t sh_toff[kTrajCap + 1], sh_tstart[kTrajCap];
  // everything below reads the scan's outputs
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // cu_seqlens / act_off: trajectory b starts at its first segment's offsets
  // (an empty trajectory at the next segment's, or at the totals)
  for (int b = blockIdx.x * kScatterThreads + threadIdx.x; b < n_traj;
       b += gridDim.x * kScatterThreads) {
    const int s0 = traj_seg_off[b];
    cu_seqlens[b] = s0 < n_seg ? seg_dst[s0] : cu_seqlens[n_traj];
    act_off[b] = s0 < n_seg ? seg_act_dst[s0] : act_off[n_traj];
  }
  const long long tile_begin = static_cast<long long>(blockIdx.x) * kTilePos;
  if (tile_begin >= n_tokens) return;
  const long long tile_end = min(n_tokens, tile_begin + kTilePos);
  // segment window [s_lo, s_hi] holding the tile's first and last positions
  const int2 sr = block_find_last_le2(seg_dst, n_seg, static_cast<int>(tile_begin),
                                      static_cast<int>(tile_end - 1));
  const int2 br = block_find_last_le2(traj_seg_off, n_traj, sr.x, sr.y);
  const int s_lo = sr.x, s_hi = sr.y, b_lo = br.x, b_hi = br.y;
  const int n_local = s_hi - s_lo + 1, n_tl = b_hi - b_lo + 1;
  const bool staged = n_local <= kSegCap && n_tl <= kTrajCap;
  if (staged) {
    for (int j = threadIdx.x; j <= n_tl; j += kScatterThreads)
      sh_toff[j] = j < n_tl ? traj_seg_off[b_lo + j] : n_seg;  // sentinel: no later start
    for (int j = threadIdx.x; j < n_tl; j += kScatterThreads) {
      const int s0 = traj_seg_off[b_lo + j];
      sh_tstart[j] = s0 < n_seg ? seg_dst[s0] : cu_seqlens[n_traj];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n_local; i += kScatterThreads) {
      const int s = s_lo + i;
      int lo = 0, hi = n_tl;  // last local trajectory starting at or before s
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (sh_toff[mid] <= s) lo = mid;
        else hi = mid;
      }
      w.dst[i] = seg_dst[s];
      w.len[i] = seg_len[s];
      w.src[i] = seg_src_off[s];
      w.act[i] = seg_act_dst[s];
      w.traj[i] = b_lo + lo;
      w.tstart[i] = sh_tstart[lo];
      w.is_act[i] = seg_is_action[s] && (!traj_drop || !traj_drop[b_lo + lo]);
    }
    __syncthreads();
  }
#pragma unroll 2  // 4: +3 % (gpu_s3o)
  for (int r = 0; r < kScatterRounds; ++r) {
    const long long p0 = tile_begin + (static_cast<long long>(r) * kScatterThreads + threadIdx.x) * 4;
    if (p0 >= tile_end) break;
    const int cnt = tile_end - p0 >= 4 ? 4 : static_cast<int>(tile_end - p0);
    int o_ids[4], o_pos[4], o_tot[4];
    uint8_t o_m[4];
    if (staged) {
      int lo = 0, hi = n_local;  // first local segment starting after p0
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (w.dst[mid] <= p0) lo = mid + 1;
        else hi = mid;
      }
      int s = lo - 1;
      const int pp = static_cast<int>(p0);
      if (cnt == 4 && pp + 4 <= w.dst[s] + w.len[s]) {
        // common case: the 4 positions lie in one segment
        const int off = pp - w.dst[s];
        const int32_t* src = pool + w.src[s] + off;
        const int ps = pp - w.tstart[s], tr = w.traj[s];
        const uint8_t act = w.is_act[s];
        *reinterpret_cast<int4*>(ids + p0) =
            make_int4(__ldg(src), __ldg(src + 1), __ldg(src + 2), __ldg(src + 3));
        *reinterpret_cast<int4*>(pos + p0) = make_int4(ps, ps + 1, ps + 2, ps + 3);
        *reinterpret_cast<int4*>(tot + p0) = make_int4(tr, tr, tr, tr);
        *reinterpret_cast<uchar4*>(mask + p0) = make_uchar4(act, act, act, act);
        if (act) {
          int32_t* ai = act_idx + w.act[s] + off;
          ai[0] = pp;
          ai[1] = pp + 1;
          ai[2] = pp + 2;
          ai[3] = pp + 3;
        }
        continue;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j >= cnt) break;
        const int p = pp + j;
        while (p >= w.dst[s] + w.len[s]) ++s;
        const int off = p - w.dst[s];
        const uint8_t act = w.is_act[s];
        o_ids[j] = __ldg(pool + w.src[s] + off);
        o_m[j] = act;
        o_tot[j] = w.traj[s];
        o_pos[j] = p - w.tstart[s];
        if (act) act_idx[w.act[s] + off] = p;
      }
    } else {  // window too wide for shared memory (many tiny segments): global
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j >= cnt) break;
        const int p = static_cast<int>(p0) + j;
        int lo = 0, hi = n_seg;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (seg_dst[mid] <= p) lo = mid + 1;
          else hi = mid;
        }
        int s = lo - 1;
        while (p >= seg_dst[s] + seg_len[s]) ++s;
        const int b = traj_of_segment(traj_seg_off, n_traj, s);
        const int off = p - seg_dst[s];
        const uint8_t act = seg_is_action[s] && (!traj_drop || !traj_drop[b]);
        o_ids[j] = __ldg(pool + seg_src_off[s] + off);
        o_m[j] = act;
        o_tot[j] = b;
        o_pos[j] = p - seg_dst[traj_seg_off[b]];
        if (act) act_idx[seg_act_dst[s] + off] = p;
      }
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
  w.take<int32_t>(n_seg);
  w.take<int32_t>(n_seg);
  w.take<unsigned long long>((n_seg + tl::kScanTile - 1) / tl::kScanTile + 1);  // status + ticket
  return w.used + 256;
}

extern "C" int tl_pack_varlen(const int32_t* token_pool, const int32_t* seg_src_off,
                              const int32_t* seg_len, const uint8_t* seg_is_action,
                              const int32_t* traj_seg_off, const uint8_t* traj_drop, int32_t n_traj,
                              int32_t n_seg, int64_t n_tokens, int32_t* input_ids, uint8_t* loss_mask,
                              int32_t* position_ids, int32_t* traj_of_token, int32_t* cu_seqlens,
                              int32_t* act_off, int32_t* act_idx, void* workspace,
                              size_t workspace_bytes, tl_stream_t stream) {
  TL_REQUIRE(n_traj >= 0 && n_seg >= 0 && n_tokens >= 0, TL_ERR_INVALID_ARG, "negative sizes");
  TL_REQUIRE(n_tokens < (1LL << 31), TL_ERR_UNSUPPORTED, "n_tokens must fit int32");
  tl::Workspace w{static_cast<char*>(workspace), workspace_bytes};
  int32_t* seg_dst = w.take<int32_t>(n_seg);
  int32_t* seg_act = w.take<int32_t>(n_seg);
  const int n_tiles = (n_seg + tl::kScanTile - 1) / tl::kScanTile;
  unsigned long long* status = w.take<unsigned long long>(n_tiles + 1);
  int* ticket = reinterpret_cast<int*>(status + n_tiles);
  TL_REQUIRE(w.ok(), TL_ERR_WORKSPACE, "pack workspace too small (%zu < %zu)", workspace_bytes,
             w.used);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  tl::ProfScope prof(tl::PROF_PACK, st);
  if (n_seg == 0) {  // no segments: every trajectory is empty
    TL_CUDA_TRY(cudaMemsetAsync(cu_seqlens, 0, (n_traj + 1) * sizeof(int32_t), st));
    TL_CUDA_TRY(cudaMemsetAsync(act_off, 0, (n_traj + 1) * sizeof(int32_t), st));
    return TL_OK;
  }
  TL_CUDA_TRY(cudaMemsetAsync(status, 0, (n_tiles + 1) * sizeof(unsigned long long), st));
  // at most one tile per SM: all tiles are resident at once, so the look-back
  // cannot wait on an unscheduled tile and blockIdx order is enough
  const bool coresident = n_tiles <= tl::num_sms();
  tl::pack_scan_kernel<<<n_tiles, tl::kScanThreads, 0, st>>>(
      seg_len, seg_is_action, traj_seg_off, traj_drop, n_traj, n_seg, seg_dst, seg_act, status,
      coresident ? nullptr : ticket, cu_seqlens, act_off);
  TL_LAUNCH_CHECK();
  tl::count_launch();
  const long long tiles = (n_tokens + tl::kTilePos - 1) / tl::kTilePos;
  const long long traj_ctas = (n_traj + tl::kScatterThreads - 1) / tl::kScatterThreads;
  const long long grid = tiles > traj_ctas ? tiles : (traj_ctas > 0 ? traj_ctas : 1);
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(static_cast<unsigned>(grid));
  lc.blockDim = dim3(tl::kScatterThreads);
  lc.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  TL_CUDA_TRY(cudaLaunchKernelEx(&lc, tl::pack_scatter_kernel, token_pool, seg_src_off, seg_len,
                                 seg_is_action, traj_seg_off, traj_drop,
                                 static_cast<const int32_t*>(seg_dst),
                                 static_cast<const int32_t*>(seg_act), n_traj, n_seg,
                                 static_cast<long long>(n_tokens), input_ids, loss_mask,
                                 position_ids, traj_of_token, act_idx, cu_seqlens, act_off));
  tl::count_launch();
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
