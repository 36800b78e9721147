// Cluster-parallel top-K selection (SURVEY.md §8(a) a9 RPN pre-NMS top-k, a11 final
// top-k rows; include/gemel.h TOPK / RPN_LEVEL give the order: key descending, ties by
// lower row index -- a total order, so the selection is unique and bit-exact).
//
// One thread-block cluster of SEL_CS CTAs per (task, frame).  CTA r stages the order
// keys of its contiguous slice of rows in shared memory once, then
//   1. four 8-bit radix passes: a per-CTA histogram (warp-aggregated smem atomics --
//      scores cluster in a few bins), summed over the cluster through distributed
//      shared memory; every CTA derives the same threshold key T and the count of rows
//      equal to T that are taken;
//   2. compaction: the CTA's rows above T (any order) and its lowest-index rows equal to
//      T (index-ordered block scan, stopping once enough are found);
//   3. the CTAs' counts are exchanged (DSMEM), and each CTA writes its survivors as
//      packed (~key << 32 | row) into the LEADER's shared memory -- the rows equal to T
//      in CTA order, so the lowest indices overall are the ones taken;
//   4. the leader sorts the <= SEL_KMAX packed survivors (bitonic, ascending = key
//      descending, row ascending).
// Work per frame is spread over SEL_CS SMs instead of one (the previous one-CTA-per-frame
// kernels ran 16-80 CTAs on a 148-SM GPU and serialised 90 000-row frames on one SM).
#pragma once
#include <cooperative_groups.h>
#include <cstdint>

namespace gemel {
namespace sel {

namespace cg = cooperative_groups;

constexpr int SEL_CS = 8;          // CTAs per cluster (portable cluster size)
constexpr int SEL_THREADS = 512;
constexpr int SEL_KMAX = 1024;     // K <= 1024 (registry-enforced)
constexpr int SEL_STAGE_CAP = 40960;   // keys staged per CTA (160 KB); larger slices re-read the source

__device__ __forceinline__ uint32_t order_key(float f) {   // order-preserving float -> uint32
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

struct Shared {
  int hist[2][256];                 // this CTA's histogram (double-buffered across passes)
  int tot[256];                     // cluster-summed histogram
  unsigned long long out[SEL_KMAX]; // leader: the packed survivors, sorted at the end
  int above[SEL_KMAX];              // this CTA's rows above T (slice-local)
  int eq[SEL_KMAX];                 // this CTA's first rows equal to T (slice-local, index order)
  int warp_tot[33];
  int n_above, n_eq;                // published to the cluster
  uint32_t prefix;
  int remaining;
};

// exclusive prefix of a per-thread flag over the block (SEL_THREADS); returns the total
__device__ __forceinline__ int block_scan(bool flag, int* warp_tot, int& excl) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned b = __ballot_sync(0xffffffffu, flag);
  __syncthreads();
  if (lane == 0) warp_tot[wid] = __popc(b);
  __syncthreads();
  if (wid == 0) {
    const int v = lane < SEL_THREADS / 32 ? warp_tot[lane] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane < SEL_THREADS / 32) warp_tot[lane] = incl - v;
    if (lane == 31) warp_tot[32] = incl;
  }
  __syncthreads();
  excl = warp_tot[wid] + __popc(b & ((1u << lane) - 1u));
  return warp_tot[32];
}

// Selects the min(K, n) best rows of one frame.  key_at(i) -> order key of row i.
// Every CTA of the cluster calls it with the same n, K.  Returns the survivor count in
// the leader (S.out[0..kt) sorted, S.out[kt..SEL_KMAX) = ~0) and -1 in the other CTAs,
// which must not touch the cluster afterwards.
template <class KeyAt>
__device__ int cluster_select(const KeyAt& key_at, int n, int K, Shared& S, uint32_t* keys) {
  cg::cluster_group cl = cg::this_cluster();
  const int r = int(cl.block_rank());
  const int tid = threadIdx.x, lane = tid & 31;
  const int chunk = ((n + SEL_CS - 1) / SEL_CS + 31) & ~31;
  const int lo = min(n, r * chunk), cnt = min(n, lo + chunk) - lo;
  const bool staged = chunk <= SEL_STAGE_CAP;
  if (staged) {
#pragma unroll 4
    for (int j = tid; j < cnt; j += SEL_THREADS) keys[j] = key_at(lo + j);   // 4 loads in flight
  }
  auto key = [&](int j) { return staged ? keys[j] : key_at(lo + j); };
  const int kt = min(K, n);

  // 1. radix select of the kt-th largest key over the cluster
  uint32_t prefix = 0, mask = 0;
  int remaining = kt;
  for (int pass = 0; pass < 4 && kt > 0; ++pass) {
    const int shift = 24 - 8 * pass;
    int* h = S.hist[pass & 1];
    for (int i = tid; i < 256; i += SEL_THREADS) h[i] = 0;
    __syncthreads();
    for (int base = 0; base < cnt; base += SEL_THREADS) {   // warp-uniform trip count
      const int j = base + tid;
      const uint32_t k = j < cnt ? key(j) : 0u;
      const int bin = (j < cnt && (k & mask) == prefix) ? int((k >> shift) & 255u) : 256;
      const unsigned peers = __match_any_sync(0xffffffffu, bin);
      if (bin < 256 && lane == __ffs(peers) - 1) atomicAdd(&h[bin], __popc(peers));
    }
    cl.sync();   // every CTA's histogram of this pass is complete
    for (int b = tid; b < 256; b += SEL_THREADS) {
      int s = 0;
#pragma unroll
      for (int q = 0; q < SEL_CS; ++q) s += cl.map_shared_rank(h, q)[b];
      S.tot[b] = s;
    }
    __syncthreads();
    if (tid < 32) {   // bins from the top: lane l owns bins 255-8l .. 248-8l
      int v[8], sum = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) { v[j] = S.tot[255 - 8 * lane - j]; sum += v[j]; }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const int excl = incl - sum;
      if (excl < remaining && incl >= remaining) {   // exactly one lane
        int cum = excl;
        for (int j = 0; j < 8; ++j) {
          if (cum + v[j] >= remaining) {
            S.prefix = prefix | (uint32_t(255 - 8 * lane - j) << shift);
            S.remaining = remaining - cum;
            break;
          }
          cum += v[j];
        }
      }
    }
    __syncthreads();
    prefix = S.prefix;
    remaining = S.remaining;
    mask |= 255u << shift;
    // the other buffer is cleared next pass: every CTA finished reading it before this
    // pass's cluster barrier
  }
  const uint32_t thr = prefix;
  const int need_eq = kt > 0 ? remaining : 0;

  // 2. this CTA's survivors: rows above T (warp-aggregated atomics), first rows equal to T
  if (tid == 0) { S.n_above = 0; S.n_eq = 0; }
  __syncthreads();
  if (kt > 0) {
    for (int base = 0; base < cnt; base += SEL_THREADS) {
      const int j = base + tid;
      const bool above = j < cnt && key(j) > thr;
      const unsigned ma = __ballot_sync(0xffffffffu, above);
      int b0 = 0;
      if (lane == 0 && ma) b0 = atomicAdd(&S.n_above, __popc(ma));
      b0 = __shfl_sync(0xffffffffu, b0, 0);
      if (above) S.above[b0 + __popc(ma & ((1u << lane) - 1u))] = j;
    }
    int seen = 0;
    for (int base = 0; base < cnt && seen < need_eq; base += SEL_THREADS) {   // block-uniform
      const int j = base + tid;
      const bool eq = j < cnt && key(j) == thr;
      int ex;
      const int tot = block_scan(eq, S.warp_tot, ex);
      if (eq && seen + ex < need_eq) S.eq[seen + ex] = j;
      seen += tot;
    }
    if (tid == 0) S.n_eq = min(seen, need_eq);
  }
  cl.sync();   // counts published

  // 3. offsets over the cluster; survivors into the leader's buffer
  int above_off = 0, tot_above = 0, eq_before = 0;
  for (int q = 0; q < SEL_CS; ++q) {
    const Shared* R = cl.map_shared_rank(&S, q);
    const int na = R->n_above, ne = R->n_eq;
    if (q < r) { above_off += na; eq_before += ne; }
    tot_above += na;
  }
  const int take = max(0, min(S.n_eq, need_eq - eq_before));
  unsigned long long* dst = cl.map_shared_rank(S.out, 0);
  for (int i = tid; i < S.n_above; i += SEL_THREADS) {
    const int j = S.above[i];
    dst[above_off + i] = (uint64_t(~key(j)) << 32) | uint32_t(lo + j);
  }
  for (int i = tid; i < take; i += SEL_THREADS)
    dst[tot_above + eq_before + i] = (uint64_t(~thr) << 32) | uint32_t(lo + S.eq[i]);
  cl.sync();   // the leader's buffer is complete; no DSMEM access after this
  if (r != 0) return -1;

  // 4. leader: ascending bitonic sort of SEL_KMAX packed keys (padding = ~0 sorts last)
  for (int i = kt + tid; i < SEL_KMAX; i += SEL_THREADS) S.out[i] = ~0ull;
  for (int k = 2; k <= SEL_KMAX; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      __syncthreads();
      for (int i = tid; i < SEL_KMAX; i += SEL_THREADS) {
        const int l = i ^ j;
        if (l > i) {
          const unsigned long long x = S.out[i], y = S.out[l];
          if ((x > y) == ((i & k) == 0)) { S.out[i] = y; S.out[l] = x; }
        }
      }
    }
  __syncthreads();
  return kt;
}

__host__ __device__ constexpr size_t stage_bytes(int max_rows) {
  return size_t(((max_rows + SEL_CS - 1) / SEL_CS + 31) & ~31) <= size_t(SEL_STAGE_CAP)
             ? size_t(((max_rows + SEL_CS - 1) / SEL_CS + 31) & ~31) * 4
             : 0;
}

}  // namespace sel
}  // namespace gemel
