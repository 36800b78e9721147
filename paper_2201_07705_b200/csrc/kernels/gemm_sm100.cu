// K1/K2: grouped implicit-GEMM convolution + linear on 5th-gen tensor cores.
//
// Persistent, warp-specialised sm_100a kernel (one CTA per SM, 352 threads), in two
// variants: gemel_gemm_sm100 (cta_group::1, 128-row tiles) and gemel_gemm_sm100_pair
// (cta_group::2: a cluster of 2 CTAs on one TPC computes a 256-row tile -- each CTA
// loads its own 128 rows of A and HALF of the N rows of B, the leader issues
// tcgen05.mma.cta_group::2 (M = 256) reading both CTAs' shared memory, each CTA's
// TMEM holds its 128 accumulator rows; operand bytes per FLOP drop by 1/3 at N = 256,
// which is what bounds the 1-CTA kernel: the L2 -> SM operand stream).
//   warp 10     : tile scheduler.  Tiles are taken from a global queue in topological
//                 order, decoded ONCE into a shared-memory ring of TILE_RING slots (the
//                 problem's scalars, its producers' counters and the last member segment
//                 cached in shared memory), and published only after every producer
//                 m-tile band it reads (conv input or residual rows) has completed, so a
//                 whole chain of dependent layers runs in ONE launch and independent
//                 chains (other models) overlap as a wavefront.
//   warp 0      : TMA producer.  A tiles from the NHWC bf16 activation via TMA *im2col*
//                 mode (128 output pixels x one (tap, channel-chunk) per box; conv padding
//                 = OOB zero fill, stride = traversal stride, dilation = tap offset) or a
//                 plain 2-D map (1x1 / linear); B tiles from the [N, K] weight via tiled
//                 TMA; both land in the same swizzle.
//   warp 1      : TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=bn<=256,
//                 K=16 per instruction), fp32 accumulators in TMEM (4 when bn <= 128,
//                 else 2), so epilogues overlap the next tiles' MMAs.
//   warps 2..9  : epilogue, two groups of four warps (one per 32-row TMEM lane quadrant)
//                 taking alternate tiles: tcgen05.ld -> fp32 scale/shift (folded BN + bias,
//                 staged per group in smem and kept across tiles of the same segment),
//                 residual (TMA-prefetched tiles or LSU), branch-free ReLU/LeakyReLU ->
//                 bf16 -> TMA stores from double-buffered smem tiles (or the LSU
//                 transpose path); then publish the tile's completion (release counter).
//                 Optional split-K: fp32 partials reduced in a fixed order by the
//                 last-arriving split (deterministic).
// A problem whose weight is shared by several models runs once over their
// concatenated batches (one weight copy), each model a segment.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "gemm.h"
#include "sm100_ptx.cuh"

namespace gemel {

namespace {

constexpr uint32_t A_STAGE_BYTES = GEMM_BM * GEMM_BK * 2;   // 16 KB
constexpr int TILE_RING = 8;
// per epilogue warp: EPI_OBUFS 2 KB output tiles (32 rows x 32 bf16, 64B swizzle -- the
// layout of GemmSeg::out_map, stored by TMA; double-buffered so a chunk's store overlaps
// the next chunk) + EPI_RES_SLOTS residual tiles prefetched by TMA
constexpr int EPI_RES_SLOTS = 2;
constexpr int EPI_OBUFS = 2;
constexpr uint32_t EPI_WARP_BYTES = 2048 * (EPI_OBUFS + EPI_RES_SLOTS);
constexpr uint32_t EPI_STAGE_BYTES = 8 * EPI_WARP_BYTES;
constexpr uint32_t EPI_VEC_BYTES = 2 * 2 * 256 * 4;          // 4 KB scale/shift staging (a group: a tile's <= 256 columns)

constexpr int MAX_SMEM_PROBS = 1024;

// Developer probes (GemmLaunch::dbg: skip MMA / operand TMA / epilogue work to locate a
// bottleneck) exist only in builds with -DGEMEL_DEV_PROBES; production code has none.
#ifdef GEMEL_DEV_PROBES
constexpr bool kProbes = true;
#else
constexpr bool kProbes = false;
#endif

// One ring slot: a tile decoded ONCE by the producer, so the MMA lane and the epilogue
// read its geometry from shared memory instead of re-fetching the problem from L2
// (after acquire fences L1 holds nothing) on every tile.
// The epilogue's view of one member segment (the fields of GemmSeg it reads).
struct SegView {
  const float* scale;
  const float* shift;
  void* out;
  const void* res;
  int64_t ldo, ldr;
  int32_t m_begin, m_end, act, res_post;
  float slope;
  int32_t out_fp32, res_up, res_w;
  int32_t res_hw, out_w, out_hw, seg;   // seg: index into GemmLaunch::segs (its TMA maps)
};

__device__ __forceinline__ void load_segview(const GemmSeg& S, int seg, SegView& v) {
  v.scale = S.scale; v.shift = S.shift; v.out = S.out; v.res = S.res; v.ldo = S.ldo; v.ldr = S.ldr;
  v.m_begin = S.m_begin; v.m_end = S.m_end; v.act = S.act; v.res_post = S.res_post; v.slope = S.slope;
  v.out_fp32 = S.out_fp32; v.res_up = S.res_up; v.res_w = S.res_w; v.res_hw = S.res_hw; v.out_w = S.out_w;
  v.out_hw = S.out_hw; v.seg = seg;
}

constexpr int MAX_MSUB = 4;   // 128-row sub-tiles per tile (skinny problems amortise per-tile costs)

struct alignas(16) TileInfo {
  int32_t tile, pi, m_tile, n_tile, kspl, nst, chunk, bn;
  int32_t M, N, n_seg, seg_begin, ksplit, cnt_off, waited, m0;
  int32_t img, w0, h0, kw, dw, dh, cin_k, n_sub;
  int32_t c_oob, ktot, a_tiled, ks_begin, ks_end, ms, pad1, pad2;
  // im2col origin of every 128-row sub-tile (sub 0 = m0 / img / w0 / h0 above)
  int32_t sub_img[MAX_MSUB], sub_w0[MAX_MSUB], sub_h0[MAX_MSUB], sub_m0[MAX_MSUB];
  // the segment holding each sub-tile's first row, decoded by the scheduler so the
  // epilogue never walks GemmSeg in global memory (L2 round trips) for single-segment rows
  SegView ps[MAX_MSUB];
};
static_assert(sizeof(TileInfo) % 16 == 0, "TileInfo is copied to the peer CTA in 16-byte stores");

__device__ __forceinline__ int find_problem_smem(const int32_t* ib, int n, int item) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (item >= ib[mid]) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ int find_problem(const GemmProblem* __restrict__ P, int n, int item) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (item >= P[mid].item_begin) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ bool kspl_first(const TileInfo& TI) { return TI.kspl == 0; }

struct KLayout {
  uint32_t layout, sbo_a, sbo_b, lbo_a, lbo_b, region_a, region_b;
};

__device__ __forceinline__ KLayout k_layout(int chunk, int bn) {
  KLayout k;
  k.region_a = GEMM_BM * chunk * 2;
  k.region_b = bn * chunk * 2;
  switch (chunk) {
    case 64: k.layout = 2; k.sbo_a = k.sbo_b = 1024; k.lbo_a = k.lbo_b = 16; break;
    case 32: k.layout = 4; k.sbo_a = k.sbo_b = 512; k.lbo_a = k.lbo_b = 16; break;
    case 16: k.layout = 6; k.sbo_a = k.sbo_b = 256; k.lbo_a = k.lbo_b = 16; break;
    default: k.layout = 0; k.sbo_a = k.sbo_b = 128; k.lbo_a = k.region_a; k.lbo_b = k.region_b; break;
  }
  return k;
}

// Branch-free activation: y = max(y, 0) + neg_slope * min(y, 0), with neg_slope
// 1 (identity), 0 (ReLU) or the LeakyReLU slope -- one rounding, same value as the
// branchy form; a per-element branch costs far more issue slots than the math.
__device__ __forceinline__ float act_neg_slope(int act, float slope) {
  return act == ACT_RELU ? 0.f : (act == ACT_LEAKY ? slope : 1.f);
}
__device__ __forceinline__ float act_apply(float y, float neg_slope) {
  return fmaf(neg_slope, fminf(y, 0.f), fmaxf(y, 0.f));
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ float bf16_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); }

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Operand loads: a CTA pair's loads complete on the leader's barrier (cta_group::2).
template <int CG>
__device__ __forceinline__ void tma_2d(uint32_t dst, const void* tmap, uint32_t bar, int32_t c0, int32_t c1) {
  if constexpr (CG == 2) ptx::tma_load_2d_pair(dst, tmap, bar, c0, c1);
  else ptx::tma_load_2d(dst, tmap, bar, c0, c1);
}
template <int CG>
__device__ __forceinline__ void tma_im2col(uint32_t dst, const void* tmap, uint32_t bar, int32_t c, int32_t w, int32_t h,
                                           int32_t n, uint16_t ow, uint16_t oh) {
  if constexpr (CG == 2) ptx::tma_load_im2col_4d_pair(dst, tmap, bar, c, w, h, n, ow, oh);
  else ptx::tma_load_im2col_4d(dst, tmap, bar, c, w, h, n, ow, oh);
}

}  // namespace

template <int CG>
__device__ __forceinline__ void gemm_body(const GemmLaunch& L) {
  static_assert(CG == 1 || CG == 2, "cta_group");
  const int DBG = kProbes ? L.dbg : 0;
  // CTA pair: rank 0 (leader) schedules tiles and issues the MMAs; both CTAs load
  // operands and run the epilogue of their own 128 rows
  const uint32_t rank = CG == 2 ? ptx::cluster_ctarank() : 0u;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int stages = L.stages;
  const uint32_t b_stage_bytes = uint32_t(L.bn_max / CG) * GEMM_BK * 2;   // this CTA's share of B
  uint8_t* sA = smem;
  uint8_t* sB = sA + stages * A_STAGE_BYTES;
  uint8_t* sEpi = sB + stages * b_stage_bytes;                         // 1024-aligned
  float* s_vec = reinterpret_cast<float*>(sEpi + EPI_STAGE_BYTES);     // [2 groups][2][256]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sEpi + EPI_STAGE_BYTES + EPI_VEC_BYTES);
  // barriers: full[stages], empty[stages], tfull[4], tempty[4], ring_full[TILE_RING], ring_empty[TILE_RING], res[4]
  TileInfo* ring = reinterpret_cast<TileInfo*>(
      (reinterpret_cast<uintptr_t>(bars + 2 * stages + 8 + 2 * TILE_RING + 4 + 8 * EPI_RES_SLOTS) + 127) & ~uintptr_t(127));
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + TILE_RING);
  // item_begin of every problem: the scheduler's grab -> problem search runs on smem
  // (global reads would miss L1 after every acquire fence)
  int32_t* s_tb = reinterpret_cast<int32_t*>(tmem_slot + 4);
  const bool tb_smem = L.n_probs <= MAX_SMEM_PROBS;
  // scheduler caches (shared memory, written and read by the scheduler lane only): the
  // scalar fields of the problem being decoded (its tensor maps are not copied -- the TMA
  // lane reads them from global memory), its producers' (n_tiles, cnt_off), and the last
  // member segment looked up.  After each dependency acquire L1 holds nothing, so without
  // them every tile's decode re-fetched these from L2 as a chain of round trips.
  GemmProblem* s_prob = reinterpret_cast<GemmProblem*>(
      (reinterpret_cast<uintptr_t>(s_tb + MAX_SMEM_PROBS) + 127) & ~uintptr_t(127));
  int32_t* s_dep = reinterpret_cast<int32_t*>(s_prob + 1);          // [GEMM_MAX_DEPS][2]
  SegView* s_seg = reinterpret_cast<SegView*>(s_dep + 2 * GEMM_MAX_DEPS);
  if (tb_smem)
    for (int i = threadIdx.x; i < L.n_probs; i += blockDim.x) s_tb[i] = L.probs[i].item_begin;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bar_full = ptx::smem_u32(bars);
  const uint32_t bar_empty = bar_full + 8 * stages;
  const uint32_t bar_tfull = bar_empty + 8 * stages;
  const uint32_t bar_tempty = bar_tfull + 32;
  const uint32_t bar_rfull = bar_tempty + 32;
  const uint32_t bar_rempty = bar_rfull + 8 * TILE_RING;
  const uint32_t bar_res = bar_rempty + 8 * TILE_RING;
  const uint32_t bar_rs = bar_res + 8 * 4;   // [8 epilogue warps][EPI_RES_SLOTS] residual tiles landed
  const GemmProblem* __restrict__ probs = L.probs;
  int32_t* sched = L.sched;
  const uint32_t sA_u32 = ptx::smem_u32(sA), sB_u32 = ptx::smem_u32(sB);

  // TMEM accumulators: 4 when they fit (bn_max <= 128), else 2.  Two epilogue groups of 4
  // warps take alternate tiles, so a tile's epilogue latency (dependent metadata loads,
  // stores, the completion release) overlaps the next tile's instead of gating the MMA.
  // an accumulator holds a tile: ms sub-tiles x bn columns (acc_w = the launch's widest)
  const int n_acc = L.acc_w <= 128 ? 4 : 2;
  uint32_t tmem_cols = 32;
  while (tmem_cols < uint32_t(n_acc * L.acc_w)) tmem_cols <<= 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      ptx::mbar_init(bar_full + 8 * s, 1);      // the (leader's) producer arrives with the pair's bytes
      ptx::mbar_init(bar_empty + 8 * s, 1);
    }
    for (int a = 0; a < 4; ++a) {
      ptx::mbar_init(bar_tfull + 8 * a, 1);
      ptx::mbar_init(bar_tempty + 8 * a, 4 * CG);   // the 4 warps of the owning epilogue group, in each CTA
    }
    for (int r = 0; r < TILE_RING; ++r) {
      ptx::mbar_init(bar_rfull + 8 * r, 1);
      // TMA lane + MMA lane + 8 epilogue warps (+ the peer's TMA lane and 8 epilogue warps)
      ptx::mbar_init(bar_rempty + 8 * r, CG == 2 ? 19 : 10);
    }
    for (int w = 0; w < 4; ++w) ptx::mbar_init(bar_res + 8 * w, 1);
    for (int w = 0; w < 8 * EPI_RES_SLOTS; ++w) ptx::mbar_init(bar_rs + 8 * w, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    if constexpr (CG == 2) ptx::tmem_alloc_pair(ptx::smem_u32(tmem_slot), tmem_cols);
    else ptx::tmem_alloc(ptx::smem_u32(tmem_slot), tmem_cols);
  }
  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync();   // the peer's barriers are initialised before any remote arrive
  else __syncthreads();
  ptx::tc_fence_after();
  // barrier operations that may cross the pair: ring slots are written by the leader's
  // scheduler into both CTAs; consumers release slots, epilogues release accumulators
  // and producers signal stages on the LEADER's barriers
  auto ring_wait = [&](uint32_t bar, uint32_t ph) {
    if constexpr (CG == 2) ptx::mbar_wait_cluster(bar, ph);
    else ptx::mbar_wait(bar, ph);
  };
  auto arrive_leader = [&](uint32_t bar) {
    if constexpr (CG == 2) ptx::mbar_arrive_cluster(ptx::mapa(bar, 0));
    else ptx::mbar_arrive(bar);
  };
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // Operand loads of the tiles the scheduler warp (warp 10) decoded into the ring.
    if (lane == 0) {
      for (int p = 0; p < L.n_probs; ++p) {
        ptx::prefetch_tmap(&probs[p].tmap_a);
        ptx::prefetch_tmap(&probs[p].tmap_b);
      }
      int s = 0;
      uint32_t ph = 0;
      for (int k = 0;; ++k) {
        const int slot = k & (TILE_RING - 1);
        ring_wait(bar_rfull + 8 * slot, (k / TILE_RING) & 1);
        const TileInfo& TI = ring[slot];   // read in place; the slot is released after the loads
        const int tile = TI.tile;
        if (tile < 0) {
          arrive_leader(bar_rempty + 8 * slot);
          break;
        }
        // the scheduler acquired this tile's producer rows; order the async-proxy reads after it
        if (TI.waited) ptx::fence_proxy_async_global();
        const GemmProblem& P = probs[TI.pi];
        const int chunk = TI.chunk, R = GEMM_BK / chunk, bn = TI.bn;
        const int kw = TI.kw, dw = TI.dw, dh = TI.dh, cin_k = TI.cin_k, n_sub = TI.n_sub;
        const int c_oob = TI.c_oob, ktot = TI.ktot, a_tiled = TI.a_tiled;
        const void* tmap_a = &P.tmap_a;
        const void* tmap_b = &P.tmap_b;
        if (DBG & 32) { ptx::prefetch_tmap(tmap_a); ptx::prefetch_tmap(tmap_b); }   // probe
        const uint32_t region_a = GEMM_BM * chunk * 2, region_b = (bn / CG) * chunk * 2;
        const uint32_t tx = uint32_t(R) * (region_a + region_b);
        const int n0 = TI.n_tile * bn + int(rank) * (bn / CG);   // this CTA's half of the N tile
        const int ks_begin = TI.ks_begin, ks_end = TI.ks_end;
        const int dbg = DBG;
        // incremental K walk: sub-tile index, filter tap (r, t), channel offset; the weight
        // column of sub-tile `sub` is sub * chunk (taps are cin_k-wide, cin_k % chunk == 0)
        int sub = ks_begin * R;
        const int cpt = cin_k / chunk;
        const int tap0 = sub / cpt;
        int c0 = (sub - tap0 * cpt) * chunk;
        int r = tap0 / kw, t = tap0 - r * kw;
        const int ms = TI.ms;
        // the epilogue's residual rows (whole rows, every n tile) into L2 now, while this
        // tile's operands stream and its MMAs run: the epilogue's per-warp TMA residual
        // loads then hit L2 instead of waiting on HBM two chunks at a time
        if ((L.epi_flags & 2) && TI.n_tile == 0 && kspl_first(TI))
          for (int jm = 0; jm < ms; ++jm) {
            const SegView& v = TI.ps[jm];
            const int rows = min(GEMM_BM, v.m_end - TI.sub_m0[jm]);
            if (v.res != nullptr && v.res_up <= 1 && rows > 0)
              ptx::bulk_prefetch_l2(static_cast<const uint8_t*>(v.res) + int64_t(TI.sub_m0[jm] - v.m_begin) * v.ldr * 2,
                                    uint32_t(rows) * uint32_t(v.ldr) * 2u);
          }
        for (int ks = ks_begin; ks < ks_end; ++ks) {
         const int sub_k = sub, c0_k = c0, r_k = r, t_k = t;   // this K stage's walk state
         for (int jm = 0; jm < ms; ++jm) {   // one smem stage per (K stage, 128-row sub-tile)
          sub = sub_k; c0 = c0_k; r = r_k; t = t_k;
          const int m0 = TI.sub_m0[jm], img = TI.sub_img[jm], w0 = TI.sub_w0[jm], h0 = TI.sub_h0[jm];
          ptx::mbar_wait(bar_empty + 8 * s, ph ^ 1);
          // the stage's completion barrier: this CTA's, or the leader's (cluster address)
          const uint32_t fb = CG == 2 ? ptx::mapa(bar_full + 8 * s, 0) : bar_full + 8 * s;
          if (dbg & 2) {
            if (rank == 0) ptx::mbar_arrive(bar_full + 8 * s);
            if (++s == stages) { s = 0; ph ^= 1; }
            continue;
          }
          // the leader expects both CTAs' bytes (equal shares); the peer's loads only
          // complete_tx on the leader's barrier -- no per-stage cross-CTA arrive
          if (rank == 0)
            ptx::mbar_arrive_expect_tx(bar_full + 8 * s,
                                       CG * ((dbg & 768) ? uint32_t(R) * ((dbg & 256) ? region_a : region_b) : tx));
          const uint32_t a_dst = sA_u32 + s * A_STAGE_BYTES;
          const uint32_t b_dst = sB_u32 + s * b_stage_bytes;
          for (int j = 0; j < R; ++j, ++sub) {
            if (dbg & 768) {   // developer probe: A only (256) or B only (512)
              if (dbg & 256)
                tma_im2col<CG>(a_dst + j * region_a, tmap_a, fb, 0, w0, h0, img, 0, 0);
              else
                tma_2d<CG>(b_dst + j * region_b, tmap_b, fb, 0, n0);
              continue;
            }
            if (a_tiled) {   // 1x1 stride-1 / linear: A is the [M, C] matrix itself
              const bool in = sub < n_sub;
              tma_2d<CG>(a_dst + j * region_a, tmap_a, fb, in ? sub * chunk : c_oob, m0);
              tma_2d<CG>(b_dst + j * region_b, tmap_b, fb, in ? sub * chunk : ktot, n0);
            } else if (sub < n_sub) {
              tma_im2col<CG>(a_dst + j * region_a, tmap_a, fb, c0, w0, h0, img, uint16_t(t * dw),
                                      uint16_t(r * dh));
              tma_2d<CG>(b_dst + j * region_b, tmap_b, fb, sub * chunk, n0);
              c0 += chunk;
              if (c0 == cin_k) {
                c0 = 0;
                if (++t == kw) { t = 0; ++r; }
              }
            } else {  // K tail of the last stage: fully out-of-bounds boxes (zero fill)
              tma_im2col<CG>(a_dst + j * region_a, tmap_a, fb, c_oob, w0, h0, img, 0, 0);
              tma_2d<CG>(b_dst + j * region_b, tmap_b, fb, ktot, n0);
            }
          }
          if (++s == stages) { s = 0; ph ^= 1; }
         }
        }
        arrive_leader(bar_rempty + 8 * slot);
        if (L.trace && rank == 0) L.trace[16 * tile + 2] = globaltimer();
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && rank == 0) {   // the pair's MMAs are issued by the leader alone
      int s = 0;
      uint32_t ph = 0;
      for (int k = 0;; ++k) {
        const int slot = k & (TILE_RING - 1);
        const uint32_t acc = uint32_t(k) & uint32_t(n_acc - 1), acc_ph = uint32_t(k / n_acc) & 1u;
        ring_wait(bar_rfull + 8 * slot, (k / TILE_RING) & 1);
        const TileInfo& TI = ring[slot];
        const int tile = TI.tile, chunk = TI.chunk, bn = TI.bn, nst = TI.nst, ms = TI.ms;
        ptx::mbar_arrive(bar_rempty + 8 * slot);
        if (tile < 0) break;
        const KLayout kl = k_layout(chunk, bn / CG);   // B regions hold this CTA's half of N
        const uint32_t idesc = CG == 2 ? ptx::idesc_bf16_m256(uint32_t(bn)) : ptx::idesc_bf16_m128(uint32_t(bn));
        const int dbg = DBG;
        // Descriptors built once per tile; per stage / K-step only the 14-bit start-address
        // field changes, so the loop adds (byte offset >> 4) -- no carries (smem < 256 KB).
        const uint64_t a_desc0 = ptx::umma_desc(sA_u32, kl.lbo_a, kl.sbo_a, kl.layout);
        const uint64_t b_desc0 = ptx::umma_desc(sB_u32, kl.lbo_b, kl.sbo_b, kl.layout);
        uint32_t a_koff[GEMM_BK / 16], b_koff[GEMM_BK / 16];
#pragma unroll
        for (int st = 0; st < GEMM_BK / 16; ++st) {
          if (chunk >= 16) {
            const int kel = st * 16, j = kel / chunk, kk = (kel - j * chunk) / 16;
            a_koff[st] = (j * kl.region_a + kk * 32) >> 4;
            b_koff[st] = (j * kl.region_b + kk * 32) >> 4;
          } else {
            a_koff[st] = (2 * st * kl.region_a) >> 4;
            b_koff[st] = (2 * st * kl.region_b) >> 4;
          }
        }
        ring_wait(bar_tempty + 8 * acc, acc_ph ^ 1);   // both CTAs' epilogues drained this accumulator
        ptx::tc_fence_after();
        const uint32_t d_acc = tmem_base + acc * uint32_t(L.acc_w);
        for (int ks = 0; ks < nst; ++ks)
         for (int jm = 0; jm < ms; ++jm) {   // sub-tile jm accumulates in columns [jm*bn, jm*bn+bn)
          const uint32_t d_tmem = d_acc + uint32_t(jm * bn);
          ring_wait(bar_full + 8 * s, ph);               // both CTAs' operand halves landed
          if (L.trace && ks == 0 && jm == 0) L.trace[16 * tile + 3] = globaltimer();
          ptx::tc_fence_after();
          const uint64_t a_st = a_desc0 + ((uint32_t(s) * A_STAGE_BYTES) >> 4);
          const uint64_t b_st = b_desc0 + ((uint32_t(s) * b_stage_bytes) >> 4);
#pragma unroll
          for (int st = 0; st < GEMM_BK / 16; ++st)
            if (!(dbg & 1)) {
              if constexpr (CG == 2)
                ptx::umma_bf16_pair(d_tmem, a_st + a_koff[st], b_st + b_koff[st], idesc, (ks | st) != 0 ? 1u : 0u);
              else
                ptx::umma_bf16(d_tmem, a_st + a_koff[st], b_st + b_koff[st], idesc, (ks | st) != 0 ? 1u : 0u);
            }
          // frees the smem stage (of both CTAs) when these MMAs retire
          if constexpr (CG == 2) ptx::umma_commit_pair(bar_empty + 8 * s, 3);
          else if (dbg & 1024) ptx::mbar_arrive(bar_empty + 8 * s);   // probe: plain arrive instead of commit
          else ptx::umma_commit(bar_empty + 8 * s);
          if (++s == stages) { s = 0; ph ^= 1; }
        }
        // accumulator ready for the epilogue (of both CTAs)
        if constexpr (CG == 2) ptx::umma_commit_pair(bar_tfull + 8 * acc, 3);
        else ptx::umma_commit(bar_tfull + 8 * acc);
        if (L.trace) L.trace[16 * tile + 4] = globaltimer();
      }
    }
  } else if (warp < 10) {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 2;
    const int q = warp & 3;                  // TMEM lane quadrant this warp may access
    const int g = ew >> 2;                   // epilogue group: tiles k with k % 2 == g
    const bool leader = (ew & 3) == 0;       // the group's first warp publishes completion
    // the group's staged folded-BN vectors (scale[256], shift[256]) of one (segment, n tile),
    // kept across tiles: restaged only when the next sub-tile's segment or columns differ
    float* g_sc = s_vec + g * 512;
    float* g_sf = g_sc + 256;
    const float* st_ptr = nullptr;
    int st_n0 = -1, st_bn = 0, st_mbegin = -1;
    uint32_t res_phase = 0;                  // bit s: parity of the next completion of residual slot s
    for (int k = 0;; ++k) {
      const int slot = k & (TILE_RING - 1);
      const uint32_t acc = uint32_t(k) & uint32_t(n_acc - 1), acc_ph = uint32_t(k / n_acc) & 1u;
      ring_wait(bar_rfull + 8 * slot, (k / TILE_RING) & 1);
      const int tile = ring[slot].tile;
      if (tile < 0) {
        __syncwarp();
        if (lane == 0) arrive_leader(bar_rempty + 8 * slot);
        break;
      }
      if ((k & 1) != g) {                      // the other group's tile
        __syncwarp();
        if (lane == 0) arrive_leader(bar_rempty + 8 * slot);
        continue;
      }
      // scalar fields copied; the sub-tiles' segment views are read from the slot, which is
      // released when the tile is done
      const TileInfo& TIs = ring[slot];
      const int pi = TIs.pi, m_tile0 = TIs.m_tile, n_tile = TIs.n_tile, kspl = TIs.kspl, ms = TIs.ms;
      struct { int N, bn, M, ksplit, n_seg, seg_begin, cnt_off, waited; } TI = {
          TIs.N, TIs.bn, TIs.M, TIs.ksplit, TIs.n_seg, TIs.seg_begin, TIs.cnt_off, TIs.waited};
      const int n_tiles_p = (TI.N + TI.bn - 1) / TI.bn;
      const bool split = TI.ksplit > 1;
      // N = this tile's column end: a chunk of 32 never spills into the next N tile when bn % 32 != 0
      const int n0 = n_tile * TI.bn, bn = TI.bn, N = min(TI.N, n0 + bn);
      bool parked = false;            // split-K partial written: no output, no completion
      bool obuf_busy = false;
      int n_st = 0;                   // TMA output stores this warp issued for the tile
      for (int jm = 0; jm < ms; ++jm) {
      const int m_tile = m_tile0 + jm;
      const int mn = m_tile * n_tiles_p + n_tile;
      const int row0 = m_tile * GEMM_BM + q * 32;
      const int row = row0 + lane;
      const bool valid = row < TI.M;
      // each lane's member segment: the scheduler-decoded one (ps[jm]) when the warp's rows
      // all lie in it (the common case), else a warp-parallel search over GemmSeg
      SegView sv = TIs.ps[jm];
      bool fast_seg = true;
      if (!__all_sync(0xffffffffu, !valid || (row >= sv.m_begin && row < sv.m_end))) {
        const GemmSeg* seg0 = L.segs + TI.seg_begin;
        // lane j loads m_end of segment base+j (one coalesced round trip per 32 segments),
        // then counts the ends at or below its row
        int si = 0;
        for (int base = 0; base < TI.n_seg; base += 32) {
          const int me = base + lane < TI.n_seg ? seg0[base + lane].m_end : 0x7fffffff;
#pragma unroll 8
          for (int j = 0; j < 32; ++j) si += row >= __shfl_sync(0xffffffffu, me, j);
        }
        load_segview(seg0[min(si, TI.n_seg - 1)], TI.seg_begin + min(si, TI.n_seg - 1), sv);
        fast_seg = false;
      }
      // the group stages the folded-BN vectors of the sub-tile's first row's segment (the
      // same TileInfo for the group's 4 warps: a uniform decision), overlapping the tile's
      // MMAs (before the tfull wait); a lane whose rows belong to another member reads its
      // own vectors from global memory
      {
        const SegView& tv = TIs.ps[jm];
        if (tv.scale != st_ptr || n0 != st_n0 || bn != st_bn) {
          ptx::named_bar_sync(1 + g, 128);   // the group's warps are done with the old vectors
          for (int i = (ew & 3) * 32 + lane; i < bn; i += 128) {
            const int col = n0 + i;
            g_sc[i] = col < N ? __ldg(tv.scale + col) : 0.f;
            g_sf[i] = col < N ? __ldg(tv.shift + col) : 0.f;
          }
          ptx::named_bar_sync(1 + g, 128);
          st_ptr = tv.scale; st_n0 = n0; st_bn = bn; st_mbegin = tv.m_begin;
        }
      }
      const int64_t lrow = row - sv.m_begin;
      const float* sc_own = sv.scale;
      const float* sf_own = sv.shift;
      const float neg_slope = act_neg_slope(sv.act, sv.slope);
      // darknet shortcut: act(conv) + residual; otherwise act(conv + residual)
      const bool res_post = sv.res_post != 0;
      const float neg_post = res_post ? 1.f : neg_slope;
      // TMA epilogue (warp's 32 rows in one segment, bf16 output, plain residual): the
      // residual's 32x32 tiles are prefetched by TMA into this warp's smem slots (issued
      // now, overlapping the MMAs, then EPI_RES_SLOTS chunks ahead) and every full output
      // chunk leaves through a TMA store -- the memory-bound 1x1 layers are limited by
      // these streams, not by the tensor cores
      const int wrow0 = m_tile * GEMM_BM + q * 32;
      const bool tma_epi = fast_seg && !split && sv.out_fp32 == 0 && (sv.res == nullptr || sv.res_up <= 1) &&
                           wrow0 < TI.M && !(DBG & (64 | 8192 | 16384));
      const bool tma_res = tma_epi && sv.res != nullptr && ms == 1;
      const int lrow0 = wrow0 - sv.m_begin;
      const GemmSeg* gseg = L.segs + sv.seg;
      uint8_t* obuf = sEpi + ew * EPI_WARP_BYTES;
      const uint32_t rbuf0 = ptx::smem_u32(obuf + 2048 * EPI_OBUFS);
      const uint32_t rbar0 = bar_rs + 8 * (ew * EPI_RES_SLOTS);
      const int n_chunks = (min(N, n0 + bn) - n0 + 31) / 32;   // chunks with col0 < N
      auto res_issue = [&](int ci) {   // lane 0: residual tile of chunk ci into slot ci % EPI_RES_SLOTS
        const int sl = ci % EPI_RES_SLOTS;
        ptx::mbar_arrive_expect_tx(rbar0 + 8 * sl, 2048);
        ptx::tma_load_2d(rbuf0 + 2048 * sl, &gseg->res_map, rbar0 + 8 * sl, n0 + 32 * ci, lrow0);
      };
      if (tma_res && lane == 0) {
        if (TI.waited) ptx::fence_proxy_async_global();   // acquired producer rows -> async-proxy reads
        for (int ci = 0; ci < min(EPI_RES_SLOTS, n_chunks); ++ci) res_issue(ci);
      }
      if (jm == 0) {   // the whole tile's accumulator (every sub-tile) is ready at once
        if (DBG & 4096) {   // probe: back-off polling so idle epilogue warps do not steal issue slots
          while (!ptx::mbar_test(bar_tfull + 8 * acc, acc_ph)) __nanosleep(200);
        } else {
          ptx::mbar_wait(bar_tfull + 8 * acc, acc_ph);
        }
        if (L.trace && leader && lane == 0 && rank == 0) L.trace[16 * tile + 5] = globaltimer();
        ptx::tc_fence_after();
      }
      const uint32_t t_acc = tmem_base + (uint32_t(q * 32) << 16) + acc * uint32_t(L.acc_w) + uint32_t(jm * bn);
      // split-K: splits 0..ks-2 park fp32 partials column-major ([split][col][128 rows],
      // so a warp's 32 rows of one column are one 128-byte line) and count in; the last
      // split (grabbed last from the queue) waits for them and reduces in a fixed order
      // (own + p0 + p1 + ...): deterministic, no partial of its own to write.
      const int wpitch = (bn + 31) & ~31;       // columns per partial (whole 32-column chunks)
      const float* ws_tile = split ? probs[pi].ws + size_t(mn) * TI.ksplit * wpitch * GEMM_BM + q * 32 + lane : nullptr;
      if (split) {
        if (kspl != TI.ksplit - 1) {
          float* wp = probs[pi].ws + (size_t(mn) * TI.ksplit + kspl) * wpitch * GEMM_BM + q * 32 + lane;
          for (int c = 0; c < bn; c += 32) {
            uint32_t v[32];
            __syncwarp();
            ptx::tmem_ld_32x32b_x32(t_acc + c, v);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) wp[size_t(c + j) * GEMM_BM] = __uint_as_float(v[j]);
          }
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_leader(bar_tempty + 8 * acc);
          // bar.sync orders the group's 128 threads' partial stores before one release add
          ptx::named_bar_sync(1 + g, 128);
          if (leader && lane == 0) ptx::red_release_gpu_add(probs[pi].tcnt + mn, 1);
          parked = true;
          break;
        }
        if (lane == 0)
          while (ptx::ld_relaxed_gpu(probs[pi].tcnt + mn) < TI.ksplit - 1) __nanosleep(64);
        __syncwarp();
        ptx::fence_acq_rel_gpu();   // acquire the other splits' partials
      }
      // Residual rows come straight from global memory (LSU path, prefetched one chunk
      // ahead): the TMA engine stays dedicated to the producer's operand stream.  The
      // accumulator being ready implies the producer warp saw every dependency complete.
      const bool res_lane = valid && sv.res != nullptr && !tma_res;   // LSU residual path
      int64_t rrow = lrow;
      if (res_lane && sv.res_up > 1) {   // nearest-upsampled residual (FPN top-down add)
        const int img = int(lrow / sv.out_hw), rem = int(lrow - int64_t(img) * sv.out_hw);
        const int y = rem / sv.out_w, x = rem - (rem / sv.out_w) * sv.out_w;
        rrow = int64_t(img) * sv.res_hw + (y / sv.res_up) * sv.res_w + x / sv.res_up;
      }
      const __nv_bfloat16* res_row =
          res_lane ? reinterpret_cast<const __nv_bfloat16*>(sv.res) + rrow * sv.ldr : nullptr;
      uint4 rnext[4] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
      // (no fence here: the scheduler's acquire of the producer rows reaches this thread
      // through the ring barrier, and the residual is read L2-coherently with ld.cg)
      if (res_lane) {
        if (n0 + 32 <= N) {
#pragma unroll
          for (int j = 0; j < 4; ++j) rnext[j] = __ldcg(reinterpret_cast<const uint4*>(res_row + n0) + j);
        }
      }
      // per-row output base (global byte address; 0 for rows beyond M) for the coalesced store
      const int esz = sv.out_fp32 ? 4 : 2;
      const unsigned long long rowp =
          valid ? reinterpret_cast<unsigned long long>(sv.out) + (unsigned long long)(lrow * sv.ldo) * esz : 0ull;
      const bool ofp32 = __shfl_sync(0xffffffffu, sv.out_fp32, 0) != 0;
      const bool coal = !(DBG & 8192) && __all_sync(0xffffffffu, !valid || (sv.out_fp32 != 0) == ofp32);
      uint8_t* wbuf = obuf;
      for (int c = 0; c < ((DBG & 64) ? 0 : bn); c += 32) {
        uint32_t v[32];
        __syncwarp();   // tcgen05.ld is .sync.aligned: the whole warp, converged
        // (loading chunk c + 32 ahead of processing chunk c measured slower: +32 registers
        // spill at the 168-register cap of 352 threads)
        ptx::tmem_ld_32x32b_x32(t_acc + c, v);
        const int col0 = n0 + c;
        uint4 r4[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) r4[j] = rnext[j];
        if (tma_res && col0 < N) {   // this chunk's residual tile (slot ci % EPI_RES_SLOTS)
          const int ci = c / 32, sl = ci % EPI_RES_SLOTS;
          ptx::mbar_wait(rbar0 + 8 * sl, (res_phase >> sl) & 1u);
          res_phase ^= 1u << sl;
          const uint8_t* rs = obuf + 2048 * (EPI_OBUFS + sl) + lane * 64;
#pragma unroll
          for (int j = 0; j < 4; ++j) r4[j] = *reinterpret_cast<const uint4*>(rs + ((j ^ ((lane >> 1) & 3)) * 16));
          // the slot is refilled at the end of this chunk, once every lane has consumed it
        }
        if (res_lane && c + 32 < bn && col0 + 64 <= N) {
#pragma unroll
          for (int j = 0; j < 4; ++j) rnext[j] = __ldcg(reinterpret_cast<const uint4*>(res_row + col0 + 32) + j);
        }
        ptx::tmem_ld_wait();
        if (split) {   // fixed-order reduction: own + p0 + p1 + ... + p(ks-2), 16 loads in flight
          const float* rp = ws_tile + size_t(c) * GEMM_BM;
          for (int s2 = 0; s2 < TI.ksplit - 1; ++s2, rp += size_t(wpitch) * GEMM_BM) {
#pragma unroll
            for (int hh = 0; hh < 32; hh += 16) {
              float pp[16];
#pragma unroll
              for (int j = 0; j < 16; ++j) pp[j] = __ldcg(rp + size_t(hh + j) * GEMM_BM);
#pragma unroll
              for (int j = 0; j < 16; ++j) v[hh + j] = __float_as_uint(__uint_as_float(v[hh + j]) + pp[j]);
            }
          }
        }
        if (col0 >= N) continue;   // warp-uniform; rows beyond M compute but never store
        const bool staged = sv.m_begin == st_mbegin;
        const float* sc = staged ? g_sc + c : sc_own + col0;
        const float* sf = staged ? g_sf + c : sf_own + col0;
        float y[32];
        if (col0 + 32 <= N) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 a = *reinterpret_cast<const float4*>(sc + j);
            const float4 b = *reinterpret_cast<const float4*>(sf + j);
            y[j + 0] = fmaf(__uint_as_float(v[j + 0]), a.x, b.x);
            y[j + 1] = fmaf(__uint_as_float(v[j + 1]), a.y, b.y);
            y[j + 2] = fmaf(__uint_as_float(v[j + 2]), a.z, b.z);
            y[j + 3] = fmaf(__uint_as_float(v[j + 3]), a.w, b.w);
          }
          if (res_post) {
#pragma unroll
            for (int j = 0; j < 32; ++j) y[j] = act_apply(y[j], neg_slope);
          }
          if (res_lane || tma_res) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              y[8 * j + 0] += bf16_lo(r4[j].x); y[8 * j + 1] += bf16_hi(r4[j].x);
              y[8 * j + 2] += bf16_lo(r4[j].y); y[8 * j + 3] += bf16_hi(r4[j].y);
              y[8 * j + 4] += bf16_lo(r4[j].z); y[8 * j + 5] += bf16_hi(r4[j].z);
              y[8 * j + 6] += bf16_lo(r4[j].w); y[8 * j + 7] += bf16_hi(r4[j].w);
            }
          }
        } else {   // partial last chunk (N not a multiple of 32): predicated, fully unrolled
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float t = 0.f;
            if (col0 + j < N) {
              t = fmaf(__uint_as_float(v[j]), sc[j], sf[j]);
              if (res_post) t = act_apply(t, neg_slope);
              if (res_lane) t += __bfloat162float(res_row[col0 + j]);
              if (tma_res) {
                const uint32_t w = (&r4[j >> 3].x)[(j >> 1) & 3];
                t += (j & 1) ? bf16_hi(w) : bf16_lo(w);
              }
            }
            y[j] = t;
          }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) y[j] = act_apply(y[j], neg_post);
        if (DBG & 16384) {
          // probe: skip stores
        } else if (tma_epi && (L.epi_flags & 1) && col0 + 32 <= N) {
          // bf16 tile in the out_map's 64B-swizzled layout, then one TMA store of 32 rows x
          // 32 columns (rows past the segment are clipped by the map)
          // buffer n_st & 1: the store issued two chunks ago (same buffer) must have read it
          const bool one_buf = (L.epi_flags & 4) != 0;   // A/B knob: single output buffer
          uint8_t* ob = obuf + (one_buf ? 0 : 2048 * (n_st & (EPI_OBUFS - 1)));
          if (one_buf ? n_st >= 1 : n_st >= EPI_OBUFS) {
            if (lane == 0) {
              if (one_buf) ptx::bulk_wait_read<0>();
              else ptx::bulk_wait_read<EPI_OBUFS - 1>();
            }
            __syncwarp();
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t slot = uint32_t(j) ^ ((lane >> 1) & 3);
            const uint4 pk = make_uint4(pack_bf16(y[8 * j + 0], y[8 * j + 1]), pack_bf16(y[8 * j + 2], y[8 * j + 3]),
                                        pack_bf16(y[8 * j + 4], y[8 * j + 5]), pack_bf16(y[8 * j + 6], y[8 * j + 7]));
            *reinterpret_cast<uint4*>(ob + lane * 64 + slot * 16) = pk;
          }
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            ptx::tma_store_2d(&gseg->out_map, ptx::smem_u32(ob), col0, lrow0);
            ptx::bulk_commit();
          }
          obuf_busy = true;
          ++n_st;
        } else if (coal && col0 + 32 <= N) {
          // Coalesced store through a per-warp smem transpose: lane = row on the TMEM side,
          // but 4 (bf16) / 8 (fp32) consecutive lanes cover one row's 64/128 contiguous bytes
          // on the global side, so every request writes whole 32-byte sectors.
          if (!ofp32) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint32_t slot = uint32_t(j) ^ ((lane >> 1) & 3);
              const uint4 pk = make_uint4(pack_bf16(y[8 * j + 0], y[8 * j + 1]), pack_bf16(y[8 * j + 2], y[8 * j + 3]),
                                          pack_bf16(y[8 * j + 4], y[8 * j + 5]), pack_bf16(y[8 * j + 6], y[8 * j + 7]));
              *reinterpret_cast<uint4*>(wbuf + lane * 64 + slot * 16) = pk;
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int r = (lane >> 2) + 8 * i, sg = lane & 3;
              const uint4 pk = *reinterpret_cast<const uint4*>(wbuf + r * 64 + ((sg ^ ((r >> 1) & 3)) * 16));
              const unsigned long long p = __shfl_sync(0xffffffffu, rowp, r);
              if (p) *reinterpret_cast<uint4*>(p + size_t(col0) * 2 + sg * 16) = pk;
            }
          } else {   // fp32: two 16-column halves through the same 2 KB buffer
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const uint32_t slot = uint32_t(j) ^ ((lane >> 1) & 3);
                *reinterpret_cast<float4*>(wbuf + lane * 64 + slot * 16) =
                    make_float4(y[16 * hh + 4 * j], y[16 * hh + 4 * j + 1], y[16 * hh + 4 * j + 2], y[16 * hh + 4 * j + 3]);
              }
              __syncwarp();
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int r = (lane >> 2) + 8 * i, sg = lane & 3;
                const float4 f = *reinterpret_cast<const float4*>(wbuf + r * 64 + ((sg ^ ((r >> 1) & 3)) * 16));
                const unsigned long long p = __shfl_sync(0xffffffffu, rowp, r);
                if (p) *reinterpret_cast<float4*>(p + size_t(col0 + 16 * hh) * 4 + sg * 16) = f;
              }
              __syncwarp();
            }
          }
          __syncwarp();
        } else if (!valid) {
          // row beyond M: nothing to store
        } else if (sv.out_fp32) {
          float* op = reinterpret_cast<float*>(sv.out) + lrow * sv.ldo + col0;
          if (col0 + 32 <= N) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              reinterpret_cast<float4*>(op)[j] = make_float4(y[4 * j], y[4 * j + 1], y[4 * j + 2], y[4 * j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col0 + j < N) op[j] = y[j];
          }
        } else {
          __nv_bfloat16* op = reinterpret_cast<__nv_bfloat16*>(sv.out) + lrow * sv.ldo + col0;
          if (col0 + 32 <= N) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              reinterpret_cast<uint4*>(op)[j] =
                  make_uint4(pack_bf16(y[8 * j + 0], y[8 * j + 1]), pack_bf16(y[8 * j + 2], y[8 * j + 3]),
                             pack_bf16(y[8 * j + 4], y[8 * j + 5]), pack_bf16(y[8 * j + 6], y[8 * j + 7]));
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col0 + j < N) op[j] = __float2bfloat16_rn(y[j]);
          }
        }
        if (tma_res) {   // refill this chunk's residual slot (every lane has used its values):
          const int ci = c / 32;   // generic-proxy reads -> async-proxy write of the same smem
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0 && ci + EPI_RES_SLOTS < n_chunks) res_issue(ci + EPI_RES_SLOTS);
        }
      }
      }   // sub-tiles
      __syncwarp();
      if (lane == 0) arrive_leader(bar_rempty + 8 * slot);   // the slot's sub-tile views are no longer read
      if (parked) continue;
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_leader(bar_tempty + 8 * acc);
      if (obuf_busy && lane == 0) ptx::bulk_wait<0>();   // this warp's TMA stores are complete
      __syncwarp();
      if (L.trace && leader && lane == 0 && rank == 0) L.trace[16 * tile + 6] = globaltimer();
      // publish completion: the group's 4 warps' stores, then one release add per sub-tile
      // (a pair's second CTA past the problem's last m-tile has nothing to publish)
      ptx::fence_proxy_async_global();
      ptx::named_bar_sync(1 + g, 128);
      if (leader && lane == 0) {
        for (int jm = 0; jm < ms; ++jm)
          if ((m_tile0 + jm) * GEMM_BM < TI.M)
            ptx::red_release_gpu_add(sched + TI.cnt_off + m_tile0 + jm, 1);   // cumulative over the bar.sync
        if (L.trace && rank == 0) L.trace[16 * tile + 7] = globaltimer();
      }
    }
  } else if (warp == 10 && rank == 0) {
    // ------------------------------------------------------------ tile scheduler
    // Pulls tiles from the global queue in topological order, decodes each ONCE into a
    // ring slot (the TMA lane, the MMA lane and the epilogue read it from shared memory)
    // and waits on the producer rows it reads -- up to TILE_RING tiles ahead of the TMA
    // lane, so the L2 round trips of decoding and dependency polls leave the operand
    // stream's critical path.
    if (lane == 0) {
      // A grab (one atomic on the queue counter) hands out a run of P.run consecutive
      // tiles of one problem; the NEXT grab is fetched as soon as a run starts, so its
      // round trip overlaps the run's tiles.
      int next = atomicAdd(sched, 1);
      int pi = 0, run_tile = 0, run_end = 0, cached_pi = -1;
      bool grab = false;   // the next queue position is claimed once this run's first tile is ready
      bool seg_valid = false;   // s_seg holds a segment of problem cached_pi
      auto cache_problem = [&](int p) {
        if (p == cached_pi) return;
        constexpr int kMaps = 2 * int(sizeof(CUtensorMap)) / 16;   // the two tensor maps lead the struct
        const int4* src = reinterpret_cast<const int4*>(probs + p);
        int4* dst = reinterpret_cast<int4*>(s_prob);
        int4 t[int(sizeof(GemmProblem)) / 16 - kMaps];
#pragma unroll
        for (int j = 0; j < int(sizeof(GemmProblem)) / 16 - kMaps; ++j) t[j] = src[kMaps + j];   // one round trip
#pragma unroll
        for (int j = 0; j < int(sizeof(GemmProblem)) / 16 - kMaps; ++j) dst[kMaps + j] = t[j];
        const int nd = s_prob->n_deps;
        for (int d = 0; d < nd; ++d) {
          s_dep[2 * d] = probs[s_prob->deps[d]].n_tiles;
          s_dep[2 * d + 1] = probs[s_prob->deps[d]].cnt_off;
        }
        cached_pi = p;
        seg_valid = false;
      };
      for (int k = 0;; ++k) {
        const int slot = k & (TILE_RING - 1);
        ptx::mbar_wait(bar_rempty + 8 * slot, ((k / TILE_RING) & 1) ^ 1);
        const unsigned long long t_grab = L.trace ? globaltimer() : 0ull;
        if (run_tile == run_end && next < L.total_items && !(DBG & 16)) {
          const int item = next;
          pi = tb_smem ? find_problem_smem(s_tb, L.n_probs, item) : find_problem(probs, L.n_probs, item);
          cache_problem(pi);
          const GemmProblem& Q = *s_prob;
          run_tile = (item - Q.item_begin) * Q.run;
          const int m_step = CG * Q.msub;
          run_end = min(run_tile + Q.run, (Q.m_tiles + m_step - 1) / m_step * Q.n_tiles * Q.ksplit);
          grab = true;
        }
        const int tile = run_tile < run_end ? s_prob->tile_begin + run_tile++ : -1;
        TileInfo& TI = ring[slot];
        TI.tile = tile;
        if (tile < 0) {
          ptx::mbar_arrive(bar_rfull + 8 * slot);
          if constexpr (CG == 2) {   // end of work for the peer too
            ptx::st_cluster_v4(ptx::mapa(ptx::smem_u32(&ring[slot]), 1), make_int4(-1, 0, 0, 0));
            ptx::mbar_arrive_cluster(ptx::mapa(bar_rfull + 8 * slot, 1));
          }
          break;
        }
        const GemmProblem& P = *s_prob;   // the cached scalars of probs[pi]
        const int local = tile - P.tile_begin;
        const int ksplit = P.ksplit, n_tiles = P.n_tiles;
        const int mn = local / ksplit, kspl = local - mn * ksplit;
        // a tile covers m_step consecutive m-tiles: ms sub-tiles of one CTA, or a pair's two
        // (the second CTA's rows)
        const int ms = P.msub, m_step = CG * ms;
        const int m_tile = (mn / n_tiles) * m_step, n_tile = mn - (mn / n_tiles) * n_tiles;
        // wait for the producer rows this tile reads: per dependency, the band of producer
        // m-tiles covering this m-tile's receptive field (conv input) or rows (residual);
        // a producer m-tile is complete when all its n-tiles published (wavefront overlap
        // of dependent layers instead of whole-layer barriers)
        bool waited = false;
        for (int dd = 0; dd < P.n_deps * m_step; ++dd) {
          const int d = dd % P.n_deps, mt_i = m_tile + dd / P.n_deps;
          if (mt_i >= P.m_tiles) break;
          const int* rg = P.dep_rng + (mt_i * P.n_deps + d) * 2;
          const int lo = rg[0], hi = rg[1], need = s_dep[2 * d];
          const int* cnt = sched + s_dep[2 * d + 1];
          for (int mt = lo; mt <= hi; mt += 16) {   // 16 independent polls in flight per round trip
            int v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = (mt + j <= hi) ? ptx::ld_relaxed_gpu(cnt + mt + j) : need;
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (v[j] < need)
                while (ptx::ld_relaxed_gpu(cnt + mt + j) < need) __nanosleep(32);
            waited = true;
          }
        }
        if (waited) ptx::fence_acq_rel_gpu();   // one acquire after the relaxed polls
        // claim the next queue position only now: a CTA whose tile still waits on its
        // producers must not also hold the tile behind it (another SM may be idle)
        if (grab) {
          next = atomicAdd(sched, 1);
          grab = false;
        }
        if (L.trace) {
          L.trace[16 * tile + 0] = t_grab;
          L.trace[16 * tile + 1] = globaltimer();
          L.trace[16 * tile + 8] = blockIdx.x;
        }
        const int m0 = m_tile * GEMM_BM;
        const int HoWo = P.HoWo, Wo = P.Wo;
        const int img = m0 / HoWo, rem = m0 - img * HoWo;
        const int oh = rem / Wo, ow = rem - oh * Wo;
        const int kst = P.kst_split;
        TI.pi = pi; TI.m_tile = m_tile; TI.n_tile = n_tile; TI.kspl = kspl;
        TI.ks_begin = kspl * kst;
        TI.ks_end = min(TI.ks_begin + kst, P.n_kstages);
        TI.nst = TI.ks_end - TI.ks_begin;
        TI.chunk = P.chunk; TI.bn = P.bn; TI.M = P.M; TI.N = P.N;
        TI.n_seg = P.n_seg; TI.seg_begin = P.seg_begin; TI.ksplit = ksplit; TI.cnt_off = P.cnt_off;
        TI.waited = waited ? 1 : 0;
        TI.m0 = m0; TI.img = img;
        TI.w0 = ow * P.sw - P.pw; TI.h0 = oh * P.sh - P.ph;
        TI.kw = P.kw; TI.dw = P.dw; TI.dh = P.dh; TI.cin_k = P.cin_k; TI.n_sub = P.n_sub;
        TI.c_oob = P.c_oob; TI.ktot = P.Ktot; TI.a_tiled = P.a_tiled;
        TI.ms = ms;
        for (int jm = 0; jm < ms; ++jm) {   // every sub-tile's im2col origin and member segment
          const int mj = m0 + jm * GEMM_BM;
          const int imgj = mj / HoWo, remj = mj - imgj * HoWo;
          const int ohj = remj / Wo, owj = remj - ohj * Wo;
          TI.sub_m0[jm] = mj; TI.sub_img[jm] = imgj;
          TI.sub_w0[jm] = owj * P.sw - P.pw; TI.sub_h0[jm] = ohj * P.sh - P.ph;
          if (jm > 0 && (mj < TI.ps[jm - 1].m_end || mj >= P.M)) {
            TI.ps[jm] = TI.ps[jm - 1];
            continue;
          }
          if (seg_valid && mj >= s_seg->m_begin && mj < s_seg->m_end) {   // the last segment looked up
            TI.ps[jm] = *s_seg;
            continue;
          }
          int lo = 0, hi = P.n_seg - 1;   // binary search on m_end
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (L.segs[P.seg_begin + mid].m_end > mj) hi = mid; else lo = mid + 1;
          }
          load_segview(L.segs[P.seg_begin + lo], P.seg_begin + lo, TI.ps[jm]);
          *s_seg = TI.ps[jm];
          seg_valid = true;
        }
        if constexpr (CG == 2) {
          // the peer's copy: the next 128 rows (m-tile + 1), written into its ring slot
          // through distributed shared memory, released by a cluster-scope arrive
          TileInfo T2 = TI;
          const int m1 = m0 + GEMM_BM;
          const int img1 = m1 / HoWo, rem1 = m1 - img1 * HoWo;
          const int oh1 = rem1 / Wo, ow1 = rem1 - oh1 * Wo;
          T2.m_tile = m_tile + 1; T2.m0 = m1; T2.img = img1;
          T2.w0 = ow1 * P.sw - P.pw; T2.h0 = oh1 * P.sh - P.ph;
          T2.sub_m0[0] = m1; T2.sub_img[0] = img1; T2.sub_w0[0] = T2.w0; T2.sub_h0[0] = T2.h0;
          if (m1 >= TI.ps[0].m_end && m1 < P.M) {
            int lo = 0, hi = P.n_seg - 1;
            while (lo < hi) {
              const int mid = (lo + hi) >> 1;
              if (L.segs[P.seg_begin + mid].m_end > m1) hi = mid; else lo = mid + 1;
            }
            load_segview(L.segs[P.seg_begin + lo], P.seg_begin + lo, T2.ps[0]);
          }
          const uint32_t dst = ptx::mapa(ptx::smem_u32(&ring[slot]), 1);
          const int4* src = reinterpret_cast<const int4*>(&T2);
#pragma unroll
          for (int j = 0; j < int(sizeof(TileInfo) / 16); ++j) ptx::st_cluster_v4(dst + 16 * j, src[j]);
          ptx::mbar_arrive_cluster(ptx::mapa(bar_rfull + 8 * slot, 1));
        }
        ptx::mbar_arrive(bar_rfull + 8 * slot);   // release: the TileInfo stores above
      }
    }
  }

  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync();   // no CTA leaves while its peer may still signal it
  else __syncthreads();
  if (warp == 1) {
    __syncwarp();
    ptx::tc_fence_after();
    if constexpr (CG == 2) ptx::tmem_dealloc_pair(tmem_base, tmem_cols);
    else ptx::tmem_dealloc(tmem_base, tmem_cols);
  }
}

extern "C" __global__ void __launch_bounds__(GEMM_THREADS, 1) gemel_gemm_sm100(const GemmLaunch L) { gemm_body<1>(L); }

extern "C" __global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GEMM_THREADS, 1)
    gemel_gemm_sm100_pair(const GemmLaunch L) {
  gemm_body<2>(L);
}

size_t gemm_smem_bytes(int bn_max, int stages, int cg) {
  return 1024 + size_t(stages) * (A_STAGE_BYTES + size_t(bn_max / cg) * GEMM_BK * 2) + EPI_STAGE_BYTES + EPI_VEC_BYTES +
         (2 * stages + 8 + 2 * TILE_RING + 4 + 8 * EPI_RES_SLOTS) * 8 + 128 + TILE_RING * sizeof(TileInfo) + 16 +
         MAX_SMEM_PROBS * 4 + 128 + sizeof(GemmProblem) + 8 * GEMM_MAX_DEPS + sizeof(SegView);
}

int gemm_pick_stages(int bn_max, int cg) {
  int s = 8;
  while (s > 2 && gemm_smem_bytes(bn_max, s, cg) > 227 * 1024) --s;
  return s;
}

int gemm_launch(const GemmLaunch& L, int grid, void* stream) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemel_gemm_sm100, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemel_gemm_sm100_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return int(e);
    attr_set = true;
  }
  const size_t smem = gemm_smem_bytes(L.bn_max, L.stages, L.cg);
  if (L.cg == 2) {   // grid: whole CTA pairs (cluster dims 2 x 1 x 1)
    gemel_gemm_sm100_pair<<<(grid + 1) & ~1, GEMM_THREADS, smem, static_cast<cudaStream_t>(stream)>>>(L);
  } else {
    gemel_gemm_sm100<<<grid, GEMM_THREADS, smem, static_cast<cudaStream_t>(stream)>>>(L);
  }
  return int(cudaGetLastError());
}

}  // namespace gemel
