// Developer self-test for the tcgen05 implicit-GEMM kernel: random conv/linear
// problems (every chunk width, stride, padding, dilation, N tails, several
// problems and segments per launch) against a naive CUDA-core fp32 reference.
// Not a parity test (tests/ compare with the fp64 oracle); it localises
// descriptor / TMA bugs quickly.  Usage: gemm_selftest [bench]
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../kernels/gemm.h"
#include "../tmap.h"

using namespace gemel;

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) {                                                            \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);  \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

struct Conv {
  int n, h, w, cs, cin, cout, k, s, p, d, act;
  bool res;
};

__global__ void ref_conv(const __nv_bfloat16* x, const __nv_bfloat16* wt, const float* sc, const float* sf,
                         const __nv_bfloat16* res, float* y, int n, int h, int w, int cs, int cin, int cin_k, int cout,
                         int k, int s, int p, int d, int ho, int wo, int act) {
  long idx = blockIdx.x * long(blockDim.x) + threadIdx.x;
  long total = long(n) * ho * wo * cout;
  if (idx >= total) return;
  int co = idx % cout;
  long m = idx / cout;
  int ow = m % wo, oh = (m / wo) % ho, img = m / (long(wo) * ho);
  float acc = 0.f;
  for (int r = 0; r < k; ++r)
    for (int t = 0; t < k; ++t) {
      int ih = oh * s - p + r * d, iw = ow * s - p + t * d;
      if (ih < 0 || ih >= h || iw < 0 || iw >= w) continue;
      for (int c = 0; c < cin; ++c)
        acc += __bfloat162float(x[((long(img) * h + ih) * w + iw) * cs + c]) *
               __bfloat162float(wt[long(co) * (k * k * cin_k) + (r * k + t) * cin_k + c]);
    }
  float v = acc * sc[co] + sf[co];
  if (res) v += __bfloat162float(res[m * cout + co]);
  if (act == 1) v = fmaxf(v, 0.f);
  y[idx] = v;
}

static int chunk_for(int cs) { return cs >= 64 ? 64 : cs; }

int main(int argc, char** argv) {
  bool bench = argc > 1;
  std::mt19937 rng(1234);
  std::normal_distribution<float> nd(0.f, 1.f);
  std::vector<Conv> cases = {
      {2, 16, 16, 64, 64, 64, 3, 1, 1, 1, 1, false},   {2, 20, 20, 8, 3, 64, 7, 2, 3, 1, 1, false},
      {1, 9, 11, 32, 32, 48, 3, 2, 1, 1, 0, false},    {3, 7, 7, 16, 16, 80, 3, 1, 1, 2, 1, false},
      {2, 14, 14, 128, 128, 256, 1, 2, 0, 1, 0, true}, {5, 1, 1, 512, 512, 1000, 1, 1, 0, 1, 0, false},
      {3, 13, 13, 192, 192, 96, 3, 1, 1, 1, 1, true},  {1, 30, 30, 64, 64, 128, 3, 2, 1, 1, 1, false},
  };
  // bench <id>: a single micro-case (TMA/L2 throughput probes)
  const std::vector<Conv> micro = {
      {16384, 1, 1, 4096, 4096, 256, 1, 1, 0, 1, 0, false},   // 0 plain GEMM (1x1 pixels)
      {64, 28, 28, 256, 256, 256, 1, 1, 0, 1, 0, false},     // 1 1x1 conv over images
      {48, 28, 28, 256, 256, 256, 3, 1, 1, 1, 0, false},     // 2 3x3 conv N=256
      {48, 28, 28, 256, 256, 64, 3, 1, 1, 1, 0, false},      // 3 3x3 conv N=64
      {16384, 1, 1, 4096, 4096, 64, 1, 1, 0, 1, 0, false},   // 4 plain GEMM N=64
      {16384, 1, 1, 1024, 1024, 256, 1, 1, 0, 1, 0, false},  // 5 K=1024
      {16384, 1, 1, 2048, 2048, 256, 1, 1, 0, 1, 0, false},  // 6 K=2048
      {16384, 1, 1, 8192, 8192, 256, 1, 1, 0, 1, 0, false},  // 7 K=8192
      {16384, 1, 1, 64, 64, 256, 1, 1, 0, 1, 0, false},      // 8 K=64 (epilogue-bound)
      {5914624, 1, 1, 32, 32, 32, 1, 1, 0, 1, 0, false},     // 9 YOLO stem shape (im2col rows K=32, N=32)
      {1478656, 1, 1, 152, 152, 64, 1, 1, 0, 1, 0, false},   // 10 FRCNN stem shape (K=152, N=64)
      {92416, 1, 1, 256, 256, 128, 1, 1, 0, 1, 0, false},    // 11 YOLO 1x1 256->128 @76 x16
      {65536, 1, 1, 4096, 4096, 256, 1, 1, 0, 1, 0, false},  // 12 plain GEMM, 512 tiles (3.5 waves)
      {192, 28, 28, 256, 256, 256, 3, 1, 1, 1, 0, false},    // 13 3x3 conv N=256, 1176 tiles
      {192, 28, 28, 128, 128, 128, 3, 1, 1, 1, 0, false},    // 14 3x3 conv N=128
      {192, 56, 56, 64, 64, 64, 3, 1, 1, 1, 0, false},       // 15 3x3 conv N=64 (4704 tiles)
      {369664, 1, 1, 256, 256, 256, 1, 1, 0, 1, 1, false},  // 16 1x1 K=256 N=256 (memory-bound), ReLU
      {369664, 1, 1, 256, 256, 256, 1, 1, 0, 1, 1, true},   // 17 same + residual
      {369664, 1, 1, 64, 64, 256, 1, 1, 0, 1, 1, true},     // 18 1x1 K=64 N=256 + residual (R50 expand)
      {369664, 1, 1, 256, 256, 128, 1, 1, 0, 1, 1, false},  // 19 1x1 K=256 N=128
  };
  if (argc > 2) cases = {micro[atoi(argv[2])]};
  else if (bench) cases = {{24, 56, 56, 64, 64, 64, 3, 1, 1, 1, 1, true},
                      {24, 28, 28, 128, 128, 128, 3, 1, 1, 1, 1, false},
                      {24, 14, 14, 256, 256, 256, 3, 1, 1, 1, 1, false},
                      {24, 56, 56, 256, 256, 64, 1, 1, 0, 1, 1, false},
                      {8, 224, 224, 8, 3, 64, 7, 2, 3, 1, 1, false},
                      {48, 28, 28, 256, 256, 512, 3, 1, 1, 1, 1, false},
                      {48, 14, 14, 512, 512, 512, 3, 1, 1, 1, 1, false}};
  // All cases run in ONE grouped launch, each problem split into 2 segments.
  std::vector<GemmProblem> probs(cases.size());
  std::vector<GemmSeg> segs;
  struct Bufs { __nv_bfloat16 *x, *w, *res, *out; float *sc, *sf, *ref; long m; int ho, wo; };
  std::vector<Bufs> bufs(cases.size());
  int tiles = 0, items = 0, bn_max = 16, n_cnt = 1;
  const int run = getenv("RUN") ? atoi(getenv("RUN")) : 1;   // tiles per queue grab
  const int cg = getenv("CG") ? atoi(getenv("CG")) : 1;       // 2: CTA-pair kernel
  const int msub = getenv("MSUB") ? atoi(getenv("MSUB")) : 1; // 128-row sub-tiles per tile   // sched[0] = tile queue, then per-m-tile counters
  double flops = 0;
  for (size_t i = 0; i < cases.size(); ++i) {
    Conv c = cases[i];
    int ho = (c.h + 2 * c.p - c.d * (c.k - 1) - 1) / c.s + 1, wo = (c.w + 2 * c.p - c.d * (c.k - 1) - 1) / c.s + 1;
    int chunk = chunk_for(c.cs), cin_k = (c.cin + chunk - 1) / chunk * chunk;
    long m = long(c.n) * ho * wo;
    int ktot = c.k * c.k * cin_k;
    std::vector<__nv_bfloat16> hx(long(c.n) * c.h * c.w * c.cs), hw(long(c.cout) * ktot), hr(m * c.cout);
    for (long j = 0; j < (long)hx.size(); ++j) hx[j] = __float2bfloat16((j % c.cs) < c.cin ? nd(rng) : 0.f);
    float ws = 1.f / std::sqrt(float(c.k * c.k * c.cin));
    for (long j = 0; j < (long)hw.size(); ++j) hw[j] = __float2bfloat16((j % cin_k) < c.cin ? nd(rng) * ws : 0.f);
    for (auto& v : hr) v = __float2bfloat16(nd(rng));
    std::vector<float> hsc(c.cout), hsf(c.cout);
    for (int j = 0; j < c.cout; ++j) { hsc[j] = 0.5f + (j % 7) * 0.1f; hsf[j] = 0.01f * (j % 5); }
    Bufs& b = bufs[i];
    b.m = m; b.ho = ho; b.wo = wo;
    CK(cudaMalloc(&b.x, hx.size() * 2)); CK(cudaMalloc(&b.w, hw.size() * 2)); CK(cudaMalloc(&b.res, hr.size() * 2));
    CK(cudaMalloc(&b.out, m * c.cout * 2)); CK(cudaMalloc(&b.sc, c.cout * 4)); CK(cudaMalloc(&b.sf, c.cout * 4));
    CK(cudaMalloc(&b.ref, m * c.cout * 4));
    CK(cudaMemcpy(b.x, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(b.w, hw.data(), hw.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(b.res, hr.data(), hr.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(b.sc, hsc.data(), c.cout * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(b.sf, hsf.data(), c.cout * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(b.out, 0xFF, m * c.cout * 2));
    GemmProblem& P = probs[i];
    memset(&P, 0, sizeof(P));
    int upper = c.p - (c.k - 1) * c.d;
    int rc = tmap_encode_im2col(&P.tmap_a, b.x, c.n, c.h, c.w, c.cs, c.cs, -c.p, -c.p, upper, upper, chunk, 128, c.s,
                                c.s);
    const bool a_tiled = argc > 6 && atoi(argv[6]) && c.k == 1 && c.s == 1 && c.p == 0;
    if (a_tiled) rc = tmap_encode_2d(&P.tmap_a, b.x, c.cs, uint64_t(m), uint64_t(c.cs) * 2, chunk, 128, chunk * 2);
    int bn = c.cout >= 256 ? 256 : ((c.cout + 15) / 16 * 16);
    rc |= tmap_encode_2d(&P.tmap_b, b.w, ktot, c.cout, uint64_t(ktot) * 2, chunk, bn / cg, chunk * 2);
    if (rc) { printf("tmap encode failed case %zu rc=%d\n", i, rc); return 1; }
    P.M = int(m); P.N = c.cout; P.Ktot = ktot; P.HoWo = ho * wo; P.Wo = wo;
    P.sh = P.sw = c.s; P.ph = P.pw = c.p; P.kw = c.k; P.dh = P.dw = c.d;
    P.cin_k = cin_k; P.chunk = chunk; P.n_sub = c.k * c.k * (cin_k / chunk);
    P.n_kstages = (P.n_sub + (64 / chunk) - 1) / (64 / chunk); P.c_oob = c.cs; P.bn = bn;
    P.ksplit = 1; P.kst_split = P.n_kstages; P.a_tiled = a_tiled ? 1 : 0;
    P.m_tiles = int((m + 127) / 128); P.n_tiles = (c.cout + bn - 1) / bn; P.tile_begin = tiles;
    P.msub = msub;
    const int m_step = cg * msub;
    const int tiles_p = (P.m_tiles + m_step - 1) / m_step * P.n_tiles;
    P.run = run; P.item_begin = items; items += (tiles_p + run - 1) / run;
    P.cnt_off = n_cnt; n_cnt += P.m_tiles;
    tiles += tiles_p;
    bn_max = std::max(bn_max, bn);
    P.seg_begin = int(segs.size()); P.n_seg = 2;
    long split = m / 3;
    for (int sgi = 0; sgi < 2; ++sgi) {
      GemmSeg g{};
      g.m_begin = sgi ? int(split) : 0; g.m_end = sgi ? int(m) : int(split);
      g.act = c.act; g.scale = b.sc; g.shift = b.sf;
      g.out = b.out + long(g.m_begin) * c.cout; g.ldo = c.cout;
      g.res = c.res ? (const void*)(b.res + long(g.m_begin) * c.cout) : nullptr; g.ldr = c.cout;
      const uint64_t rows = uint64_t(g.m_end - g.m_begin);
      if (tmap_encode_2d(&g.out_map, g.out, c.cout, rows, uint64_t(c.cout) * 2, 32, 32, 64)) return 2;
      if (g.res && tmap_encode_2d(&g.res_map, g.res, c.cout, rows, uint64_t(c.cout) * 2, 32, 32, 64)) return 3;
      segs.push_back(g);
    }
    flops += 2.0 * m * c.cout * c.k * c.k * c.cin;
    long tot = m * c.cout;
    ref_conv<<<(tot + 255) / 256, 256>>>(b.x, b.w, b.sc, b.sf, c.res ? b.res : nullptr, b.ref, c.n, c.h, c.w, c.cs,
                                         c.cin, cin_k, c.cout, c.k, c.s, c.p, c.d, ho, wo, c.act);
  }
  GemmProblem* dprobs; GemmSeg* dsegs;
  CK(cudaMalloc(&dprobs, probs.size() * sizeof(GemmProblem)));
  CK(cudaMalloc(&dsegs, segs.size() * sizeof(GemmSeg)));
  CK(cudaMemcpy(dprobs, probs.data(), probs.size() * sizeof(GemmProblem), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dsegs, segs.data(), segs.size() * sizeof(GemmSeg), cudaMemcpyHostToDevice));
  int32_t* dsched;
  const size_t sched_bytes = size_t(n_cnt) * 4;
  CK(cudaMalloc(&dsched, sched_bytes));
  CK(cudaMemset(dsched, 0, sched_bytes));
  GemmLaunch L{dprobs, dsegs, dsched, nullptr, int(probs.size()), tiles, items, bn_max, gemm_pick_stages(bn_max, cg), cg,
               bn_max * msub, getenv("TMA_STORE") ? atoi(getenv("TMA_STORE")) : 1, 0};
  if (argc > 4 && atoi(argv[4]) > 0) L.stages = atoi(argv[4]);
  const int dbg = argc > 3 ? atoi(argv[3]) : 0;
  int grid = std::min(tiles * cg, 148);
  if (cg == 1 && bn_max * msub > 256) { printf("MSUB x bn_max > 256\n"); return 1; }
  if (argc > 5) grid = atoi(argv[5]);
  printf("tiles=%d bn_max=%d stages=%d cg=%d smem=%zu\n", tiles, bn_max, L.stages, cg, gemm_smem_bytes(bn_max, L.stages, cg));
  CK((cudaError_t)gemm_launch(L, grid, 0));
  CK(cudaDeviceSynchronize());
  int bad = 0;
  for (size_t i = 0; i < cases.size(); ++i) {
    Bufs& b = bufs[i];
    long tot = b.m * cases[i].cout;
    std::vector<__nv_bfloat16> o(tot);
    std::vector<float> r(tot);
    CK(cudaMemcpy(o.data(), b.out, tot * 2, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(r.data(), b.ref, tot * 4, cudaMemcpyDeviceToHost));
    double mx = 0; long where = -1;
    for (long j = 0; j < tot; ++j) {
      double e = std::fabs(double(__bfloat162float(o[j])) - r[j]) / (std::fabs(r[j]) + 1e-2);
      if (!(e <= mx)) { mx = e; where = j; }
    }
    printf("case %zu M=%ld N=%d k=%d s=%d cs=%d: max rel err %.3e at %ld (got %f ref %f)\n", i, b.m, cases[i].cout,
           cases[i].k, cases[i].s, cases[i].cs, mx, where, where >= 0 ? __bfloat162float(o[where]) : 0.f,
           where >= 0 ? r[where] : 0.f);
    if (!(mx < 2e-2)) bad++;
  }
  if (bench) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    L.dbg = dbg;
    for (int it = 0; it < 3; ++it) { cudaMemsetAsync(dsched, 0, sched_bytes); gemm_launch(L, grid, 0); }
    cudaEventRecord(e0);
    const int iters = 20;
    for (int it = 0; it < iters; ++it) { cudaMemsetAsync(dsched, 0, sched_bytes); gemm_launch(L, grid, 0); }
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    ms /= iters;
    double tma = 0;
    for (auto& P : probs) {
      const double stage_bytes = 16384.0 + P.bn * 128.0;
      tma += double(P.m_tiles) * P.n_tiles * P.n_kstages * stage_bytes;
    }
    printf("grouped launch: %.3f ms, %.1f TFLOP/s (%.3f GFLOP), TMA operand traffic %.2f GB = %.2f TB/s\n", ms,
           flops / ms / 1e9, flops / 1e9, tma / 1e9, tma / ms / 1e9);
  }
  printf(bad ? "SELFTEST FAIL (%d)\n" : "SELFTEST OK\n", bad);
  return bad ? 1 : 0;
}
