// One recurrence step as a single tcgen05 kernel with a split-K cluster
// reduction in distributed shared memory (sm_100a, bf16 operands).
//
// Replaces, per time step, matmul_nt(h_t, W_rec) + input_forward + activate
// (backprop.hpp:102-112, rnn.hpp:209-216) in the forward direction and
// matmul_nn(dpre_{t+1}, W_rec) + the dh_out add + activate_deriv
// (backprop.hpp:204-218) in the backward direction.  The step is a small,
// latency-bound contraction (M = B streams <= 128, N = K = H), so instead of
// a split-K GEMM that round-trips S partial products through HBM, one
// cluster of S CTAs owns each 128 x BN output tile:
//   * CTA r of the cluster computes the partial product over K-slice r with
//     tcgen05.mma into TMEM (operands staged by TMA, SWIZZLE_128B),
//   * drains its fp32 partial to its own shared memory,
//   * after a cluster barrier, reduces rows [r*128/S, (r+1)*128/S) across
//     all S CTAs' shared memory (DSMEM) in fixed rank order -- deterministic --
//     and applies the fused epilogue (W_in row gather + sigmoid/tanh, or
//     + dh_out and * act'(h)), writing fp32 and bf16 copies.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "tc_common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace dl {
namespace tc {

constexpr int kRecThreads = 256;
constexpr int kRecCounters = 256;  // per-column-tile step counters (PersistParams::counter)
constexpr int kTrSlots = 8;        // DL_REC_TRACE stamps per step
#ifndef DL_REC_DIAG
#define DL_REC_DIAG 0  // timing diagnostics only (wrong results): 1 no MMAs in the persistent kernel
#endif

struct RecParams {
  int M, N, K;          // rows (streams), H, H
  int S, kbs;           // cluster size (K splits), k-blocks per split
  int mode;             // 0 forward, 1 backward
  int act;
  const float* w_in;    // fwd: embedding rows
  const uint32_t* x;    // fwd: input ids [M]
  const float* dh_out;  // bwd: [M x N]
  const float* hnext;   // bwd: h_{t+1} [M x N]
  float* out;           // h_{t+1} or dpre_t  [M x N]
  bf16* outb;           // bf16 copy (nullable)
};

template <int BN>
struct RecCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int NST = (160 * 1024) / STAGE > 8 ? 8 : (160 * 1024) / STAGE;
  static constexpr int PSTRIDE = BN + 4;  // fp32 partial row pitch (bank spread)
  static constexpr int PART_BYTES = BM * PSTRIDE * 4;
  static constexpr int RING = NST * STAGE;
  static constexpr int BODY = RING > PART_BYTES ? RING : PART_BYTES;
  static constexpr int SMEM = BODY + 1024 + 256;
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
};

template <int BN, bool B_MN>
__global__ void __launch_bounds__(kRecThreads, 1)
rec_step_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                RecParams p) {
  using C = RecCfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BODY);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::NST + 1);
  float* part = reinterpret_cast<float*>(smem);  // aliases the ring after the MMAs
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nt = blockIdx.y, mt = blockIdx.z;
  const uint32_t sbase = smem_u32(smem);
  auto full = [&](int s) { return smem_u32(&bars[s]); };
  auto empty = [&](int s) { return smem_u32(&bars[C::NST + s]); };
  const uint32_t tfull = smem_u32(&bars[2 * C::NST]);

  if (threadIdx.x == 32) {
    for (int s = 0; s < C::NST; ++s) { mbar_init(full(s), 1); mbar_init(empty(s), 1); }
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const int kb0 = rank * p.kbs;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    int stage = 0;
    uint32_t phase = 0;
    for (int i = 0; i < p.kbs; ++i) {
      const int kb = kb0 + i;
      mbar_wait(empty(stage), phase ^ 1);
      const uint32_t a_s = sbase + stage * C::STAGE;
      const uint32_t b_s = a_s + C::A_BYTES;
      mbar_expect_tx(full(stage), C::STAGE);
      tma_load_2d(a_s, &tmA, full(stage), kb * BK, mt * BM);
      if (!B_MN) {
        tma_load_2d(b_s, &tmB, full(stage), kb * BK, nt * BN);
      } else {
#pragma unroll
        for (int j = 0; j < BN / 64; ++j)
          tma_load_2d(b_s + j * 8192, &tmB, full(stage), nt * BN + 64 * j, kb * BK);
      }
      if (++stage == C::NST) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) |
                               (static_cast<uint32_t>(B_MN) << 16) |
                               (static_cast<uint32_t>(BN >> 3) << 17) |
                               (static_cast<uint32_t>(BM >> 4) << 24);
    int stage = 0;
    uint32_t phase = 0;
    for (int i = 0; i < p.kbs; ++i) {
      mbar_wait(full(stage), phase);
      fence_after();
      const uint32_t a_s = sbase + stage * C::STAGE;
      const uint32_t b_s = a_s + C::A_BYTES;
#pragma unroll
      for (int ks = 0; ks < BK / UMMA_K; ++ks) {
        const uint64_t ad = make_desc(a_s + ks * 32, 16, 1024);
        const uint64_t bd = B_MN ? make_desc(b_s + ks * 2048, 8192, 1024)
                                 : make_desc(b_s + ks * 32, 16, 1024);
        mma_bf16(tmem, ad, bd, idesc, (i > 0 || ks > 0) ? 1u : 0u);
      }
      mma_commit(empty(stage));
      if (++stage == C::NST) { stage = 0; phase ^= 1; }
    }
    mma_commit(tfull);
  }
  __syncwarp();

  // ---- drain TMEM -> own shared memory (fp32 partial of this K slice)
  mbar_wait(tfull, 0);
  fence_after();
  {
    const int quarter = warp % 4;
    const int half = warp / 4;  // 8 warps: two column halves per lane quarter
    const int row = quarter * 32 + lane;
    float* prow = part + row * C::PSTRIDE;
#pragma unroll 1
    for (int c = half * (BN / 64); c < (half + 1) * (BN / 64); ++c) {
      float v[32];
      tmem_ld32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + c * 32, v);
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(prow + c * 32 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    }
  }
  fence_before();
  cluster.sync();  // every CTA's partial is visible cluster-wide

  // ---- reduce my row slice across the cluster (rank order), fused epilogue
  // 16-byte DSMEM loads: each thread owns 4 consecutive columns (N % 8 == 0
  // in bf16 mode, so a 4-column group never straddles the N edge)
  const int rows = BM / p.S;
  const int r0 = rank * rows;
  constexpr int Q = BN / 4;
  for (int idx = threadIdx.x; idx < rows * Q; idx += kRecThreads) {
    const int row = r0 + idx / Q, col = 4 * (idx % Q);
    const int m = mt * BM + row, n = nt * BN + col;
    if (m >= p.M || n >= p.N) continue;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int q = 0; q < p.S; ++q) {
      const float* peer = cluster.map_shared_rank(part, q);
      const float4 v = *reinterpret_cast<const float4*>(peer + row * C::PSTRIDE + col);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    const int64_t o = static_cast<int64_t>(m) * p.N + n;
    float4 y;
    if (p.mode == 0) {
      const float4 e = *reinterpret_cast<const float4*>(p.w_in + static_cast<int64_t>(p.x[m]) * p.N + n);
      y = make_float4(act_f(p.act, acc.x + e.x), act_f(p.act, acc.y + e.y),
                      act_f(p.act, acc.z + e.z), act_f(p.act, acc.w + e.w));
    } else {
      const float4 d = *reinterpret_cast<const float4*>(p.dh_out + o);
      const float4 h = *reinterpret_cast<const float4*>(p.hnext + o);
      y = make_float4((acc.x + d.x) * act_deriv_f(p.act, h.x), (acc.y + d.y) * act_deriv_f(p.act, h.y),
                      (acc.z + d.z) * act_deriv_f(p.act, h.z), (acc.w + d.w) * act_deriv_f(p.act, h.w));
    }
    *reinterpret_cast<float4*>(p.out + o) = y;
    if (p.outb) {
      __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(p.outb + o);
      ob[0] = __floats2bfloat162_rn(y.x, y.y);
      ob[1] = __floats2bfloat162_rn(y.z, y.w);
    }
  }
  cluster.sync();  // peers are done reading my shared memory
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(C::TMEM_COLS));
  }
}

template <int BN, bool B_MN>
void rec_launch(const void* A, const void* Bw, RecParams p, cudaStream_t st) {
  using Cf = RecCfg<BN>;
  auto kern = rec_step_kernel<BN, B_MN>;
  static std::once_flag once;
  std::call_once(once, [&] {
    DL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
    DL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  });
  const CUtensorMap ta = make_map(A, p.M, p.K, p.K, BM);
  const CUtensorMap tb = B_MN ? make_map(Bw, p.K, p.N, p.N, 64) : make_map(Bw, p.N, p.K, p.K, BN);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.S, (p.N + BN - 1) / BN, (p.M + BM - 1) / BM);
  cfg.blockDim = dim3(kRecThreads);
  cfg.dynamicSmemBytes = Cf::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DL_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, p));
}

// --------------------------------------------------------------------------
// Persistent variant: ONE launch runs all T steps of the forward (or
// backward) recurrence of a window.  Each CTA keeps its W_rec slice
// (BN x K/S bf16) resident in shared memory for the whole window and only
// streams its K-slice of h_t (or dpre_{t+1}) per step; steps are separated
// by a grid-wide barrier on a global arrival counter (all CTAs co-resident:
// cooperative cluster launch).  Per step: TMA A -> tcgen05.mma -> TMEM ->
// shared fp32 partial -> cluster barrier -> DSMEM rank-ordered reduction +
// fused epilogue -> global h_{t+1} / dpre_t (fp32 + bf16) -> arrive.
struct PersistParams {
  int M, N, K, S, kbs, T, mode, act;
  int64_t MN;
  const float* w_in;
  const uint32_t* x;      // fwd: ids of step s at x + s*M
  const float* dh_out;    // bwd: [T][M][N]
  const float* htape;     // bwd: h tape [T+1][M][N] (act' argument)
  float* out;             // fwd: htape (writes step s+1); bwd: dpre (writes step s)
  bf16* outb;
  unsigned* counter;      // [kRecCounters] per column-tile cluster, zeroed before the launch
  unsigned long long* trace;  // DL_REC_TRACE: [4 CTAs][T][kTrSlots] %globaltimer stamps, or null
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <int BN>
struct PersistCfg {
  static constexpr int A_BLK = BM * BK * 2;  // 16 KB
  static constexpr int B_BLK = BN * BK * 2;
  static constexpr int PSTRIDE = BN + 4;
  static constexpr int PART = BM * PSTRIDE * 4;
  static constexpr int MAXKB = BN <= 64 ? 8 : 4;  // resident W_rec k-blocks per CTA
  // A ring: every k-block of the CTA's K-slice in flight at once; the fp32
  // partial reuses it once the step's MMAs have completed (peers read it
  // before anyone passes the next step's dependency wait)
  static constexpr int NA = MAXKB;
  static constexpr int RING = NA * A_BLK > PART ? NA * A_BLK : PART;
  static constexpr int SMEM = RING + MAXKB * B_BLK + 1024 + 256;
  static constexpr int NPRE = 4;  // epilogue float4 operands prefetched per thread
};

__device__ __forceinline__ unsigned rec_ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Step dependencies are tracked per producing cluster: counter[c] counts
// the CTAs of column-tile cluster c that have published a step (S per
// step).  The k-block of A holding columns [64 kb, 64 kb + 64) was written
// by cluster 64 kb / BN, so each A load waits only for its own producers
// -- no grid-wide barrier -- and the TMA stream starts as soon as the first
// needed tile is out.
template <int BN, bool B_MN>
__global__ void __launch_bounds__(kRecThreads, 1)
rec_persist_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   PersistParams p) {
  using C = PersistCfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;                                 // NA-stage ring of 16 KB
  uint8_t* sB = smem + C::RING;                       // kbs x B_BLK, resident
  float* part = reinterpret_cast<float*>(sA);         // fp32 partial (after the MMAs)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + C::MAXKB * C::B_BLK);
  // bars: full[NA], empty[NA], barB, tfull
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::NA + 2);
  auto fullA = [&](int s) { return smem_u32(&bars[s]); };
  auto emptyA = [&](int s) { return smem_u32(&bars[C::NA + s]); };
  const uint32_t barB = smem_u32(&bars[2 * C::NA]), tfull = smem_u32(&bars[2 * C::NA + 1]);
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nt = blockIdx.y;

  if (threadIdx.x == 32) {
    for (int s = 0; s < C::NA; ++s) { mbar_init(fullA(s), 1); mbar_init(emptyA(s), 1); }
    mbar_init(barB, 1);
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  int a_stage = 0;       // A ring position, persistent across steps
  uint32_t a_phase = 0;  // (producer and MMA lanes advance identical copies)
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(BN < 32 ? 32 : BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const int kb0 = rank * p.kbs;
  const int rows = BM / p.S, r0 = rank * rows;
  constexpr int Q = BN / 4;
  const int nwork = rows * Q;  // float4 outputs of this CTA per step

  // resident W_rec slice, loaded once
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    mbar_expect_tx(barB, p.kbs * C::B_BLK);
    for (int i = 0; i < p.kbs; ++i) {
      const uint32_t b_s = smem_u32(sB + i * C::B_BLK);
      if (!B_MN) {
        tma_load_2d(b_s, &tmB, barB, (kb0 + i) * BK, nt * BN);
      } else {
#pragma unroll
        for (int j = 0; j < BN / 64; ++j)
          tma_load_2d(b_s + j * 8192, &tmB, barB, nt * BN + 64 * j, (kb0 + i) * BK);
      }
    }
  }

  // trace: CTAs (rank 0, column tiles 0, 8, 16, 24)
  unsigned long long* tr =
      (p.trace && rank == 0 && nt % 8 == 0 && nt < 32) ? p.trace + (nt / 8) * p.T * kTrSlots : nullptr;
  for (int j = 0; j < p.T; ++j) {
    const int s = p.mode == 0 ? j : p.T - 1 - j;   // time step written this iteration
    const bool gemm = p.mode == 0 || j > 0;        // bwd t = T-1 has no recurrent term
    const uint32_t ph = (p.mode == 0 ? j : j - 1) & 1;
    if (tr && threadIdx.x == 0) tr[j * kTrSlots + 0] = gtimer();
    // epilogue operands do not depend on the recurrence: issue their loads
    // now so they land while this step waits for its inputs
    float4 pre_a[C::NPRE], pre_b[C::NPRE];
#pragma unroll
    for (int k = 0; k < C::NPRE; ++k) {
      const int idx = threadIdx.x + k * kRecThreads;
      if (idx >= nwork) break;
      const int m = r0 + idx / Q, n = nt * BN + 4 * (idx % Q);
      if (m >= p.M || n >= p.N) continue;
      const int64_t o = static_cast<int64_t>(m) * p.N + n;
      if (p.mode == 0) {
        pre_a[k] = *reinterpret_cast<const float4*>(
            p.w_in + static_cast<int64_t>(p.x[s * p.M + m]) * p.N + n);
      } else {
        pre_a[k] = *reinterpret_cast<const float4*>(p.dh_out + s * p.MN + o);
        pre_b[k] = *reinterpret_cast<const float4*>(p.htape + (s + 1) * p.MN + o);
      }
    }
    if (gemm) {
      if (warp == 0) {
        const int arow = p.mode == 0 ? s * p.M : (s + 1) * p.M;
        const unsigned target = (unsigned)p.S * (unsigned)j;
        if (j > 0) {
          // wait for (a) my cluster peers -- they have finished reading my
          // partial, which lives in the A ring these loads overwrite -- and
          // (b) the producers of each k-block of my K-slice.  Lane i < kbs
          // polls k-block i's producer counter, lane kbs my own cluster's,
          // all in parallel (acquire loads: a fence would also wait for the
          // in-flight epilogue prefetches)
          const unsigned* cnt = lane < p.kbs ? p.counter + ((kb0 + lane) * BK) / BN
                                             : p.counter + nt;
          long spins = 0;
          bool ok = lane > p.kbs;
          while (!__all_sync(0xffffffffu, ok)) {
            if (!ok) ok = rec_ld_acquire(cnt) >= target;
            if (++spins > (1l << 28)) __trap();
          }
          __syncwarp();  // order lane 0's loads after every lane's acquire
        }
        if (lane == 0) {
          if (tr) tr[j * kTrSlots + 1] = gtimer();
          if (j > 0) asm volatile("fence.proxy.async.global;" ::: "memory");
          for (int i = 0; i < p.kbs; ++i) {
            mbar_wait(emptyA(a_stage), a_phase ^ 1);
            mbar_expect_tx(fullA(a_stage), C::A_BLK);
            tma_load_2d(smem_u32(sA + a_stage * C::A_BLK), &tmA, fullA(a_stage), (kb0 + i) * BK,
                        arow);
            if (++a_stage == C::NA) { a_stage = 0; a_phase ^= 1; }
          }
          if (tr) tr[j * kTrSlots + 7] = gtimer();
        }
      } else if (warp == 2 && lane == 0 && tr) {
        // (trace) when the first / last k-block of the step has landed
        int st2 = a_stage;
        uint32_t ph2 = a_phase;
        for (int i = 0; i < p.kbs; ++i) {
          mbar_wait(fullA(st2), ph2);
          if (i == 0 || i == p.kbs - 1) tr[j * kTrSlots + (i == 0 ? 5 : 6)] = gtimer();
          if (++st2 == C::NA) { st2 = 0; ph2 ^= 1; }
        }
      } else if (warp == 1 && lane == 0) {
        constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) |
                                   (static_cast<uint32_t>(B_MN) << 16) |
                                   (static_cast<uint32_t>(BN >> 3) << 17) |
                                   (static_cast<uint32_t>(BM >> 4) << 24);
        if (j == (p.mode == 0 ? 0 : 1)) mbar_wait(barB, 0);
        for (int i = 0; i < p.kbs; ++i) {
          mbar_wait(fullA(a_stage), a_phase);
          fence_after();
          const uint32_t a_s = smem_u32(sA + a_stage * C::A_BLK);
          const uint32_t b_s = smem_u32(sB + i * C::B_BLK);
#pragma unroll
          for (int ks = 0; ks < BK / UMMA_K; ++ks) {
            const uint64_t ad = make_desc(a_s + ks * 32, 16, 1024);
            const uint64_t bd = B_MN ? make_desc(b_s + ks * 2048, 8192, 1024)
                                     : make_desc(b_s + ks * 32, 16, 1024);
#if !(DL_REC_DIAG & 1)
            mma_bf16(tmem, ad, bd, idesc, (i > 0 || ks > 0) ? 1u : 0u);
#endif
          }
          mma_commit(emptyA(a_stage));
          if (++a_stage == C::NA) { a_stage = 0; a_phase ^= 1; }
        }
        mma_commit(tfull);
      }
      __syncwarp();
      mbar_wait(tfull, ph);
      fence_after();
      if (tr && threadIdx.x == 64) tr[j * kTrSlots + 2] = gtimer();
      {
        // the A ring is idle now (all MMAs of the step completed): drain the
        // accumulator into it as this CTA's fp32 partial (peers pull their
        // row slices from it; pushing instead -- DSMEM stores -- measured
        // slower: the cluster barrier then waits for the remote stores)
        const int quarter = warp % 4, half = warp / 4;
        float* prow = part + (quarter * 32 + lane) * C::PSTRIDE;
#pragma unroll 1
        for (int c = half * (BN / 64); c < (half + 1) * (BN / 64); ++c) {
          float v[32];
          tmem_ld32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + c * 32, v);
#pragma unroll
          for (int q = 0; q < 32; q += 4)
            *reinterpret_cast<float4*>(prow + c * 32 + q) =
                make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
        }
      }
      fence_before();
      cluster.sync();
      if (tr && threadIdx.x == 64) tr[j * kTrSlots + 3] = gtimer();
    }
    // reduce my row slice over the cluster (rank order) + fused epilogue.
    // Only the bf16 copy feeds the next step (its TMA loads): it is stored
    // and published first, the fp32 copy (read by later kernels) after.
    float4 ys[C::NPRE];
    int64_t yo[C::NPRE];
#pragma unroll
    for (int k = 0; k < C::NPRE; ++k) yo[k] = -1;
#pragma unroll 1
    for (int k = 0; k * kRecThreads < nwork; ++k) {
      const int idx = threadIdx.x + k * kRecThreads;
      if (idx >= nwork) break;
      const int row = r0 + idx / Q, col = 4 * (idx % Q);
      const int m = row, n = nt * BN + col;
      if (m >= p.M || n >= p.N) continue;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gemm) {
        // every peer's partial in flight at once (distributed shared memory
        // round trips dominate), then summed in rank order as before
        float4 pv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < p.S) {
            const float* peer = cluster.map_shared_rank(part, q);
            pv[q] = *reinterpret_cast<const float4*>(peer + row * C::PSTRIDE + col);
          }
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < p.S) {
            acc.x += pv[q].x; acc.y += pv[q].y; acc.z += pv[q].z; acc.w += pv[q].w;
          }
      }
      const int64_t o = static_cast<int64_t>(m) * p.N + n;
      float4 ea, eb;
      if (k < C::NPRE) {
        // (k is uniform, the prefetch arrays are indexed by a constant)
#pragma unroll
        for (int kk = 0; kk < C::NPRE; ++kk)
          if (kk == k) { ea = pre_a[kk]; eb = pre_b[kk]; }
      } else if (p.mode == 0) {
        ea = *reinterpret_cast<const float4*>(
            p.w_in + static_cast<int64_t>(p.x[s * p.M + m]) * p.N + n);
      } else {
        ea = *reinterpret_cast<const float4*>(p.dh_out + s * p.MN + o);
        eb = *reinterpret_cast<const float4*>(p.htape + (s + 1) * p.MN + o);
      }
      float4 y;
      int64_t oo;
      if (p.mode == 0) {
        y = make_float4(act_f(p.act, acc.x + ea.x), act_f(p.act, acc.y + ea.y),
                        act_f(p.act, acc.z + ea.z), act_f(p.act, acc.w + ea.w));
        oo = (s + 1) * p.MN + o;
      } else {
        y = make_float4((acc.x + ea.x) * act_deriv_f(p.act, eb.x),
                        (acc.y + ea.y) * act_deriv_f(p.act, eb.y),
                        (acc.z + ea.z) * act_deriv_f(p.act, eb.z),
                        (acc.w + ea.w) * act_deriv_f(p.act, eb.w));
        oo = s * p.MN + o;
      }
      __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(p.outb + oo);
      ob[0] = __floats2bfloat162_rn(y.x, y.y);
      ob[1] = __floats2bfloat162_rn(y.z, y.w);
      bool kept = false;
#pragma unroll
      for (int kk = 0; kk < C::NPRE; ++kk)
        if (kk == k) { ys[kk] = y; yo[kk] = oo; kept = true; }
      if (!kept) *reinterpret_cast<float4*>(p.out + oo) = y;
    }
    // publish this step to the consumers of this column tile (generic
    // stores -> visible to their TMA loads)
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncthreads();
    if (tr && threadIdx.x == 0) tr[j * kTrSlots + 4] = gtimer();
    if (threadIdx.x == 0)
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.counter + nt) : "memory");
#pragma unroll
    for (int k = 0; k < C::NPRE; ++k)
      if (yo[k] >= 0) *reinterpret_cast<float4*>(p.out + yo[k]) = ys[k];
  }
  cluster.sync();  // peers are done reading my shared memory
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(BN < 32 ? 32 : BN));
  }
}

template <int BN, bool B_MN>
bool persist_launch(const void* A_tape, int64_t a_rows, const void* Bw, PersistParams p,
                    cudaStream_t st) {
  using Cf = PersistCfg<BN>;
  auto kern = rec_persist_kernel<BN, B_MN>;
  static std::once_flag once;
  std::call_once(once, [&] {
    DL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
    DL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  });
  const CUtensorMap ta = make_map(A_tape, a_rows, p.K, p.K, BM);
  const CUtensorMap tb = B_MN ? make_map(Bw, p.K, p.N, p.N, 64) : make_map(Bw, p.N, p.K, p.K, BN);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.S, (p.N + BN - 1) / BN, 1);
  cfg.blockDim = dim3(kRecThreads);
  cfg.dynamicSmemBytes = Cf::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // The grid barrier needs every CTA resident at once: only launch when the
  // device can host all clusters simultaneously (then nothing can starve
  // them: other work on the GPU is finite and never waits on this kernel).
  static int max_clusters[4] = {-1, -1, -1, -1};  // per cluster size 1, 2, 4, 8
  const int si = p.S == 1 ? 0 : p.S == 2 ? 1 : p.S == 4 ? 2 : 3;
  if (max_clusters[si] < 0) {
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    max_clusters[si] = n;
  }
  const int need = (int)(cfg.gridDim.x * cfg.gridDim.y / p.S);
  if (max_clusters[si] < need) return false;
  DL_REQUIRE((p.N + BN - 1) / BN <= kRecCounters, 1, "recurrence: too many column tiles");
  DL_CUDA(cudaMemsetAsync(p.counter, 0, kRecCounters * sizeof(unsigned), st));
  DL_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, p));
  return true;
}

}  // namespace tc

// All T steps of a window's recurrence in one persistent launch; returns
// false (nothing launched) when the shape or the device cannot host it, in
// which case the caller uses the per-step kernels.
bool rec_window_tc(int mode, int T, int M, int H, int act, const bf16* a_tape, int64_t a_rows,
                   const bf16* w_rec_bf, const float* w_in, const uint32_t* x,
                   const float* dh_out, const float* htape, float* out, bf16* outb,
                   unsigned* counter, cudaStream_t st) {
  static const bool enabled = [] {
    const char* e = std::getenv("DL_REC_PERSIST");
    return !(e && std::atoi(e) == 0);
  }();
  if (!enabled || M > tc::BM || T < 1) return false;
  const int kb_total = (H + 63) / 64;
  // candidates in preference order (BN = 256 cannot keep W_rec + partials
  // resident); the first whose clusters all fit on the device launches
  int cand[8][2] = {{64, 4}, {128, 8}, {64, 8}, {128, 4}, {64, 2}, {128, 2}, {64, 1}, {128, 1}};
  if (const char* e = std::getenv("DL_REC_PCAND")) {  // tuning: "BN,S" tried first
    int b = 0, k = 0;
    if (std::sscanf(e, "%d,%d", &b, &k) == 2) { cand[0][0] = b; cand[0][1] = k; }
  }
  tc::PersistParams p{};
  p.M = M; p.N = H; p.K = H; p.T = T; p.mode = mode; p.act = act;
  p.MN = (int64_t)M * H;
  p.w_in = w_in; p.x = x; p.dh_out = dh_out; p.htape = htape;
  p.out = out; p.outb = outb; p.counter = counter;
  static unsigned long long* trace = nullptr;
  static const bool tracing = std::getenv("DL_REC_TRACE") != nullptr;
  if (tracing) {
    if (!trace) DL_CUDA(cudaMalloc(&trace, 4 * 64 * tc::kTrSlots * sizeof(unsigned long long)));
    DL_CUDA(cudaMemsetAsync(trace, 0, 4 * 64 * tc::kTrSlots * sizeof(unsigned long long), st));
    p.trace = T <= 64 ? trace : nullptr;
  }
  const bool bmn = mode == 1;
  bool ok = false;
  int bn = 0, S = 0;
  for (int ci = 0; ci < 8 && !ok; ++ci) {
    bn = cand[ci][0];
    S = cand[ci][1];
    const int maxkb = bn <= 64 ? tc::PersistCfg<64>::MAXKB : tc::PersistCfg<128>::MAXKB;
    if (H % bn || kb_total % S || kb_total / S > maxkb || (H / bn) * S > 148) continue;
    p.S = S;
    p.kbs = kb_total / S;
    if (bn == 64)
      ok = bmn ? tc::persist_launch<64, true>(a_tape, a_rows, w_rec_bf, p, st)
               : tc::persist_launch<64, false>(a_tape, a_rows, w_rec_bf, p, st);
    else
      ok = bmn ? tc::persist_launch<128, true>(a_tape, a_rows, w_rec_bf, p, st)
               : tc::persist_launch<128, false>(a_tape, a_rows, w_rec_bf, p, st);
  }
  if (std::getenv("DL_DEBUG"))
    fprintf(stderr, "[desklm] persistent recurrence mode=%d T=%d M=%d H=%d BN=%d S=%d -> %s\n",
            mode, T, M, H, bn, S, ok ? "launched" : "fallback");
  if (ok && p.trace) {
    // per-step phase durations (ns, CTA-averaged): wait, load+mma, reduce
    // (drain + cluster sync), epilogue+publish; and step-to-step period
    std::vector<unsigned long long> h(4 * T * tc::kTrSlots);
    DL_CUDA(cudaStreamSynchronize(st));
    DL_CUDA(cudaMemcpy(h.data(), p.trace, h.size() * 8, cudaMemcpyDeviceToHost));
    double ph[5] = {0, 0, 0, 0, 0}, ex[3] = {0, 0, 0};
    int n = 0;
    for (int c = 0; c < 4; ++c)
      for (int j = 1; j + 1 < T; ++j) {
        const unsigned long long* r = &h[(c * T + j) * tc::kTrSlots];
        const unsigned long long* q = &h[(c * T + j + 1) * tc::kTrSlots];
        if (!r[0] || !r[4] || !q[0]) continue;
        ph[0] += (double)(r[1] - r[0]);
        ph[1] += (double)(r[2] - r[1]);
        ph[2] += (double)(r[3] - r[2]);
        ph[3] += (double)(r[4] - r[3]);
        ph[4] += (double)(q[0] - r[0]);
        if (r[5] && r[6] && r[7]) {
          ex[0] += (double)(r[7] - r[1]);  // TMA issue loop
          ex[1] += (double)(r[5] - r[1]);  // first k-block landed
          ex[2] += (double)(r[6] - r[1]);  // last k-block landed
        }
        ++n;
      }
    if (n)
      fprintf(stderr, "[desklm] rec trace mode=%d: wait %.0f  load+mma %.0f  drain+sync %.0f  "
              "epilogue %.0f  period %.0f ns\n", mode, ph[0] / n, ph[1] / n, ph[2] / n,
              ph[3] / n, ph[4] / n);
    if (n)
      fprintf(stderr, "[desklm] rec trace mode=%d: after deps: issue loop %.0f  first k-block %.0f  "
              "last k-block %.0f ns\n", mode, ex[0] / n, ex[1] / n, ex[2] / n);
  }
  return ok;
}

// Tile choice for a recurrence step: BN in {64,128,256} and S in {1,2,4,8}
// K-slices (each >= one 64-wide k-block) to put ~128 CTAs on the 148 SMs.
void rec_plan(int M, int H, int& bn, int& S) {
  const int kb_total = (H + 63) / 64;
  const int m_tiles = (M + 127) / 128;
  int best = -1;
  double best_score = 1e30;
  const int bns[3] = {256, 128, 64};
  for (int bi = 0; bi < 3; ++bi)
    for (int s = 8; s >= 1; s >>= 1) {
      const int b = bns[bi];
      if (s > kb_total || (kb_total % s) != 0) continue;
      if (b > 64 && H < b) continue;
      const int ctas = m_tiles * ((H + b - 1) / b) * s;
      if (ctas > 148) continue;
      // prefer ~128 CTAs, then fewer K slices (less DSMEM traffic)
      const double score = std::abs(128 - ctas) + 0.5 * s;
      if (score < best_score) { best_score = score; best = bi * 16 + s; }
    }
  if (best < 0) { bn = 64; S = 1; return; }
  bn = bns[best / 16];
  S = best % 16;
  // tuning overrides (bench sweeps): DL_REC_BN, DL_REC_S
  if (const char* e = std::getenv("DL_REC_BN")) {
    const int v = std::atoi(e);
    if ((v == 64 || v == 128 || v == 256) && H >= v) bn = v;
  }
  if (const char* e = std::getenv("DL_REC_S")) {
    const int v = std::atoi(e);
    if ((v == 1 || v == 2 || v == 4 || v == 8) && kb_total % v == 0) S = v;
  }
}

void rec_step_tc(int mode, int M, int H, int act, const bf16* A, const bf16* w_rec_bf,
                 const float* w_in, const uint32_t* x, const float* dh_out, const float* hnext,
                 float* out, bf16* outb, cudaStream_t st) {
  int bn, S;
  rec_plan(M, H, bn, S);
  tc::RecParams p{};
  p.M = M; p.N = H; p.K = H;
  p.S = S;
  p.kbs = ((H + 63) / 64) / S;
  p.mode = mode;
  p.act = act;
  p.w_in = w_in; p.x = x; p.dh_out = dh_out; p.hnext = hnext;
  p.out = out; p.outb = outb;
  const bool bmn = mode == 1;  // backward contracts over the first index of W_rec
#define DL_REC_CASE(BN_)                                           \
  if (bn == BN_) {                                                 \
    if (bmn) tc::rec_launch<BN_, true>(A, w_rec_bf, p, st);        \
    else tc::rec_launch<BN_, false>(A, w_rec_bf, p, st);           \
    return;                                                        \
  }
  DL_REC_CASE(256)
  DL_REC_CASE(128)
  DL_REC_CASE(64)
#undef DL_REC_CASE
}

}  // namespace dl
