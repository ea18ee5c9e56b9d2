// tcgen05 / TMEM / TMA GEMM for sm_100a (bf16 operands, fp32 accumulate).
//
// One persistent, warp-specialised kernel serves every dense contraction of
// the RNNLM window, replacing mat.hpp:116-184:
//   logits      S  = Hs . W_out^T    (A K-major, B K-major)  + online-LSE epilogue
//   dh_out      dH = dS . W_out      (A K-major, B MN-major)
//   dW_out      dW = dS^T . Hs       (A MN-major, B MN-major) + clip epilogue
//   recurrence  h  . W_rec^T / dpre . W_rec                     (split-K slices)
//   dW_rec      dW = dpre^T . Hprev  (A MN-major, B MN-major)   (split-K slices)
//
// Roles (192 threads): warp 0 = TMA producer (one elected lane), warp 1 =
// MMA issuer (one lane issues tcgen05.mma for the whole CTA), warps 2-5 =
// epilogue (tcgen05.ld TMEM -> registers; warp w owns TMEM lanes
// 32*(w%4)..+31, i.e. one accumulator row per thread).  Tiles are 128 x BN
// with BK = 64 (one 128-byte swizzle row of bf16); the accumulator is double
// buffered in TMEM (2 x BN fp32 columns) so the epilogue of tile i overlaps
// the MMAs of tile i+1.  Operands arrive by TMA with SWIZZLE_128B into the
// canonical UMMA layouts:
//   K-major  tile: rows of 128 B, 8-row groups 1024 B apart (SBO = 1024)
//   MN-major tile: 64-element (128 B) MN chunks 8 KB apart (LBO = 8192),
//                  each chunk 64 K-rows of 128 B, 8-row groups (SBO = 1024)
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "tc_common.cuh"

namespace dl {
namespace tc {

// warp 0 TMA producer, warp 1 MMA issuer, warps 2..9 epilogue: two warps
// per TMEM lane quarter, each draining half of the tile's columns
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES = (192 * 1024) / STAGE > 8 ? 8 : (192 * 1024) / STAGE;
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
};

struct Sched {
  int m_tiles, n_tiles, k_splits, kb_total, kbps, raster;
  __device__ void decode(int u, int& mt, int& nt, int& kb0, int& kb1) const {
    const int s = u % k_splits;
    const int t = u / k_splits;
    if (raster == 0) { mt = t % m_tiles; nt = t / m_tiles; }
    else { nt = t % n_tiles; mt = t / n_tiles; }
    kb0 = s * kbps;
    kb1 = min(kb_total, kb0 + kbps);
  }
};

template <int BN>
__device__ __forceinline__ void epilogue_row(const GemmDesc& g, uint32_t taddr, int m, int nt,
                                             int split, bool& bad, int c0, int c1, int sub);

// 2^x on the SFU (ex2.approx, flush-to-zero): the online-LSE epilogue's
// exponentials never need the denormal range
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(kThreads, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               GemmDesc g, Sched sc) {
  using C = Cfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  // bars: full[STAGES], empty[STAGES], tfull[2], tempty[2]; then tmem slot
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::STAGES + 4);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t sbase = smem_u32(smem);
  auto full = [&](int s) { return smem_u32(&bars[s]); };
  auto empty = [&](int s) { return smem_u32(&bars[C::STAGES + s]); };
  auto tfull = [&](int a) { return smem_u32(&bars[2 * C::STAGES + a]); };
  auto tempty = [&](int a) { return smem_u32(&bars[2 * C::STAGES + 2 + a]); };

  if (threadIdx.x == 32) {
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(full(s), 1); mbar_init(empty(s), 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(tfull(a), 1); mbar_init(tempty(a), kEpiWarps); }
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
  const uint32_t tmem_base = *tmem_slot;
  const int total = sc.m_tiles * sc.n_tiles * sc.k_splits;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < total; u += gridDim.x) {
        int mt, nt, kb0, kb1;
        sc.decode(u, mt, nt, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(empty(stage), phase ^ 1);
          const uint32_t a_s = sbase + stage * C::STAGE;
          const uint32_t b_s = a_s + C::A_BYTES;
          mbar_expect_tx(full(stage), C::STAGE);
          if (!A_MN) {
            tma_load_2d(a_s, &tmA, full(stage), kb * BK, mt * BM);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              tma_load_2d(a_s + j * 8192, &tmA, full(stage), mt * BM + 64 * j, kb * BK);
          }
          if (!B_MN) {
            tma_load_2d(b_s, &tmB, full(stage), kb * BK, nt * BN);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d(b_s + j * 8192, &tmB, full(stage), nt * BN + 64 * j, kb * BK);
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) |
                                 (static_cast<uint32_t>(A_MN) << 15) |
                                 (static_cast<uint32_t>(B_MN) << 16) |
                                 (static_cast<uint32_t>(BN >> 3) << 17) |
                                 (static_cast<uint32_t>(BM >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = blockIdx.x; u < total; u += gridDim.x) {
        int mt, nt, kb0, kb1;
        sc.decode(u, mt, nt, kb0, kb1);
        mbar_wait(tempty(acc), acc_phase ^ 1);
        fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(full(stage), phase);
          fence_after();
          const uint32_t a_s = sbase + stage * C::STAGE;
          const uint32_t b_s = a_s + C::A_BYTES;
#pragma unroll
          for (int ks = 0; ks < BK / UMMA_K; ++ks) {
            const uint64_t ad = A_MN ? make_desc(a_s + ks * 2048, 8192, 1024)
                                     : make_desc(a_s + ks * 32, 16, 1024);
            const uint64_t bd = B_MN ? make_desc(b_s + ks * 2048, 8192, 1024)
                                     : make_desc(b_s + ks * 32, 16, 1024);
            mma_bf16(d, ad, bd, idesc, (kb > kb0 || ks > 0) ? 1u : 0u);
          }
          mma_commit(empty(stage));
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(tfull(acc));
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ---------------- epilogue (warps 2..5)
    const int quarter = warp % 4, half = (warp - 2) / 4;
    const int row = quarter * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    bool bad = false;
    for (int u = blockIdx.x; u < total; u += gridDim.x) {
      int mt, nt, kb0, kb1;
      sc.decode(u, mt, nt, kb0, kb1);
      const int split = u % sc.k_splits;
      mbar_wait(tfull(acc), acc_phase);
      fence_after();
      const int m = mt * BM + row;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN;
      epilogue_row<BN>(g, taddr, m, nt, split, bad, half * (BN / 64), (half + 1) * (BN / 64),
                       2 * nt + half);
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty(acc));
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (g.do_clip && g.nonfinite && bad) atomicExch(g.nonfinite, 1);
  }
  fence_before();
  __syncthreads();
  if (warp == 0) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(C::TMEM_COLS));
  }
}

// --------------------------------------------------------------------------
// CTA-pair variant (tcgen05 cta_group::2): a cluster of 2 CTAs on one TPC
// computes a 256 x 256 tile with M = 256 MMAs issued by the even CTA.  Each
// CTA stages its own 128 rows of A and half (128 columns) of B, so every
// CTA moves 32 KB per 64-deep k-block instead of 48 KB for the same tensor
// work (1/3 less L2->SM traffic) and fits a 6-deep pipeline.  Both CTAs'
// TMA transactions complete on the even CTA's full barrier; its MMA commits
// multicast to both CTAs' empty / tmem-full barriers; both epilogues drain
// their own TMEM half (128 rows x 256 columns) and arrive remotely on the
// even CTA's tmem-empty barrier.
// RMS: the fused-rmsprop variant trades k-stages (3 instead of 6) for a
// per-epilogue-warp buffer of the warp's whole pass-2 master slice: four
// 32 x 32 fp32 chunks (4 KB each, 16-byte units XOR swizzled by row) filled
// by cp.async, all in flight at once (measured: 3 stages + 4 chunks beat
// 5 + 2 and 4 + 2/3 by 1-2% on the C3 dW_out).
#ifndef DL_PAIR_STAGES
#define DL_PAIR_STAGES 6
#endif
#ifndef DL_RMS_STAGES
#define DL_RMS_STAGES 3
#endif
#ifndef DL_RMS_RING
#define DL_RMS_RING 4  // cp.async chunks of the fp32 master in flight per warp (all of pass 2)
#endif
#ifndef DL_XF_DIAG
#define DL_XF_DIAG 0  // timing diagnostics of the dS transform (wrong results): 1 no math,
                      // 2 no proxy fence, 4 no cross-CTA handshake, 8 no smem pass,
                      // 16 no dS stores, 32 producer ignores `stored`
#endif
#ifndef DL_RMS_PREFETCH
#define DL_RMS_PREFETCH 0  // L2 prefetch of the next tile's A (dS^T) in the fused kernel
#endif                     // (measured: 0.564 vs 0.527 ms at C3 -- off)
template <bool RMS>
struct Cfg2 {
  static constexpr int A_BYTES = BM * BK * 2;   // 128 rows of A
  static constexpr int B_BYTES = 128 * BK * 2;  // this CTA's 128 columns of B
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES = RMS ? DL_RMS_STAGES : DL_PAIR_STAGES;
  static constexpr int TMEM_COLS = 512;         // 2 accumulator stages x 256 columns
  // barriers: full, empty [STAGES]; tfull, tempty [2]; (xf) afull, xready,
  // stored [STAGES]; then the TMEM address slot
  static constexpr int BAR_BYTES = (5 * STAGES + 4) * 8 + 16;
  static constexpr int EPI_OFF = STAGES * STAGE + (BAR_BYTES + 255) / 256 * 256;
  static constexpr int EPI_CHUNK_BYTES = 32 * 32 * 4;
  static constexpr int EPI_WARP_BYTES = RMS ? DL_RMS_RING * EPI_CHUNK_BYTES : 0;
  static constexpr int SMEM = EPI_OFF + kEpiWarps * EPI_WARP_BYTES + 1024;
};
static_assert(Cfg2<true>::SMEM <= 227 * 1024 && Cfg2<false>::SMEM <= 227 * 1024,
              "pair kernel shared memory");

__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map,
                                                 uint32_t bar, int c0, int c1) {
  // completes on the even CTA's barrier (peer bit cleared), as CUTLASS's
  // SM100_TMA_2SM_LOAD does
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar & 0xFEFFFFFFu), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_pair(uint32_t tmem_d, uint64_t a, uint64_t b,
                                              uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void mma_commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(bar),
      "h"((uint16_t)0x3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_rank0(uint32_t bar) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(bar), "r"(0));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}
// The accumulator-empty arrive of the epilogue warps: relaxed -- it orders
// only the warp's completed tcgen05.ld (tcgen05.wait::ld + fence::
// before_thread_sync), not its global stores; a release arrive waits for
// every store the warp has in flight (MEMBAR.ALL.GPU) -- the whole pass-2
// stream of the fused rmsprop epilogue.
__device__ __forceinline__ void mbar_arrive_rank0_relaxed(uint32_t bar) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(bar), "r"(0));
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int c0,
                                             int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(src), "r"(c0), "r"(c1)
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// wait with cluster-scope acquire: the arrivals are the peer CTA's
// release.cluster arrives after its shared-memory writes
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n.reg .pred p;\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// relaxed poll (an acquire load would invalidate L1 on every iteration);
// the caller fences once after the condition holds
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_shared_f32(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ float ld_shared_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ float4 ld_shared_v4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a)
               : "memory");
  return v;
}
__device__ __forceinline__ void st_shared_v4(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
// byte offset of 16-byte unit u (0..7) of row r in a 32 x 32 fp32 chunk: the
// unit index is XOR-swizzled by r % 8, so both a row per thread and eight
// threads per row touch eight distinct bank groups per quarter warp
__device__ __forceinline__ uint32_t chunk_off(int r, int u) {
  return static_cast<uint32_t>(r * 128 + ((u ^ (r & 7)) << 4));
}

// Fused dense W_out rmsprop epilogue (rmsprop.hpp:94-107) for one
// accumulator row of a 256 x 256 pair tile: this warp drains columns
// [c0, c0 + 128) of its TMEM lane quarter (32 rows, thread = row).
//   pass 1: clip (rnn.hpp:158-159), partial sum of squares -> rowsq[sub][m];
//           the warp arrives on its M block's counter, then waits until all
//           2 * 8 * n_tiles warps of the block have arrived;
//   pass 2: mean_sq over the row's partials in fixed order,
//           m = float(rho m + (1-rho) mean_sq) exactly as the reference, and
//           w -= s * g with s = float(eta / sqrt(m + eps)) in fp32 (the bf16
//           mode's update; the reference rounds eta*g/denom once instead),
//           then the bf16 shadow.
// The fp32 master slice streams through the warp's cp.async buffer in shared
// memory (issued right after the warp's arrival, so the loads overlap the
// block sync): read coalesced (eight lanes per 128-byte row), updated a row
// per thread against the TMEM accumulator, stored coalesced.
// The old m is read before arriving; the nt == 0, half 0 warp writes the new
// m after every warp of the block has arrived, so no reader sees it early.
constexpr int kRmsChunks = 4;  // 32-column chunks per epilogue warp (half of 256)
//   DL_RMS_DIAG  timing diagnostics only (wrong results): 1 no block sync,
//                2 no pass 2, 4 no pass 1 tmem loads
#ifndef DL_RMS_DIAG
#define DL_RMS_DIAG 0
#endif

__device__ __forceinline__ void epilogue_rms(const GemmDesc& g, uint32_t taddr, int m, int mt,
                                             int nt, int half, int c0, int nsub, unsigned target,
                                             uint32_t ring, unsigned long long* tr = nullptr,
                                             unsigned long long* arrt = nullptr) {
  const int lane = threadIdx.x % 32;
  const bool mvalid = m < g.M;
  const int sub = 2 * nt + half;
  const int rbase = m - lane;
  const float m_old = mvalid ? g.rms_m[m] : 0.f;
  // coalesced role: lane -> rows 4i + lane/8, 16-byte unit lane % 8
  const int cr = lane >> 3, cu = lane & 7;
  const int64_t col0 = static_cast<int64_t>(nt) * 256 + c0 * 32 + 4 * cu;
  auto issue = [&](int k, uint32_t buf) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int rr = 4 * i + cr;
      if (!(DL_RMS_DIAG & 16) && rbase + rr < g.M)
        cp_async16(buf + chunk_off(rr, cu),
                   g.rms_w + static_cast<int64_t>(rbase + rr) * g.ldc + col0 + k * 32);
    }
    cp_async_commit();
  };
  double sq = 0.0;
  // two 32-column TMEM loads in flight per wait
#pragma unroll 1
  for (int c = c0; c < ((DL_RMS_DIAG & 4) ? c0 : c0 + kRmsChunks); c += 2) {
    uint32_t r0[32], r1[32];
    tmem_ld32_async(taddr + c * 32, r0);
    tmem_ld32_async(taddr + (c + 1) * 32, r1);
    tmem_wait_ld();
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float x0 = clip1(__uint_as_float(r0[j]), g.clip);
      const float x1 = clip1(__uint_as_float(r1[j]), g.clip);
      s0 = fmaf(x0, x0, s0);
      s1 = fmaf(x1, x1, s1);
    }
    sq += (double)s0;
    sq += (double)s1;
  }
  if (mvalid) g.rowsq[static_cast<int64_t>(sub) * g.M + m] = sq;
  __syncwarp();
  if (lane == 0) {
    if (tr) tr[1] = gtimer_ns();
    // release the partials (before any cp.async is in flight: a fence
    // would wait for those loads too; issuing the loads before pass 1 with a
    // release reduction instead measured slower)
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    atomicAdd(g.rms_cnt + mt, 1u);
    if (arrt) *arrt = gtimer_ns();
  }
  // the master's chunks load while the block's other warps publish
#pragma unroll
  for (int k = 0; k < DL_RMS_RING; ++k) issue(k, ring + k * 4096);
  if (lane == 0) {
#if !(DL_RMS_DIAG & 1)
    // bounded: the block's other pairs are co-resident by construction
    // (launch2 checks cudaOccupancyMaxActiveClusters and the runtime never
    // fuses beside another spinning kernel); if that is ever violated the
    // kernel traps -- a loud launch failure, not a silent hang (~4 s)
    long spins = 0;
    while (ld_relaxed(g.rms_cnt + mt) < target) {
      __nanosleep(32);
      if (++spins > (1l << 27)) __trap();
    }
#endif
    ld_acquire_u32(g.rms_cnt + mt);  // acquire without waiting for the loads
    if (tr) tr[2] = gtimer_ns();
  }
  __syncwarp();
  float step = 0.f, mw = 0.f;
  if (mvalid) {
    double tot = 0.0;
    for (int k = 0; k < nsub; ++k) tot += __ldcg(g.rowsq + static_cast<int64_t>(k) * g.M + m);
    mw = (float)(g.rho * (double)m_old + (1.0 - g.rho) * (tot / (double)g.N));
    step = (float)(g.eta / sqrt((double)mw + g.eps));
  }
#pragma unroll 1
  for (int k = 0; k < ((DL_RMS_DIAG & 2) ? 0 : kRmsChunks); ++k) {
    const uint32_t buf = ring + (k % DL_RMS_RING) * 4096;
    // chunks issued so far: min(k + ... ) -- wait until chunk k has landed
    if (kRmsChunks - 1 - k >= DL_RMS_RING - 1) cp_async_wait<DL_RMS_RING - 1>();
    else if (kRmsChunks - 1 - k == 2) cp_async_wait<2>();
    else if (kRmsChunks - 1 - k == 1) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncwarp();
    // row per thread: w -= step * clip(g) in place
    float v[32];
    tmem_ld32(taddr + (c0 + k) * 32, v);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t a = buf + chunk_off(lane, u);
      float4 w = ld_shared_v4(a);
      w.x -= step * clip1(v[4 * u + 0], g.clip);
      w.y -= step * clip1(v[4 * u + 1], g.clip);
      w.z -= step * clip1(v[4 * u + 2], g.clip);
      w.w -= step * clip1(v[4 * u + 3], g.clip);
      st_shared_v4(a, w);
    }
    __syncwarp();
    // coalesced stores of the master and its bf16 shadow
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int rr = 4 * i + cr;
      const float4 w = ld_shared_v4(buf + chunk_off(rr, cu));
      if (!(DL_RMS_DIAG & 8) && rbase + rr < g.M) {
        const int64_t off = static_cast<int64_t>(rbase + rr) * g.ldc + col0 + k * 32;
        *reinterpret_cast<float4*>(g.rms_w + off) = w;
        __nv_bfloat162 p0 = __floats2bfloat162_rn(w.x, w.y);
        __nv_bfloat162 p1 = __floats2bfloat162_rn(w.z, w.w);
        uint2 q;
        q.x = *reinterpret_cast<uint32_t*>(&p0);
        q.y = *reinterpret_cast<uint32_t*>(&p1);
        *reinterpret_cast<uint2*>(g.rms_wb + off) = q;
      }
    }
    __syncwarp();
    if (k + DL_RMS_RING < kRmsChunks) issue(k + DL_RMS_RING, buf);
  }
  if (DL_RMS_DIAG & 2) cp_async_wait<0>();
  if (mvalid && nt == 0 && half == 0) g.rms_m[m] = mw;
  if (tr && lane == 0) tr[3] = gtimer_ns();
}

// XF: the A tile (bf16 logits, K-major) is turned into dS in shared memory
// by the epilogue warps before the MMAs read it (GemmDesc::xf): the A load
// completes on a CTA-local barrier (afull), the eight epilogue warps of both
// CTAs rewrite their tile and arrive on the leader's xready, the leader's MMA
// waits for B (full) and both transformed A halves (xready).  On N tile 0 the
// rewritten tile is also stored to xf_out by TMA; `stored` holds the stage
// until that store has read it.  The epilogue warps transform tile u's k-
// blocks, then drain its accumulator, then move on (the dh GEMM has one or
// two long-K tiles per pair).
template <bool A_MN, bool B_MN, bool RMS, bool XF = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
tc_gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmD, GemmDesc g, Sched sc) {
  using C = Cfg2<RMS>;
  static_assert(!XF || (!A_MN && !RMS), "xf: K-major A, plain epilogue");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 5 * C::STAGES + 4);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const uint32_t sbase = smem_u32(smem);
  auto full = [&](int s) { return smem_u32(&bars[s]); };
  auto empty = [&](int s) { return smem_u32(&bars[C::STAGES + s]); };
  auto tfull = [&](int a) { return smem_u32(&bars[2 * C::STAGES + a]); };
  auto tempty = [&](int a) { return smem_u32(&bars[2 * C::STAGES + 2 + a]); };
  auto afull = [&](int s) { return smem_u32(&bars[2 * C::STAGES + 4 + s]); };
  auto xready = [&](int s) { return smem_u32(&bars[3 * C::STAGES + 4 + s]); };
  auto stored = [&](int s) { return smem_u32(&bars[4 * C::STAGES + 4 + s]); };

  if (threadIdx.x == 32) {
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(full(s), 1); mbar_init(empty(s), 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(tfull(a), 1); mbar_init(tempty(a), 2 * kEpiWarps); }
    if (XF)
      for (int s = 0; s < C::STAGES; ++s) {
        mbar_init(afull(s), 1);
        mbar_init(xready(s), 2 * kEpiWarps);
        mbar_init(stored(s), kEpiWarps);
      }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  cluster_sync_all();  // peer barriers initialised before any remote arrive / TMA
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total = sc.m_tiles * sc.n_tiles * sc.k_splits;
  const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      for (int u = pair; u < total; u += npairs) {
        int mt, nt, kb0, kb1;
        sc.decode(u, mt, nt, kb0, kb1);
        const int m0 = mt * 256 + (int)rank * 128;
        const int n0 = nt * 256 + (int)rank * 128;
#if DL_RMS_PREFETCH
        if (RMS && u + npairs < total) {
          // the fused dW_out kernel's A (dS^T, read once from HBM per M
          // block): pull the next tile's half into L2 while this tile runs,
          // so the short-K mainloop (32 k-blocks) never waits on HBM
          int mt2, nt2, kc0, kc1;
          sc.decode(u + npairs, mt2, nt2, kc0, kc1);
          if (nt2 == 0) {  // one pair per M block (the others read it from L2)
            const int pm0 = mt2 * 256 + (int)rank * 128;
            for (int kb = kc0; kb < kc1; ++kb) {
              tma_prefetch_2d(&tmA, pm0, kb * BK);
              tma_prefetch_2d(&tmA, pm0 + 64, kb * BK);
            }
          }
        }
#endif
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(empty(stage), phase ^ 1);
          const uint32_t a_s = sbase + stage * C::STAGE;
          const uint32_t b_s = a_s + C::A_BYTES;
          if (XF) {
            // A on this CTA's own barrier (the epilogue warps transform it);
            // the stage's previous dS store must have read the tile
            if (!(DL_XF_DIAG & 32)) mbar_wait(stored(stage), phase ^ 1);
            if (leader) mbar_expect_tx(full(stage), 2 * C::B_BYTES);
            mbar_expect_tx(afull(stage), C::A_BYTES);
            tma_load_2d(a_s, &tmA, afull(stage), kb * BK, m0);
          } else if (leader) {
            mbar_expect_tx(full(stage), 2 * C::STAGE);
          }
          if (XF) {
          } else if (!A_MN) {
            tma_load_2d_pair(a_s, &tmA, full(stage), kb * BK, m0);
          } else {
            tma_load_2d_pair(a_s, &tmA, full(stage), m0, kb * BK);
            tma_load_2d_pair(a_s + 8192, &tmA, full(stage), m0 + 64, kb * BK);
          }
          if (!B_MN) {
            tma_load_2d_pair(b_s, &tmB, full(stage), kb * BK, n0);
          } else {
            tma_load_2d_pair(b_s, &tmB, full(stage), n0, kb * BK);
            tma_load_2d_pair(b_s + 8192, &tmB, full(stage), n0 + 64, kb * BK);
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) |
                                 (static_cast<uint32_t>(A_MN) << 15) |
                                 (static_cast<uint32_t>(B_MN) << 16) |
                                 (static_cast<uint32_t>(256 >> 3) << 17) |
                                 (static_cast<uint32_t>(256 >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = pair; u < total; u += npairs) {
        int mt, nt, kb0, kb1;
        sc.decode(u, mt, nt, kb0, kb1);
        mbar_wait(tempty(acc), acc_phase ^ 1);
        fence_after();
        const uint32_t d = tmem_base + acc * 256;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(full(stage), phase);
          if (XF && !(DL_XF_DIAG & 4)) mbar_wait_cluster(xready(stage), phase);
          fence_after();
          const uint32_t a_s = sbase + stage * C::STAGE;
          const uint32_t b_s = a_s + C::A_BYTES;
#pragma unroll
          for (int ks = 0; ks < BK / UMMA_K; ++ks) {
            const uint64_t ad = A_MN ? make_desc(a_s + ks * 2048, 8192, 1024)
                                     : make_desc(a_s + ks * 32, 16, 1024);
            const uint64_t bd = B_MN ? make_desc(b_s + ks * 2048, 8192, 1024)
                                     : make_desc(b_s + ks * 32, 16, 1024);
            mma_bf16_pair(d, ad, bd, idesc, (kb > kb0 || ks > 0) ? 1u : 0u);
          }
          mma_commit_pair(empty(stage));
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit_pair(tfull(acc));
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    const int quarter = warp % 4, half = (warp - 2) / 4;
    const int row = quarter * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    bool bad = false;
    // trace (g.trace): pairs 0, 1, 35, warp 2 -- per tile: tfull observed,
    // pass 1 done, block sync done, pass 2 done (%globaltimer ns)
    const int trace_slot = (blockIdx.x == 0) ? 0 : (blockIdx.x == 2) ? 1 : (blockIdx.x == 70) ? 2 : -1;
    // (and every pair's pass-1 arrival time per tile at g.trace + 3*64*4)
    unsigned long long* arr = (g.trace && lane == 0 && !g.trace_warps)
                                  ? g.trace + 3 * 64 * 4 + (blockIdx.x * 8 + (warp - 2)) * 32
                                  : nullptr;
    int it = 0;
    // xf: ring position of the transform (advances like the MMA's) and the
    // stage whose dS store has not been retired yet (thread 64 owns stores)
    int xs = 0;
    uint32_t xph = 0;
    int pend = -1;
    for (int u = pair; u < total; u += npairs, ++it) {
      int mt, nt, kb0, kb1;
      sc.decode(u, mt, nt, kb0, kb1);
      const int split = u % sc.k_splits;
      if constexpr (XF) {
        // epilogue warp w' (0..7) rewrites rows [16 w', 16 w' + 16) of the
        // CTA's 128-row A tile: lane owns physical 16-byte chunk lane % 8 of
        // rows 16 w' + lane / 8 + 4 j (j = 0..3); the logical 8-column group
        // of a chunk is its physical index XOR row % 8 (SWIZZLE_128B)
        const int wq = warp - 2;
        const int pc = lane & 7;
        const int m0 = mt * 256 + (int)rank * 128;
        float xnl[4], xsc[4];
        int xy[4], xc[4], xr[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r = 16 * wq + (lane >> 3) + 4 * j;
          const int m = m0 + r;
          const bool ok = m < g.M;
          xr[j] = r;
          xnl[j] = ok ? g.xf_lse[m] : 0.f;
          xsc[j] = ok ? g.xf_sc[m] : 0.f;
          xy[j] = ok ? (int)g.xf_tgt[m] : -1;
          xc[j] = pc ^ (r & 7);
        }
        const bool writer = nt == 0 && g.xf_out != nullptr && !(DL_XF_DIAG & 16);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(afull(xs), xph);
          const uint32_t a_s = sbase + xs * C::STAGE;
#pragma unroll
          for (int j = 0; j < ((DL_XF_DIAG & 8) ? 0 : 4); ++j) {
            const uint32_t addr = a_s + xr[j] * 128 + pc * 16;
            uint32_t q[4];
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3])
                         : "r"(addr));
            const int dt = xy[j] - (kb * BK + xc[j] * 8);
            if (DL_XF_DIAG & 1) {
            } else if (static_cast<unsigned>(dt) >= 8u) {
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float lo = __uint_as_float(q[e] << 16);
                const float hi = __uint_as_float(q[e] & 0xFFFF0000u);
                const __nv_bfloat162 p = __floats2bfloat162_rn(ds_of_logit(lo, xnl[j], xsc[j]),
                                                               ds_of_logit(hi, xnl[j], xsc[j]));
                q[e] = *reinterpret_cast<const uint32_t*>(&p);
              }
            } else {
              // the chunk holds the target column: dS[y] -= scale
              // (backprop.hpp:184-185), subtracted before the bf16 rounding
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float lo = __uint_as_float(q[e] << 16);
                const float hi = __uint_as_float(q[e] & 0xFFFF0000u);
                const float a0 = ds_of_logit(lo, xnl[j], xsc[j]) - (2 * e == dt ? xsc[j] : 0.f);
                const float a1 =
                    ds_of_logit(hi, xnl[j], xsc[j]) - (2 * e + 1 == dt ? xsc[j] : 0.f);
                const __nv_bfloat162 p = __floats2bfloat162_rn(a0, a1);
                q[e] = *reinterpret_cast<const uint32_t*>(&p);
              }
            }
            asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(q[0]),
                         "r"(q[1]), "r"(q[2]), "r"(q[3])
                         : "memory");
          }
          if (!(DL_XF_DIAG & 2)) fence_async_smem();  // generic writes -> async proxy
          __syncwarp();
          if (lane == 0) {
            if (DL_XF_DIAG & 4) mbar_arrive(xready(xs));
            else mbar_arrive_rank0(xready(xs));
            // N tile 0: store this warp's 16 rewritten rows (dS for dW_out),
            // then retire the previous stage's store -- its tile is read --
            // so the producer may refill that stage
            if (writer) tma_store_2d(&tmD, a_s + 16 * wq * 128, kb * BK, m0 + 16 * wq);
            if (pend >= 0) {
              if (writer) bulk_wait_read<1>();
              else bulk_wait_read<0>();
              mbar_arrive(stored(pend));
            }
            pend = xs;
          }
          if (++xs == C::STAGES) { xs = 0; xph ^= 1; }
        }
      }
      mbar_wait(tfull(acc), acc_phase);
      fence_after();
      // (slots 0..2: warp 2 of pairs 0, 1, 35; with DL_GEMM_TRACE_WARPS the
      // three slots are warps 2, 5 and 9 of pair 0)
      const int tslot = g.trace_warps ? (blockIdx.x == 0 && (warp == 2 || warp == 5 || warp == 9)
                                             ? (warp == 2 ? 0 : warp == 5 ? 1 : 2) : -1)
                                      : (warp == 2 ? trace_slot : -1);
      unsigned long long* tr = (g.trace && tslot >= 0 && it < 64)
                                   ? g.trace + (tslot * 64 + it) * 4 : nullptr;
      if (tr && lane == 0) tr[0] = gtimer_ns();
      const int m = mt * 256 + (int)rank * 128 + row;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * 256;
      if constexpr (RMS)
        epilogue_rms(g, taddr, m, mt, nt, half, half * 4, 2 * sc.n_tiles, 16u * sc.n_tiles,
                     sbase + C::EPI_OFF + (warp - 2) * C::EPI_WARP_BYTES, tr,
                     (arr && it < 32) ? arr + it : nullptr);
      else
        epilogue_row<256>(g, taddr, m, nt, split, bad, half * 4, half * 4 + 4, 2 * nt + half);
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_rank0_relaxed(tempty(acc));
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (g.do_clip && g.nonfinite && bad) atomicExch(g.nonfinite, 1);
    if (XF && lane == 0) {
      bulk_wait_read<0>();
      if (pend >= 0) mbar_arrive(stored(pend));
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // dS stores complete
    }
  }
  fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 0) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(C::TMEM_COLS));
  }
}

// Epilogue of one accumulator row (this thread's TMEM lane) of a 128 x BN
// tile: fp32 store (+ clip / finite flag, split-K slice) or the logits
// epilogue (online max / sum-exp over the tile's columns, target-logit
// capture, optional bf16 logits).
template <int BN>
__device__ __forceinline__ void epilogue_row(const GemmDesc& g, uint32_t taddr, int m, int nt,
                                             int split, bool& bad, int c0, int c1, int sub) {
      const bool mvalid = m < g.M;
      if (!g.logits && g.Cb) {
        // bf16 gradient rows + per-(half tile, row) partial sum of squares of
        // the clipped fp32 values (the dense rmsprop's mean_sq, rmsprop.hpp:100)
        bf16* Brow = g.Cb + static_cast<int64_t>(m) * g.ldc;
        double sq = 0.0;
#pragma unroll 1
        for (int c = c0; c < c1; ++c) {
          float v[32];
          tmem_ld32(taddr + c * 32, v);
          const int n0 = nt * BN + c * 32;
          float s = 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            v[j] = clip1(v[j], g.clip);
            if (n0 + j < g.N) s = fmaf(v[j], v[j], s);
          }
          sq += (double)s;
          if (!mvalid) continue;
          if (n0 + 32 <= g.N && (g.ldc % 8) == 0) {
            uint4* dst = reinterpret_cast<uint4*>(Brow + n0);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint4 q;
              __nv_bfloat162 p0 = __floats2bfloat162_rn(v[8 * j + 0], v[8 * j + 1]);
              __nv_bfloat162 p1 = __floats2bfloat162_rn(v[8 * j + 2], v[8 * j + 3]);
              __nv_bfloat162 p2 = __floats2bfloat162_rn(v[8 * j + 4], v[8 * j + 5]);
              __nv_bfloat162 p3 = __floats2bfloat162_rn(v[8 * j + 6], v[8 * j + 7]);
              q.x = *reinterpret_cast<uint32_t*>(&p0);
              q.y = *reinterpret_cast<uint32_t*>(&p1);
              q.z = *reinterpret_cast<uint32_t*>(&p2);
              q.w = *reinterpret_cast<uint32_t*>(&p3);
              dst[j] = q;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (n0 + j < g.N) Brow[n0 + j] = __float2bfloat16_rn(v[j]);
          }
        }
        if (mvalid && g.rowsq) g.rowsq[static_cast<int64_t>(sub) * g.M + m] = sq;
      } else if (!g.logits) {
        float* Crow = g.C + split * g.split_stride + static_cast<int64_t>(m) * g.ldc;
        const float rs = (g.row_scale && mvalid) ? g.row_scale[m] : 1.f;
        const float rr = (g.row_resid && mvalid && split == 0) ? g.row_resid[m] : 0.f;  // once over splits
        const bf16* rw = rr != 0.f ? g.resid_w + static_cast<int64_t>(g.resid_idx[m]) * g.N : nullptr;
#pragma unroll 1
        for (int c = c0; c < c1; ++c) {
          float v[32];
          tmem_ld32(taddr + c * 32, v);
          const int n0 = nt * BN + c * 32;
          if (g.row_scale) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] *= rs;
          }
          if (rw && n0 + 32 <= g.N) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint4 u = *reinterpret_cast<const uint4*>(rw + n0 + 8 * q);
              const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(h2[e]);
                v[8 * q + 2 * e] = fmaf(rr, f.x, v[8 * q + 2 * e]);
                v[8 * q + 2 * e + 1] = fmaf(rr, f.y, v[8 * q + 2 * e + 1]);
              }
            }
          } else if (rw) {
            for (int j = 0; j < 32 && n0 + j < g.N; ++j)
              v[j] = fmaf(rr, __bfloat162float(rw[n0 + j]), v[j]);
          }
          if (g.do_clip) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              v[j] = clip1(v[j], g.clip);
              bad |= mvalid && (n0 + j < g.N) && !isfinite(v[j]);
            }
          }
          if (!mvalid) continue;
          if (n0 + 32 <= g.N && (g.ldc % 4) == 0) {
            float4* dst = reinterpret_cast<float4*>(Crow + n0);
#pragma unroll
            for (int j = 0; j < 8; ++j)
              dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (n0 + j < g.N) Crow[n0 + j] = v[j];
          }
        }
      } else {
        const float kLog2e = 1.4426950408889634f;
        float mrun = -INFINITY, srun = 0.f, tval = 0.f;
        bool thit = false;
        const int tg = mvalid ? static_cast<int>(g.tgt[m]) : -1;
        bf16* Srow = g.S ? g.S + static_cast<int64_t>(m) * g.lds : nullptr;
        if (g.shift) {
          // shifted exponentials E = e^(s - shift) (bf16) replace the logits:
          // dS = row_scale * E with row_scale = scale e^(shift - lse) comes
          // out of the row's lse alone (k_pfac_rows), so no pass over the
          // logits after this GEMM.  The exponent is capped at 2^120 (a
          // 128-column partial sum stays below 2^127; rows far above their
          // shift are rescaled by k_pfac_rows).
          const float sb = (mvalid ? g.shift[m] : 0.f) * kLog2e;
          bool capped = false;  // an element of this half tile reached the cap
#pragma unroll 1
          for (int c = c0; c < c1; ++c) {
            float v[32];
            tmem_ld32(taddr + c * 32, v);
            const int n0 = nt * BN + c * 32;
            const bool whole = n0 + 32 <= g.N;
            if (static_cast<unsigned>(tg - n0) < 32u) {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (n0 + j == tg) tval = v[j];
              thit = true;
            }
            float part_sum = 0.f;
            if (whole) {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                v[j] = fast_exp2(fminf(fmaf(v[j], kLog2e, -sb), 120.f));
                part_sum += v[j];
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                v[j] = fast_exp2(fminf(fmaf(v[j], kLog2e, -sb), 120.f));
                part_sum += n0 + j < g.N ? v[j] : 0.f;
              }
            }
            srun += part_sum;
            capped |= mvalid && part_sum >= 0x1p120f;
            if (!mvalid) continue;
            if (whole && (g.lds % 8) == 0) {
              uint4* dst = reinterpret_cast<uint4*>(Srow + n0);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                uint4 q;
                __nv_bfloat162 p0 = __floats2bfloat162_rn(v[8 * j + 0], v[8 * j + 1]);
                __nv_bfloat162 p1 = __floats2bfloat162_rn(v[8 * j + 2], v[8 * j + 3]);
                __nv_bfloat162 p2 = __floats2bfloat162_rn(v[8 * j + 4], v[8 * j + 5]);
                __nv_bfloat162 p3 = __floats2bfloat162_rn(v[8 * j + 6], v[8 * j + 7]);
                q.x = *reinterpret_cast<uint32_t*>(&p0);
                q.y = *reinterpret_cast<uint32_t*>(&p1);
                q.z = *reinterpret_cast<uint32_t*>(&p2);
                q.w = *reinterpret_cast<uint32_t*>(&p3);
                dst[j] = q;
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (n0 + j < g.N) Srow[n0 + j] = __float2bfloat16_rn(v[j]);
            }
          }
          // (rare) a logit of this half tile more than 83 nats above the
          // row's shift: the half tile is redone from TMEM relative to its
          // own maximum, the offset (nats) recorded in the partial's .x --
          // k_pfac_rows rescales the row to one shift, so nothing is lost
          float off = 0.f;
          if (__any_sync(0xffffffffu, capped)) {
            float mx = -INFINITY;
#pragma unroll 1
            for (int c = c0; c < c1; ++c) {
              float v[32];
              tmem_ld32(taddr + c * 32, v);
              const int n0 = nt * BN + c * 32;
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (n0 + j < g.N) mx = fmaxf(mx, v[j]);
            }
            off = capped ? mx - sb / kLog2e : 0.f;
            const float sb2 = sb + off * kLog2e;
            srun = 0.f;
#pragma unroll 1
            for (int c = c0; c < c1; ++c) {
              float v[32];
              tmem_ld32(taddr + c * 32, v);
              const int n0 = nt * BN + c * 32;
              float part_sum = 0.f;  // (as the first pass: per chunk, then into srun)
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                v[j] = fast_exp2(fminf(fmaf(v[j], kLog2e, -sb2), 120.f));
                part_sum += n0 + j < g.N ? v[j] : 0.f;
              }
              srun += part_sum;
              if (!mvalid) continue;
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (n0 + j < g.N) Srow[n0 + j] = __float2bfloat16_rn(v[j]);
            }
          }
          if (mvalid) {
            // row-major [M][part_n] (k_pfac_rows reads a row's sums
            // contiguously); .x: the half tile's shift offset (normally 0)
            g.part[static_cast<int64_t>(m) * g.part_n + sub] = make_float2(off, srun);
            if (thit) g.tgt_logit[m] = tval;
          }
          return;
        }
#pragma unroll 1
        for (int c = c0; c < c1; ++c) {
          float v[32];
          tmem_ld32(taddr + c * 32, v);
          const int n0 = nt * BN + c * 32;
          float cmax = -INFINITY;
          const bool whole = n0 + 32 <= g.N;
          if (whole) {
#pragma unroll
            for (int j = 0; j < 32; ++j) cmax = fmaxf(cmax, v[j]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (n0 + j < g.N) cmax = fmaxf(cmax, v[j]);
          }
          if (static_cast<unsigned>(tg - n0) < 32u) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (n0 + j == tg) tval = v[j];
            thit = true;
          }
          if (cmax > mrun) {
            srun *= fast_exp2((mrun - cmax) * kLog2e);
            mrun = cmax;
          }
          const float mb = mrun * kLog2e;
          float part_sum = 0.f;
          if (whole) {
#pragma unroll
            for (int j = 0; j < 32; ++j) part_sum += fast_exp2(fmaf(v[j], kLog2e, -mb));
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (n0 + j < g.N) part_sum += fast_exp2(fmaf(v[j], kLog2e, -mb));
          }
          srun += part_sum;
          if (Srow && mvalid) {
            if (n0 + 32 <= g.N && (g.lds % 8) == 0) {
              uint4* dst = reinterpret_cast<uint4*>(Srow + n0);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                uint4 q;
                __nv_bfloat162 p0 = __floats2bfloat162_rn(v[8 * j + 0], v[8 * j + 1]);
                __nv_bfloat162 p1 = __floats2bfloat162_rn(v[8 * j + 2], v[8 * j + 3]);
                __nv_bfloat162 p2 = __floats2bfloat162_rn(v[8 * j + 4], v[8 * j + 5]);
                __nv_bfloat162 p3 = __floats2bfloat162_rn(v[8 * j + 6], v[8 * j + 7]);
                q.x = *reinterpret_cast<uint32_t*>(&p0);
                q.y = *reinterpret_cast<uint32_t*>(&p1);
                q.z = *reinterpret_cast<uint32_t*>(&p2);
                q.w = *reinterpret_cast<uint32_t*>(&p3);
                dst[j] = q;
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (n0 + j < g.N) Srow[n0 + j] = __float2bfloat16_rn(v[j]);
            }
          }
        }
        if (mvalid) {
          // row-major [M][part_n]: a row's partials contiguous for the
          // combining kernels
          g.part[static_cast<int64_t>(m) * g.part_n + sub] = make_float2(mrun, srun);
          if (thit) g.tgt_logit[m] = tval;
        }
      }
}

// --------------------------------------------------------------------------
// 3xTF32: the fp32 parity mode's GEMMs on the tensor cores (tcgen05
// kind::tf32, fp32 accumulation in TMEM).  fp32 operands arrive by TMA
// (SWIZZLE_128B, 32 elements per 128-byte row, BK = 32); four converter warps
// split every stage in shared memory into hi = tf32(x) (in place, exact
// round-to-nearest) and lo = x - hi, and the MMA warp issues
// hi.hi + hi.lo + lo.hi -- about 21 significant bits per product, fp32
// accumulation like the SIMT kernel it replaces (the reference accumulates
// in double, mat.hpp:59-78; the parity bar is 1e-4).  128 x 128 tiles.
// Roles: warp 0 TMA, warp 1 MMA, warps 2..9 epilogue (two per TMEM lane
// quarter), warps 10..13 converters.
constexpr int kXBK = 32;  // fp32 elements per k-block (one 128-byte swizzle row)
constexpr int kXBN = 128;
constexpr int kXConvWarps = 4;
constexpr int kXChunk = 8;  // k-blocks (K = 256) per fresh TMEM accumulation
constexpr int kXThreads = 64 + 32 * kEpiWarps + 32 * kXConvWarps;
struct CfgX {
  static constexpr int A_BYTES = BM * kXBK * 4;   // 16 KB
  static constexpr int B_BYTES = kXBN * kXBK * 4;  // 16 KB
  static constexpr int STAGE = 2 * (A_BYTES + B_BYTES);  // hi (in place) + lo copies
  static constexpr int STAGES = 3;
  static constexpr int TMEM_COLS = 2 * kXBN;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
};
static_assert(CfgX::SMEM <= 227 * 1024, "tf32 kernel shared memory");

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}

template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(kXThreads, 1)
tc_tf32x3_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 GemmDesc g, Sched sc) {
  using C = CfgX;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  // full[S], split[S], empty[S], tfull[2], tempty[2]; then the TMEM slot
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * C::STAGES + 4);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t sbase = smem_u32(smem);
  auto full = [&](int s) { return smem_u32(&bars[s]); };
  auto split = [&](int s) { return smem_u32(&bars[C::STAGES + s]); };
  auto empty = [&](int s) { return smem_u32(&bars[2 * C::STAGES + s]); };
  auto tfull = [&](int a) { return smem_u32(&bars[3 * C::STAGES + a]); };
  auto tempty = [&](int a) { return smem_u32(&bars[3 * C::STAGES + 2 + a]); };
  // stage layout: A hi | B hi | A lo | B lo
  auto a_hi = [&](int s) { return sbase + s * C::STAGE; };
  auto b_hi = [&](int s) { return sbase + s * C::STAGE + C::A_BYTES; };
  auto a_lo = [&](int s) { return sbase + s * C::STAGE + C::A_BYTES + C::B_BYTES; };
  auto b_lo = [&](int s) { return sbase + s * C::STAGE + 2 * C::A_BYTES + C::B_BYTES; };

  if (threadIdx.x == 32) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(full(s), 1);
      mbar_init(split(s), kXConvWarps);
      mbar_init(empty(s), 1);
    }
    for (int a = 0; a < 2; ++a) { mbar_init(tfull(a), 1); mbar_init(tempty(a), kEpiWarps); }
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
  const uint32_t tmem_base = *tmem_slot;
  const int total = sc.m_tiles * sc.n_tiles * sc.k_splits;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < total; u += gridDim.x) {
        int mt, nt, kb0, kb1;
        sc.decode(u, mt, nt, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(empty(stage), phase ^ 1);
          mbar_expect_tx(full(stage), C::A_BYTES + C::B_BYTES);
          if (!A_MN) {
            tma_load_2d(a_hi(stage), &tmA, full(stage), kb * kXBK, mt * BM);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 32; ++j)
              tma_load_2d(a_hi(stage) + j * 4096, &tmA, full(stage), mt * BM + 32 * j, kb * kXBK);
          }
          if (!B_MN) {
            tma_load_2d(b_hi(stage), &tmB, full(stage), kb * kXBK, nt * kXBN);
          } else {
#pragma unroll
            for (int j = 0; j < kXBN / 32; ++j)
              tma_load_2d(b_hi(stage) + j * 4096, &tmB, full(stage), nt * kXBN + 32 * j,
                          kb * kXBK);
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // kind::tf32: D f32 (bits 4-5 = 1), A / B tf32 (bits 7-9 / 10-12 = 2)
      constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) |
                                 (static_cast<uint32_t>(A_MN) << 15) |
                                 (static_cast<uint32_t>(B_MN) << 16) |
                                 (static_cast<uint32_t>(kXBN >> 3) << 17) |
                                 (static_cast<uint32_t>(BM >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = blockIdx.x; u < total; u += gridDim.x) {
        int mt, nt, kb0, kb1;
        sc.decode(u, mt, nt, kb0, kb1);
        // the tile's K range in chunks of kXChunk k-blocks, each accumulated
        // afresh in alternating TMEM buffers and summed by the epilogue in
        // registers (round-to-nearest): the tensor core's fp32 accumulation
        // truncates, and over a long K that bias would reach 1e-4
        for (int c0 = kb0; c0 < kb1; c0 += kXChunk) {
          const int c1 = min(kb1, c0 + kXChunk);
          mbar_wait(tempty(acc), acc_phase ^ 1);
          fence_after();
          const uint32_t d = tmem_base + acc * kXBN;
          for (int kb = c0; kb < c1; ++kb) {
            mbar_wait(split(stage), phase);
            fence_after();
            const uint32_t ah = a_hi(stage), bh = b_hi(stage), al = a_lo(stage),
                           bl = b_lo(stage);
#pragma unroll
            for (int ks = 0; ks < kXBK / 8; ++ks) {
              auto da = [&](uint32_t base) {
                return A_MN ? make_desc(base + ks * 1024, 4096, 1024)
                            : make_desc(base + ks * 32, 16, 1024);
              };
              auto db = [&](uint32_t base) {
                return B_MN ? make_desc(base + ks * 1024, 4096, 1024)
                            : make_desc(base + ks * 32, 16, 1024);
              };
              // small terms first, then hi.hi
              mma_tf32(d, da(al), db(bh), idesc, (kb > c0 || ks > 0) ? 1u : 0u);
              mma_tf32(d, da(ah), db(bl), idesc, 1u);
              mma_tf32(d, da(ah), db(bh), idesc, 1u);
            }
            mma_commit(empty(stage));
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
          }
          mma_commit(tfull(acc));
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
      }
    }
  } else if (warp >= 2 + kEpiWarps) {
    // ---------------- converters: x -> hi = tf32_rna(x) in place, lo = x - hi
    const int t = threadIdx.x - (64 + 32 * kEpiWarps);
    int stage = 0;
    uint32_t phase = 0;
    for (int u = blockIdx.x; u < total; u += gridDim.x) {
      int mt, nt, kb0, kb1;
      sc.decode(u, mt, nt, kb0, kb1);
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(full(stage), phase);
        constexpr int kVec = (C::A_BYTES + C::B_BYTES) / 16;  // 16-byte vectors of A hi | B hi
#pragma unroll 4
        for (int i = t; i < kVec; i += 32 * kXConvWarps) {
          const uint32_t src = a_hi(stage) + i * 16;
          const uint32_t dst = a_lo(stage) + i * 16;
          float4 x = ld_shared_v4(src), h, l;
          uint32_t hb;
          asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(x.x)); h.x = __uint_as_float(hb);
          asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(x.y)); h.y = __uint_as_float(hb);
          asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(x.z)); h.z = __uint_as_float(hb);
          asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(x.w)); h.w = __uint_as_float(hb);
          l.x = x.x - h.x; l.y = x.y - h.y; l.z = x.z - h.z; l.w = x.w - h.w;
          st_shared_v4(src, h);
          st_shared_v4(dst, l);
        }
        fence_async_smem();  // generic writes -> the MMA's async proxy
        __syncwarp();
        if (lane == 0) mbar_arrive(split(stage));
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // ---------------- epilogue (warps 2..9)
    const int quarter = warp % 4, half = (warp - 2) / 4;
    const int row = quarter * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    bool bad = false;
    for (int u = blockIdx.x; u < total; u += gridDim.x) {
      int mt, nt, kb0, kb1;
      sc.decode(u, mt, nt, kb0, kb1);
      const int split_i = u % sc.k_splits;
      // this thread's row, columns [64 half, 64 half + 64): the chunks'
      // partial sums added in registers
      float sum[64];
#pragma unroll
      for (int j = 0; j < 64; ++j) sum[j] = 0.f;
      for (int c0 = kb0; c0 < kb1; c0 += kXChunk) {
        mbar_wait(tfull(acc), acc_phase);
        fence_after();
        const uint32_t taddr =
            tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * kXBN + half * 64;
        uint32_t r0[32], r1[32];
        tmem_ld32_async(taddr, r0);
        tmem_ld32_async(taddr + 32, r1);
        tmem_wait_ld();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty(acc));
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          sum[j] += __uint_as_float(r0[j]);
          sum[32 + j] += __uint_as_float(r1[j]);
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      // fp32 store (+ clip / finite flag, split-K slice) as epilogue_row
      const int m = mt * BM + row;
      const bool mvalid = m < g.M;
      const int n0 = nt * kXBN + half * 64;
      if (g.do_clip) {
#pragma unroll
        for (int j = 0; j < 64; ++j) {
          sum[j] = clip1(sum[j], g.clip);
          bad |= mvalid && (n0 + j < g.N) && !isfinite(sum[j]);
        }
      }
      if (mvalid) {
        float* Crow = g.C + split_i * g.split_stride + static_cast<int64_t>(m) * g.ldc;
        if (n0 + 64 <= g.N && (g.ldc % 4) == 0) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            reinterpret_cast<float4*>(Crow + n0)[j] =
                make_float4(sum[4 * j], sum[4 * j + 1], sum[4 * j + 2], sum[4 * j + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < 64; ++j)
            if (n0 + j < g.N) Crow[n0 + j] = sum[j];
        }
      }
    }
    if (g.do_clip && g.nonfinite && bad) atomicExch(g.nonfinite, 1);
  }
  fence_before();
  __syncthreads();
  if (warp == 0) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(C::TMEM_COLS));
  }
}

// ------------------------------------------------------------------- host
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    DL_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    DL_REQUIRE(p && q == cudaDriverEntryPointSuccess, 3, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D bf16 tensor map over a row-major [rows x cols] matrix with leading
// dimension ld (elements), box {64 cols, box_rows}, 128-byte swizzle.
CUtensorMap make_map(const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  DL_REQUIRE((reinterpret_cast<uintptr_t>(base) % 16) == 0, 1, "tma: base not 16B aligned");
  DL_REQUIRE((ld * 2) % 16 == 0, 1, "tma: leading dimension must be a multiple of 8 elements");
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  cuuint32_t box[2] = {64u, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DL_REQUIRE(r == CUDA_SUCCESS, 3, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return m;
}

// fp32 variant for the 3xTF32 kernel: box {32 cols (128 bytes), box_rows}
CUtensorMap make_map_f32(const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  DL_REQUIRE((reinterpret_cast<uintptr_t>(base) % 16) == 0, 1, "tma: base not 16B aligned");
  DL_REQUIRE((ld * 4) % 16 == 0, 1, "tma: leading dimension must be a multiple of 4 elements");
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 4)};
  cuuint32_t box[2] = {32u, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DL_REQUIRE(r == CUDA_SUCCESS, 3, "cuTensorMapEncodeTiled (fp32) failed: " + std::to_string(r));
  return m;
}

template <bool A_MN, bool B_MN>
void launch_tf32x3(const GemmDesc& g, cudaStream_t st) {
  using C = CfgX;
  auto kern = tc_tf32x3_kernel<A_MN, B_MN>;
  static std::once_flag once;
  std::call_once(once, [&] {
    DL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  });
  const CUtensorMap ta = A_MN ? make_map_f32(g.A, g.K, g.M, g.lda, kXBK)
                              : make_map_f32(g.A, g.M, g.K, g.lda, BM);
  const CUtensorMap tb = B_MN ? make_map_f32(g.B, g.K, g.N, g.ldb, kXBK)
                              : make_map_f32(g.B, g.N, g.K, g.ldb, kXBN);
  Sched sc;
  sc.m_tiles = (g.M + BM - 1) / BM;
  sc.n_tiles = (g.N + kXBN - 1) / kXBN;
  sc.kb_total = (g.K + kXBK - 1) / kXBK;
  sc.k_splits = std::max(1, std::min(g.k_splits, sc.kb_total));
  sc.kbps = (sc.kb_total + sc.k_splits - 1) / sc.k_splits;
  sc.k_splits = (sc.kb_total + sc.kbps - 1) / sc.kbps;
  DL_REQUIRE(sc.k_splits == std::max(1, g.k_splits), 1,
             "tf32x3 gemm: k_splits not normalised with tf32_splits()");
  sc.raster = g.raster;
  const int total = sc.m_tiles * sc.n_tiles * sc.k_splits;
  const int grid = std::min(total, kNumSMs);
  kern<<<grid, kXThreads, C::SMEM, st>>>(ta, tb, g, sc);
  DL_CUDA(cudaGetLastError());
}

template <int BN, bool A_MN, bool B_MN>
void launch(const GemmDesc& g, cudaStream_t st) {
  using C = Cfg<BN>;
  auto kern = tc_gemm_kernel<BN, A_MN, B_MN>;
  static std::once_flag once;
  std::call_once(once, [&] {
    DL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  });
  const CUtensorMap ta = A_MN ? make_map(g.A, g.K, g.M, g.lda, 64) : make_map(g.A, g.M, g.K, g.lda, BM);
  const CUtensorMap tb = B_MN ? make_map(g.B, g.K, g.N, g.ldb, 64) : make_map(g.B, g.N, g.K, g.ldb, BN);
  Sched sc;
  sc.m_tiles = (g.M + BM - 1) / BM;
  sc.n_tiles = (g.N + BN - 1) / BN;
  sc.kb_total = (g.K + BK - 1) / BK;
  sc.k_splits = tc_splits(g.K, g.k_splits);
  sc.kbps = (sc.kb_total + sc.k_splits - 1) / sc.k_splits;
  DL_REQUIRE(sc.k_splits == std::max(1, g.k_splits), 1,
             "tc gemm: k_splits not normalised with tc_splits()");
  sc.raster = g.raster;
  const int total = sc.m_tiles * sc.n_tiles * sc.k_splits;
  const int grid = std::min(total, kNumSMs);
  kern<<<grid, kThreads, C::SMEM, st>>>(ta, tb, g, sc);
  DL_CUDA(cudaGetLastError());
}

// Co-resident CTA pairs of the pair kernel (queried once per variant).
template <bool A_MN, bool B_MN, bool RMS>
int max_pairs() {
  static const int n = [] {
    auto kern = tc_gemm2_kernel<A_MN, B_MN, RMS, false>;
    DL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 Cfg2<RMS>::SMEM));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kNumSMs, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = Cfg2<RMS>::SMEM;
    int k = 0;
    DL_CUDA(cudaOccupancyMaxActiveClusters(&k, kern, &cfg));
    return k;
  }();
  return n;
}

template <bool A_MN, bool B_MN, bool RMS, bool XF = false>
void launch2(const GemmDesc& g, cudaStream_t st) {
  using C = Cfg2<RMS>;
  auto kern = tc_gemm2_kernel<A_MN, B_MN, RMS, XF>;
  static std::once_flag once;
  std::call_once(once, [&] {
    DL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  });
  const CUtensorMap ta = A_MN ? make_map(g.A, g.K, g.M, g.lda, 64) : make_map(g.A, g.M, g.K, g.lda, BM);
  const CUtensorMap tb = B_MN ? make_map(g.B, g.K, g.N, g.ldb, 64) : make_map(g.B, g.N, g.K, g.ldb, 128);
  Sched sc;
  sc.m_tiles = (g.M + 255) / 256;
  sc.n_tiles = (g.N + 255) / 256;
  sc.kb_total = (g.K + BK - 1) / BK;
  sc.k_splits = tc_splits(g.K, g.k_splits);
  sc.kbps = (sc.kb_total + sc.k_splits - 1) / sc.k_splits;
  DL_REQUIRE(sc.k_splits == std::max(1, g.k_splits), 1,
             "tc gemm: k_splits not normalised with tc_splits()");
  sc.raster = g.raster;
  const int total = sc.m_tiles * sc.n_tiles * sc.k_splits;
  int pairs = std::min(total, kNumSMs / 2);
  DL_REQUIRE(RMS == (g.rms != 0), 1, "pair kernel variant mismatch");
  if (RMS) {
    // every N tile of an M block in the same round (N-fastest raster, a
    // multiple of n_tiles pairs), all pairs co-resident: the blocks'
    // row-sum exchange spins on the other pairs
    DL_REQUIRE(sc.raster == 1 && sc.k_splits == 1 && g.N % 256 == 0, 1,
               "fused rmsprop epilogue: raster 1, no split-K, N % 256 == 0");
    pairs = std::min((kNumSMs / 2 / sc.n_tiles) * sc.n_tiles, total);
    DL_REQUIRE(pairs > 0 && (kNumSMs / 2 / sc.n_tiles) * sc.n_tiles <= (max_pairs<A_MN, B_MN, true>()),
               1, "fused rmsprop epilogue: not enough co-resident CTA pairs");
  }
  // xf: the dS store map has the A map's geometry over xf_out
  const CUtensorMap td = XF && g.xf_out ? make_map(g.xf_out, g.M, g.K, g.lda, 16) : ta;
  kern<<<2 * pairs, kThreads, C::SMEM, st>>>(ta, tb, td, g, sc);
  DL_CUDA(cudaGetLastError());
}

}  // namespace tc

// Number of K slices actually produced for a requested split count: every
// slice gets ceil(kb_total / splits) k-blocks and none is empty.
int tc_splits(int K, int desired) {
  const int kb_total = (K + tc::BK - 1) / tc::BK;
  const int s = std::max(1, std::min(desired, kb_total));
  const int kbps = (kb_total + s - 1) / s;
  return (kb_total + kbps - 1) / kbps;
}

// Number of (max, sum-exp) partials per row the logits epilogue writes: one
// per half N-tile (two epilogue warps per TMEM lane quarter).
int tc_n_tiles(int N) {
  const int bn = N >= 256 ? 256 : (N >= 128 ? 128 : 64);
  return 2 * ((N + bn - 1) / bn);
}

// Whether the fused dW_out + dense rmsprop epilogue can run for an M x N
// gradient (pair tiles, N a multiple of 256, enough co-resident pairs).
// Queries occupancy: call outside stream capture.
bool tc_rms_fusable(int M, int N) {
  const char* e = std::getenv("DL_GEMM_2CTA");
  if ((e && std::atoi(e) == 0) || N % 256 != 0 || M < 256) return false;
  const int nt = N / 256;
  const int pairs = (kNumSMs / 2 / nt) * nt;
  return pairs > 0 && pairs <= tc::max_pairs<true, true, true>();
}

// k-slices the 3xTF32 kernel produces for a requested split count (BK = 32)
int tf32_splits(int K, int desired) {
  const int kb_total = (K + tc::kXBK - 1) / tc::kXBK;
  const int s = std::max(1, std::min(desired, kb_total));
  const int kbps = (kb_total + s - 1) / s;
  return (kb_total + kbps - 1) / kbps;
}

// Whether the 3xTF32 kernel can take this fp32 GEMM (TMA: 16-byte aligned
// bases and leading dimensions) -- else the SIMT kernel runs.
bool tf32x3_ok(const GemmDesc& g) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) % 16) == 0; };
  return !g.logits && !g.Cb && !g.rms && !g.xf && al(g.A) && al(g.B) && g.lda % 4 == 0 &&
         g.ldb % 4 == 0;
}

int gemm_tf32x3(const GemmDesc& g, cudaStream_t st) {
  DL_REQUIRE(tf32x3_ok(g), 1, "tf32x3: unsupported GEMM (alignment / epilogue)");
  const bool am = g.a_major == MN_MAJOR, bm = g.b_major == MN_MAJOR;
  if (!am && !bm) tc::launch_tf32x3<false, false>(g, st);
  else if (!am && bm) tc::launch_tf32x3<false, true>(g, st);
  else if (am && !bm) tc::launch_tf32x3<true, false>(g, st);
  else tc::launch_tf32x3<true, true>(g, st);
  return (g.N + tc::kXBN - 1) / tc::kXBN;
}

bool tc_pair_tiles(int M, int N) {
  const char* e = std::getenv("DL_GEMM_2CTA");
  return !(e && std::atoi(e) == 0) && N >= 256 && M >= 256;
}

int gemm_tc(const GemmDesc& g, cudaStream_t st) {
  const int bn = g.N >= 256 ? 256 : (g.N >= 128 ? 128 : 64);
  const bool am = g.a_major == MN_MAJOR, bm = g.b_major == MN_MAJOR;
  static const bool pair_ok = [] {
    const char* e = std::getenv("DL_GEMM_2CTA");
    return !(e && std::atoi(e) == 0);
  }();
  if (pair_ok && !g.no_pair && bn == 256 && g.M >= 256) {
    if (g.xf) {
      DL_REQUIRE(!am && bm && !g.rms, 1, "xf: dS.W_out operands (A K-major, B MN-major)");
      tc::launch2<false, true, false, true>(g, st);
    } else if (g.rms) {
      DL_REQUIRE(am && bm, 1, "fused rmsprop epilogue: dW_out operands are MN-major");
      tc::launch2<true, true, true>(g, st);
    } else if (!am && !bm) tc::launch2<false, false, false>(g, st);
    else if (!am && bm) tc::launch2<false, true, false>(g, st);
    else if (am && !bm) tc::launch2<true, false, false>(g, st);
    else tc::launch2<true, true, false>(g, st);
    return (g.N + 255) / 256;
  }
  DL_REQUIRE(!g.xf, 1, "xf: needs CTA-pair tiles (tc_pair_tiles)");
#define DL_TC_CASE(BN_)                                            \
  if (bn == BN_) {                                                 \
    if (!am && !bm) tc::launch<BN_, false, false>(g, st);          \
    else if (!am && bm) tc::launch<BN_, false, true>(g, st);       \
    else if (am && !bm) tc::launch<BN_, true, false>(g, st);       \
    else tc::launch<BN_, true, true>(g, st);                       \
    return (g.N + BN_ - 1) / BN_;                                  \
  }
  DL_TC_CASE(256)
  DL_TC_CASE(128)
  DL_TC_CASE(64)
#undef DL_TC_CASE
  return 0;
}

}  // namespace dl
