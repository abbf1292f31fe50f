// Dense projections on the 5th-generation tensor cores: a persistent,
// warp-specialised tcgen05 GEMM fed by TMA, with the module epilogues fused.
//
//   D[b] = act(alpha * op(A[b]) op(B[b]) + bias) + beta * C[b]      (row-major)
//
// These are the Evoformer's projections (src/attention.py:133-173 merged
// Q|K|V|gate and output projections; src/model.py:344-348 transition W1/W2;
// src/model.py:361-378 OPM projections and w_out) and their data / weight
// gradients, plus TriangleMultiplication's channel-batched contractions.
//
// Structure (one CTA per SM, 10 warps):
//   warp 0      TMA producer: A and B k-blocks (BK = 64 bf16 = one 128-byte
//               swizzle row) into a STAGES-deep shared-memory ring
//               (mbarrier full/empty pairs, transaction-count completion);
//   warp 1      allocates TMEM and issues tcgen05.mma (M = 128, N = BN,
//               K = 16) from one elected lane into one of two TMEM
//               accumulators, committing each stage back to the producer;
//   warps 2..9  epilogue: tcgen05.ld of the accumulator (lane quarter =
//               warp % 4, one column half each), alpha / bias / ReLU /
//               residual (beta * C, the
//               residual tile itself fetched by TMA), conversion, and a TMA
//               store through a swizzled, double-buffered staging tile.
// Operands may be K-major or MN-major in HBM (the weight-gradient GEMMs read
// activations transposed): both are staged with 128-byte swizzling and
// described to the tensor core accordingly, so no transpose pass exists.
// Tiles are walked persistently (tile = blockIdx.x + i * gridDim.x); the
// double-buffered accumulator lets tile i+1's MMAs run under tile i's
// epilogue.  Problems with few output tiles and a long K (weight gradients:
// K = tokens) are split along K; the partial tiles go to a per-stream fp32
// workspace and one reduction kernel sums them in a fixed order (results are
// deterministic) and applies the epilogue.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "reduce.cuh"
#include "tc_common.cuh"

namespace evo {

#ifdef EVO_GEMM_TRACE
// per-tile phase stamps of CTA 0 (tools/gemm_trace.py): [it][0] MMA waits the
// accumulator, [1] MMA has it, [2] MMAs issued, [3] epilogue warp 2 sees tfull,
// [4] epilogue done; [it][5] producer starts the tile, [6] producer done
__device__ long long g_gemm_trace[4096];
#define GT_STAMP(it, k) do { if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && (it) < 512) g_gemm_trace[(it) * 8 + (k)] = clock64(); } while (0)
#else
#define GT_STAMP(it, k) do {} while (0)
#endif

namespace {

using bf16 = __nv_bfloat16;

constexpr int BM = 128, BK = 64;
constexpr int EPI_WARPS = 8;                    // 2 per TMEM lane quarter (column halves)
constexpr int GT_THREADS = 64 + 32 * EPI_WARPS;  // + producer and MMA warps
constexpr int A_BYTES = BM * BK * 2;  // 16 KB
constexpr int STG_BYTES = 32 * 128;   // one staging tile: 32 rows x 128 B

constexpr int KB_RES = 4;             // B-resident mode: K <= 256 (four 64-wide k-blocks)
constexpr int SMEM_LIMIT = 232448;     // 227 KB of dynamic shared memory per CTA

// BRES (B resident): the whole [BN x K] B tile of the CTA's fixed N-tile is
// loaded once and stays in shared memory; only A k-blocks stream through
// the ring.  For the K <= 256 projections this halves-to-thirds the bytes
// each MMA waits for (the streamed operand is the MMA's latency bound).
// CG2 (CTA pair, tcgen05 cta_group::2): a 256 x BN tile per pair; each CTA
// holds its 128 rows of A and half (BN/2 columns) of B, the leader's MMAs
// read both CTAs' halves and each CTA's TMEM receives its 128 rows x BN.
template <int BN, bool BRES, bool CG2 = false>
struct Cfg {
  static constexpr int B_BYTES = (CG2 ? BN / 2 : BN) * BK * 2;
  static constexpr int BRES_BYTES = BRES ? KB_RES * B_BYTES : 0;
  static constexpr int STAGE = BRES ? A_BYTES : A_BYTES + B_BYTES;
  // epilogue staging buffers per warp: two (store i+1 staged while i drains)
  // for the short-K B-resident tiles, one elsewhere -- long-K tiles spend the
  // shared memory better on a deeper operand ring (more bytes in flight)
  static constexpr int STG_BUFS = BRES ? 2 : 1;
  static constexpr int STG_TOTAL = EPI_WARPS * STG_BUFS * STG_BYTES;
  static constexpr int FIT = (SMEM_LIMIT - 1024 - 512 - BRES_BYTES - STG_TOTAL) / STAGE;
  static constexpr int STAGES = FIT > 8 ? 8 : FIT;
  static constexpr int OFF_RING = BRES_BYTES;
  static constexpr int OFF_STG = OFF_RING + STAGES * STAGE;
  static constexpr int OFF_BAR = OFF_STG + STG_TOTAL;
  static constexpr int NBAR = 2 * STAGES + 4 + 2 * EPI_WARPS + 1;
  static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16 + 1024;  // +1 KB: runtime 1024-B alignment
  static constexpr int TMEM_COLS = 2 * BN;                      // two accumulators (128/256/512)
  static_assert(SMEM <= SMEM_LIMIT, "shared memory budget");
  static_assert(STAGES >= 2, "ring depth");
};

struct Params {
  int M, N, K;
  int batch, n_mt, n_nt, kblocks, kb_per_split;
  int tiles;
  int a_mn, b_mn;
  int has_res, relu, partial;
  float alpha, beta;
  const float* bias;
  // OPM layouts (k = 32): 1 = outn (rows (i, p), cols (j, q), scale rec[i*R + j]),
  // 2 = dnum (rows (i, j), cols (p, q), scale rec[row]); D is then a 4-D view
  // written through [2][32][32] staging tiles (see gemm_tc_opm)
  int pmode, R;
  const float* rec;
  int cmask;  // the C tile masks instead of adding: D = (C > 0) ? acc : 0 (ReLU backward)
  // per-warp column sums of the stored (bf16) D tile: row (m-tile * 4 + TMEM
  // lane quarter) of a [n_mt * 4, N] partial block (the bias gradient of the
  // next layer, finalised in fixed order by finalize_partials)
  float* csum;
};

// --- TMA / bulk-async helpers -------------------------------------------------

__device__ __forceinline__ void tma_load3(const CUtensorMap* m, void* dst, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(tc::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(tc::smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store3(const CUtensorMap* m, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1), "r"(c2), "r"(tc::smem_u32(src))
               : "memory");
}
// TMA load whose completion is signalled on the pair leader's mbarrier
// (``bar_cluster`` is a shared::cluster address, from mapa)
__device__ __forceinline__ void tma_load3_pair(const CUtensorMap* m, void* dst, uint32_t bar_cluster, int c0, int c1,
                                               int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(tc::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ uint32_t mapa_rank0(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(tc::smem_u32(p)));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void mma2_ss_w(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// completion of the pair's MMAs arrives on ``bar`` in both CTAs
__device__ __forceinline__ void mma2_commit_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          tc::smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_alloc2(uint32_t* slot_smem) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(slot_smem)),
               "n"(NCOLS));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS));
}

__device__ __forceinline__ void tma_store4(const CUtensorMap* m, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(tc::smem_u32(src))
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}

// UMMA shared-memory descriptor, 128-byte swizzle (layout type 2), version 1
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Operand tile of `rows` MN-rows x 64 K in shared memory, as TMA wrote it:
//  K-major : row r (128 B = 64 k) at r*128, 8-row swizzle atoms of 1 KB
//            (SBO = 1 KB); a K = 16 step advances 32 B inside the row.
//  MN-major: atom a (64 MN elements = 128 B) x 64 k-rows at a*8 KB (LBO),
//            8-k-row groups of 1 KB (SBO); a K = 16 step advances 2 KB.
__device__ __forceinline__ uint64_t op_desc(uint32_t base, int mn_major, int ks) {
  return mn_major ? sdesc_sw128(base + ks * 2048, 8192, 1024) : sdesc_sw128(base + ks * 32, 16, 1024);
}

struct TileCoord {
  int b, m0, n0, kb0, kb1, split;
};

// pair mode: tiles count M-tile pairs; ``crank`` picks the CTA's M-tile
__device__ __forceinline__ TileCoord decode(const Params& p, int t, int pair = 0, int crank = 0) {
  const int n_m = pair ? (p.n_mt + 1) / 2 : p.n_mt;
  const int per_split = p.batch * n_m * p.n_nt;
  TileCoord c;
  c.split = t / per_split;
  int r = t - c.split * per_split;
  c.b = r / (n_m * p.n_nt);
  r -= c.b * n_m * p.n_nt;
  c.m0 = (pair ? 2 * (r / p.n_nt) + crank : r / p.n_nt) * BM;
  c.n0 = (r % p.n_nt);
  c.kb0 = c.split * p.kb_per_split;
  c.kb1 = min(p.kblocks, c.kb0 + p.kb_per_split);
  return c;
}

template <int BN, bool OUT_F32, bool BRES, bool CG2>
__global__ void __launch_bounds__(GT_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmC, Params p) {
  using F = Cfg<BN, BRES, CG2>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + F::OFF_BAR);
  uint64_t* empty = full + F::STAGES;
  uint64_t* tfull = empty + F::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* rbar = tempty + 2;
  uint64_t* bfull = rbar + 2 * EPI_WARPS;  // resident B landed (BRES)
  uint32_t* slot = reinterpret_cast<uint32_t*>(bfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // CG2: CTA pair on adjacent M-tiles; rank 0 (the leader) issues the MMAs
  // and owns the smem-full and accumulator-empty barriers the pair shares
  GT_STAMP(511, 7);
  const int crank = CG2 ? (int)cluster_rank() : 0;
  const int cid = CG2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int ncl = CG2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    prefetch_tmap(&tmD);
    if (p.has_res) prefetch_tmap(&tmC);
    for (int s = 0; s < F::STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], ((BN == 64 && !OUT_F32) ? EPI_WARPS / 2 : EPI_WARPS) * (CG2 ? 2 : 1));
    }
    for (int w = 0; w < 2 * EPI_WARPS; ++w) tc::mbar_init(&rbar[w], 1);
    tc::mbar_init(bfull, 1);
  }
  if (warp == 1) {
    if constexpr (CG2) tmem_alloc2<F::TMEM_COLS>(slot);
    else tc::tmem_alloc<F::TMEM_COLS>(slot);
  }
  tc::fence_before();
  __syncthreads();
  if constexpr (CG2) cluster_sync_all();  // the leader's barriers exist before the peer signals them
  tc::fence_after();
  const uint32_t tmem = *slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      auto load_b = [&](uint8_t* sb, uint64_t* bar, int k0, int n0, int b) {
        if (!p.b_mn) {
          tma_load3(&tmB, sb, bar, k0, n0, b);
        } else {
#pragma unroll
          for (int i = 0; i < BN / 64; ++i) tma_load3(&tmB, sb + i * 8192, bar, n0 + 64 * i, k0, b);
        }
      };
      if constexpr (BRES) {  // the CTA's N-tile is fixed (gridDim.x % n_nt == 0): load its B once
        const TileCoord c = decode(p, blockIdx.x);
        expect_tx(bfull, (uint32_t)(p.kblocks * F::B_BYTES));
        for (int kb = 0; kb < p.kblocks; ++kb) load_b(smem + kb * F::B_BYTES, bfull, kb * BK, c.n0 * BN, c.b);
      }
      int stage = 0;
      uint32_t phase = 0;
      int pit = 0;
      for (int t = cid; t < p.tiles; t += ncl, ++pit) {
        const TileCoord c = decode(p, t, CG2, crank);
        const int n0 = c.n0 * BN;
        GT_STAMP(pit, 5);
        for (int kb = c.kb0; kb < c.kb1; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + F::OFF_RING + stage * F::STAGE;
          const int k0 = kb * BK;
          if constexpr (CG2) {
            // both CTAs' halves complete on the leader's full barrier
            const uint32_t fb = mapa_rank0(&full[stage]);
            if (crank == 0) expect_tx(&full[stage], 2 * F::STAGE);
            if (!p.a_mn) {
              tma_load3_pair(&tmA, sa, fb, k0, c.m0, c.b);
            } else {
              tma_load3_pair(&tmA, sa, fb, c.m0, k0, c.b);
              tma_load3_pair(&tmA, sa + 8192, fb, c.m0 + 64, k0, c.b);
            }
            uint8_t* sb = sa + A_BYTES;
            const int nh = n0 + crank * (BN / 2);  // this CTA's half of the N-tile
            if (!p.b_mn) {
              tma_load3_pair(&tmB, sb, fb, k0, nh, c.b);
            } else {
#pragma unroll
              for (int i = 0; i < BN / 128; ++i) tma_load3_pair(&tmB, sb + i * 8192, fb, nh + 64 * i, k0, c.b);
            }
          } else {
            expect_tx(&full[stage], F::STAGE);
            if (!p.a_mn) {
              tma_load3(&tmA, sa, &full[stage], k0, c.m0, c.b);
            } else {
              tma_load3(&tmA, sa, &full[stage], c.m0, k0, c.b);
              tma_load3(&tmA, sa + 8192, &full[stage], c.m0 + 64, k0, c.b);
            }
            if constexpr (!BRES) load_b(sa + A_BYTES, &full[stage], k0, n0, c.b);
          }
          if (++stage == F::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one elected lane; CG2: the leader only) ----------------
    const uint32_t idesc = tc::idesc_bf16(CG2 ? 2 * BM : BM, BN, p.a_mn != 0, p.b_mn != 0);
    if constexpr (BRES) {
      tc::mbar_wait(bfull, 0);
      tc::fence_after();
    }
    if (!CG2 || crank == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = cid; t < p.tiles; t += ncl, ++it) {
        const TileCoord c = decode(p, t, CG2, crank);
        const int acc = it & 1;
        GT_STAMP(it, 0);
        tc::mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);  // epilogue(s) drained this accumulator
        GT_STAMP(it, 1);
        tc::fence_after();
        const uint32_t dacc = tmem + (uint32_t)(acc * BN);
        for (int kb = c.kb0; kb < c.kb1; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::fence_after();
          const uint32_t sa = tc::smem_u32(smem + F::OFF_RING + stage * F::STAGE);
          const uint32_t sb = BRES ? tc::smem_u32(smem + kb * F::B_BYTES) : sa + A_BYTES;
#pragma unroll
          for (int ks = 0; ks < BK / 16; ++ks) {
            const uint32_t accum = (kb > c.kb0 || ks > 0) ? 1u : 0u;
            if constexpr (CG2)
              mma2_ss_w(dacc, op_desc(sa, p.a_mn, ks), op_desc(sb, p.b_mn, ks), idesc, accum);
            else
              tc::mma_bf16_ss_w(dacc, op_desc(sa, p.a_mn, ks), op_desc(sb, p.b_mn, ks), idesc, accum);
          }
          if constexpr (CG2) mma2_commit_w(&empty[stage]);  // both CTAs' stage is free once read
          else tc::mma_commit_w(&empty[stage]);             // the stage is free once these MMAs have read it
          if (++stage == F::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        GT_STAMP(it, 2);
        if constexpr (CG2) mma2_commit_w(&tfull[acc]);  // accumulator complete, in both CTAs' TMEM
        else tc::mma_commit_w(&tfull[acc]);
      }
    }
  } else {
    // ---------------- epilogue ----------------
    constexpr int CW = OUT_F32 ? 32 : 64;  // columns per 128-byte staging row
    // column halves of the tile (a 64-column bf16 tile has one: half the warps idle)
    constexpr int HALVES = (BN / 2 >= CW) ? 2 : 1;
    constexpr int HCOLS = BN / HALVES;
    const int ew = warp - 2;
    const int quarter = warp & 3;  // TMEM lanes this warp may access
    const int half = ew >> 2;
    if (half < HALVES) {
    uint8_t* stg = smem + F::OFF_STG + ew * F::STG_BUFS * STG_BYTES;
    int buf = 0;
    uint32_t rphase = 0;
    int it = 0;
    for (int t = cid; t < p.tiles; t += ncl, ++it) {
      const TileCoord c = decode(p, t, CG2, crank);
      const int acc = it & 1;
      const int n0 = c.n0 * BN;
      const int row0 = c.m0 + quarter * 32;
      const int zout = p.partial ? c.split : c.b;
      // residual tiles of the first two chunks are fetched before the
      // accumulator is ready, so their latency hides under this tile's MMAs
      const int nchunk = max(0, min(HCOLS, p.N - n0 - half * HCOLS) + CW - 1) / CW;
      if (p.has_res) {
        if (lane == 0) {
          bulk_wait_all_read();  // both staging buffers free
          for (int j = 0; j < nchunk && j < F::STG_BUFS; ++j) {
            const int b = buf ^ j;
            expect_tx(&rbar[2 * ew + b], STG_BYTES);
            tma_load3(&tmC, stg + b * STG_BYTES, &rbar[2 * ew + b], n0 + half * HCOLS + j * CW, row0, c.b);
          }
        }
        __syncwarp();
      }
      tc::mbar_wait(&tfull[acc], (it >> 1) & 1);
      if (warp == 2) GT_STAMP(it, 3);
      tc::fence_after();
      const uint32_t tacc = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * BN);
#pragma unroll 1
      for (int ch = 0; ch < nchunk; ++ch) {
        const int cc = half * HCOLS + ch * CW;
        uint8_t* sbuf = stg + buf * STG_BYTES;
        if (!p.has_res || ch >= F::STG_BUFS) {
          if (lane == 0) bulk_wait_read<F::STG_BUFS - 1>();  // the store that last read this buffer is done
          __syncwarp();
          if (p.has_res && lane == 0) {
            expect_tx(&rbar[2 * ew + buf], STG_BYTES);
            tma_load3(&tmC, sbuf, &rbar[2 * ew + buf], n0 + cc, row0, c.b);
          }
        }
        float v[CW];
        tc::tmem_ld32(tacc + cc, *reinterpret_cast<float(*)[32]>(&v[0]));
        if constexpr (CW == 64) tc::tmem_ld32(tacc + cc + 32, *reinterpret_cast<float(*)[32]>(&v[32]));
        tc::wait_ld();
        if (!p.partial) {
#pragma unroll
          for (int j = 0; j < CW; ++j) v[j] = p.alpha == 1.f ? v[j] : v[j] * p.alpha;
          if (p.bias) {
            if (n0 + cc + CW <= p.N && (p.N & 3) == 0) {  // 16-B vector loads of the bias slice
              const float4* b4 = reinterpret_cast<const float4*>(p.bias + n0 + cc);
#pragma unroll
              for (int j = 0; j < CW / 4; ++j) {
                const float4 b = __ldg(b4 + j);
                v[4 * j] += b.x;
                v[4 * j + 1] += b.y;
                v[4 * j + 2] += b.z;
                v[4 * j + 3] += b.w;
              }
            } else {
#pragma unroll
              for (int j = 0; j < CW; ++j) {
                const int col = n0 + cc + j;
                v[j] += col < p.N ? __ldg(p.bias + col) : 0.f;
              }
            }
          }
          if (p.relu) {
#pragma unroll
            for (int j = 0; j < CW; ++j) v[j] = fmaxf(v[j], 0.f);
          }
        }
        uint8_t* rowp = sbuf + lane * 128;
        const int sw = lane & 7;
        if (p.has_res) {
          tc::mbar_wait(&rbar[2 * ew + buf], (rphase >> buf) & 1);
          rphase ^= 1u << buf;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const uint4 r = *reinterpret_cast<const uint4*>(rowp + ((u ^ sw) << 4));
            if constexpr (OUT_F32) {
              const float rr[4] = {__uint_as_float(r.x), __uint_as_float(r.y), __uint_as_float(r.z),
                                   __uint_as_float(r.w)};
#pragma unroll
              for (int q = 0; q < 4; ++q)
                v[4 * u + q] = p.cmask ? (rr[q] > 0.f ? v[4 * u + q] : 0.f) : fmaf(p.beta, rr[q], v[4 * u + q]);
            } else {
              const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float2 f = tc::bf16x2_f2(w[q]);
                if (p.cmask) {
                  v[8 * u + 2 * q] = f.x > 0.f ? v[8 * u + 2 * q] : 0.f;
                  v[8 * u + 2 * q + 1] = f.y > 0.f ? v[8 * u + 2 * q + 1] : 0.f;
                } else {
                  v[8 * u + 2 * q] = fmaf(p.beta, f.x, v[8 * u + 2 * q]);
                  v[8 * u + 2 * q + 1] = fmaf(p.beta, f.y, v[8 * u + 2 * q + 1]);
                }
              }
            }
          }
        }
        if constexpr (!OUT_F32 && CW == 64) {
          if (p.pmode != 0) {
            // OPM layouts: scale, then this lane's two 32-value runs go to
            // [g][lane][32] (g = the chunk's two 32-column groups), the order
            // of the 4-D TMA box
            if (p.pmode == 1) {
              const int i = (c.m0 >> 5) + quarter, jc = (n0 + cc) >> 5;
              const float r0 = __ldg(p.rec + (int64_t)i * p.R + jc), r1 = __ldg(p.rec + (int64_t)i * p.R + jc + 1);
#pragma unroll
              for (int e = 0; e < 32; ++e) v[e] *= r0, v[32 + e] *= r1;
            } else {
              const float r = __ldg(p.rec + row0 + lane);
#pragma unroll
              for (int e = 0; e < 64; ++e) v[e] *= r;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              // 16-B piece (u & 3) of row g*32 + lane, 64-B swizzled (the map's
              // SWIZZLE_64B: piece ^= (row >> 1) & 3) -- at most 4-way conflicts
              const int g = u >> 2, row = g * 32 + lane;
              const int e0 = g * 32 + (u & 3) * 8;
              *reinterpret_cast<uint4*>(sbuf + row * 64 + (((u & 3) ^ ((row >> 1) & 3)) << 4)) =
                  make_uint4(tc::pack_bf16(v[e0], v[e0 + 1]), tc::pack_bf16(v[e0 + 2], v[e0 + 3]),
                             tc::pack_bf16(v[e0 + 4], v[e0 + 5]), tc::pack_bf16(v[e0 + 6], v[e0 + 7]));
            }
            tc::fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
              if (p.pmode == 1) {
                tma_store4(&tmD, sbuf, 0, 0, (n0 + cc) >> 5, (c.m0 >> 5) + quarter);
              } else {
                tma_store4(&tmD, sbuf, 0, row0 % p.R, (n0 + cc) >> 5, row0 / p.R);
              }
              bulk_commit();
            }
            if constexpr (F::STG_BUFS == 2) buf ^= 1;
            continue;
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          uint4 w;
          if constexpr (OUT_F32) {
            w = make_uint4(__float_as_uint(v[4 * u]), __float_as_uint(v[4 * u + 1]), __float_as_uint(v[4 * u + 2]),
                           __float_as_uint(v[4 * u + 3]));
          } else {
            w = make_uint4(tc::pack_bf16(v[8 * u], v[8 * u + 1]), tc::pack_bf16(v[8 * u + 2], v[8 * u + 3]),
                           tc::pack_bf16(v[8 * u + 4], v[8 * u + 5]), tc::pack_bf16(v[8 * u + 6], v[8 * u + 7]));
          }
          *reinterpret_cast<uint4*>(rowp + ((u ^ sw) << 4)) = w;
        }
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          tma_store3(&tmD, sbuf, n0 + cc, row0, zout);
          bulk_commit();
        }
        if constexpr (!OUT_F32) {
          if (p.csum) {
            // columns 2*lane, 2*lane+1 of this chunk summed over the warp's
            // 32 staged rows (the rounded values D holds; rows past M are 0)
            float2 cs = make_float2(0.f, 0.f);
#pragma unroll 8
            for (int r = 0; r < 32; ++r) {
              const uint32_t wv = *reinterpret_cast<const uint32_t*>(
                  sbuf + r * 128 + ((((lane >> 2) ^ (r & 7))) << 4) + ((lane & 3) << 2));
              cs = __fadd2_rn(cs, tc::bf16x2_f2(wv));
            }
            const int col = n0 + cc + 2 * lane;
            float* dst = p.csum + (int64_t)((c.m0 / BM) * 4 + quarter) * p.N + col;
            if (col < p.N) dst[0] = cs.x;
            if (col + 1 < p.N) dst[1] = cs.y;
          }
        }
        if constexpr (F::STG_BUFS == 2) buf ^= 1;
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) {  // accumulator may be overwritten (CG2: on the leader's barrier)
        if constexpr (CG2) mbar_arrive_cluster(mapa_rank0(&tempty[acc]));
        else tc::mbar_arrive(&tempty[acc]);
        if (warp == 2) GT_STAMP(it, 4);
      }
    }
    if (lane == 0) bulk_wait_all();
    }
  }
  tc::fence_before();
  __syncthreads();
  if constexpr (CG2) cluster_sync_all();  // neither CTA leaves while the pair's MMAs / signals are in flight
  tc::fence_after();
  if (warp == 1) {
    if constexpr (CG2) tmem_dealloc2<F::TMEM_COLS>(tmem);
    else tc::tmem_dealloc<F::TMEM_COLS>(tmem);
  }
}

__device__ __forceinline__ void store4(float* p, const float (&r)[4]) {
  if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
    *reinterpret_cast<float4*>(p) = make_float4(r[0], r[1], r[2], r[3]);
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) p[j] = r[j];
  }
}
__device__ __forceinline__ void store4(bf16* p, const float (&r)[4]) {
  if ((reinterpret_cast<uintptr_t>(p) & 7) == 0) {
    *reinterpret_cast<uint2*>(p) = make_uint2(tc::pack_bf16(r[0], r[1]), tc::pack_bf16(r[2], r[3]));
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) p[j] = __float2bfloat16(r[j]);
  }
}

// Split-K close-out: D = act(alpha * sum_s P[s] + bias) + beta * C, summed
// in split-index order (a fixed order: results are deterministic).
template <typename TD>
__device__ __forceinline__ void splitk_finish(float4 t, int64_t m, int64_t n, TD* D, int64_t ldd, const TD* Cin,
                                              int64_t ldc, float alpha, float beta, const float* __restrict__ bias,
                                              int relu) {
  float r[4] = {t.x * alpha, t.y * alpha, t.z * alpha, t.w * alpha};
  if (bias) {
    const float4 b = __ldg(reinterpret_cast<const float4*>(bias + n));
    r[0] += b.x;
    r[1] += b.y;
    r[2] += b.z;
    r[3] += b.w;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (relu) r[j] = fmaxf(r[j], 0.f);
    if (Cin) r[j] = fmaf(beta, to_f(Cin[m * ldc + n + j]), r[j]);
  }
  store4(D + m * ldd + n, r);
}

__device__ __forceinline__ void add4(float4& t, const float4 v) {
  t.x += v.x;
  t.y += v.y;
  t.z += v.z;
  t.w += v.w;
}

// Few splits, many outputs (e.g. OPM d(a), d(c): 4 splits of a 128 x 8192
// plane): one thread per 4 consecutive columns of one row walks all splits
// with up to eight 16-byte loads in flight.
template <typename TD>
__global__ void __launch_bounds__(256) splitk_reduce_quad_kernel(const float* __restrict__ ws, int splits, int64_t M,
                                                                 int64_t N, TD* D, int64_t ldd, const TD* Cin,
                                                                 int64_t ldc, float alpha, float beta,
                                                                 const float* __restrict__ bias, int relu) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nq = N >> 2;
  if (q >= M * nq) return;
  const int64_t m = q / nq;
  const int64_t n = (q - m * nq) * 4;
  const int64_t plane = M * N;
  const float* src = ws + m * N + n;
  float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
  int k = 0;
  for (; k + 8 <= splits; k += 8) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcs(reinterpret_cast<const float4*>(src + (k + u) * plane));
#pragma unroll
    for (int u = 0; u < 8; ++u) add4(t, v[u]);
  }
  for (; k < splits; ++k) add4(t, __ldcs(reinterpret_cast<const float4*>(src + k * plane)));
  splitk_finish(t, m, n, D, ldd, Cin, ldc, alpha, beta, bias, relu);
}

// Many splits, few outputs (weight gradients: up to 64 splits of a small
// plane): a block owns 32 quads (128 columns) of one row; warp w sums splits
// w, w + 8, ... (four loads in flight), and the 8 warp partials are added in
// warp order through shared memory.
template <typename TD>
__global__ void __launch_bounds__(256) splitk_reduce_wide_kernel(const float* __restrict__ ws, int splits, int64_t M,
                                                                 int64_t N, TD* D, int64_t ldd, const TD* Cin,
                                                                 int64_t ldc, float alpha, float beta,
                                                                 const float* __restrict__ bias, int relu) {
  __shared__ float4 part[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t cblocks = (N + 127) / 128;
  const int64_t m = blockIdx.x / cblocks;
  const int64_t n = (blockIdx.x % cblocks) * 128 + lane * 4;
  const bool ok = n < N;
  const int64_t plane = M * N;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (ok) {
    const float* src = ws + m * N + n;
    int k = w;
    for (; k + 24 < splits; k += 32) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(reinterpret_cast<const float4*>(src + (k + 8 * u) * plane));
#pragma unroll
      for (int u = 0; u < 4; ++u) add4(acc, v[u]);
    }
    for (; k < splits; k += 8) add4(acc, __ldcs(reinterpret_cast<const float4*>(src + k * plane)));
  }
  part[w][lane] = acc;
  __syncthreads();
  if (w != 0 || !ok) return;
  float4 t = part[0][lane];
#pragma unroll
  for (int k = 1; k < 8; ++k) add4(t, part[k][lane]);
  splitk_finish(t, m, n, D, ldd, Cin, ldc, alpha, beta, bias, relu);
}

// --- host side ----------------------------------------------------------------

}  // namespace

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda);
// shared with the attention kernels (attention_tc_fwd2.cu)
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

namespace {

// 3-D tiled map over a row-major [z][rows][cols] view (cols contiguous), box
// {box_cols, box_rows, 1}, 128-byte swizzle.  false when TMA cannot address it.
bool make_map(CUtensorMap* m, const void* base, bool f32, int64_t cols, int64_t rows, int64_t ld, int64_t zs,
              int64_t nz, int box_cols, int box_rows) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  const int64_t es = f32 ? 4 : 2;
  if (((uintptr_t)base & 15) || (ld * es) % 16 || (zs * es) % 16) return false;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)nz};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * es), (cuuint64_t)((nz > 1 ? zs : rows * ld) * es)};
  if (strides[1] == 0 || strides[1] % 16) strides[1] = (cuuint64_t)(rows * ld * es);
  cuuint32_t box[3] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = enc(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                         const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

struct SplitWs {
  float* ptr = nullptr;
  size_t bytes = 0;
};
constexpr size_t SPLIT_WS_BYTES = size_t(32) << 20;

// per-device, per-stream-slot split-K workspaces, all allocated on the first
// use (never inside a CUDA-graph capture, which forbids cudaMalloc)
SplitWs& split_ws(cudaStream_t s) {
  static SplitWs ws[16][EVO_STREAM_SLOTS];
  static std::mutex mu;
  int dev = 0;
  EVO_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (!ws[dev & 15][0].ptr) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    EVO_CUDA(cudaStreamIsCapturing(s, &cap));
    if (cap == cudaStreamCaptureStatusNone) {
      for (int k = 0; k < EVO_STREAM_SLOTS; ++k) {
        EVO_CUDA(cudaMalloc(&ws[dev & 15][k].ptr, SPLIT_WS_BYTES));
        ws[dev & 15][k].bytes = SPLIT_WS_BYTES;
      }
    }
  }
  return ws[dev & 15][stream_slot(s)];
}

int64_t g_tc_gemms = 0;  // tensor-core GEMMs launched (evo_gemm_tc_launches)

template <int BN, bool OUT_F32, bool BRES, bool CG2 = false>
void launch(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& d, const CUtensorMap& c, const Params& p,
            int grid, cudaStream_t s) {
  using F = Cfg<BN, BRES, CG2>;
  auto k = gemm_tc_kernel<BN, OUT_F32, BRES, CG2>;
  static std::once_flag once;
  std::call_once(once, [&] { EVO_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, F::SMEM)); });
  if constexpr (CG2) {  // CTA pairs: a 2 x 1 x 1 cluster
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(GT_THREADS);
    cfg.dynamicSmemBytes = F::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    EVO_CUDA(cudaLaunchKernelEx(&cfg, k, a, b, d, c, p));
  } else {
    k<<<grid, GT_THREADS, F::SMEM, s>>>(a, b, d, c, p);
  }
  EVO_LAUNCH_CHECK();
  count_launch(1);
  ++g_tc_gemms;
}

bool cg2_disabled() {  // A/B switch (EVO_GEMM_CG2=0): single-CTA kernels only
  static const bool v = [] {
    const char* e = getenv("EVO_GEMM_CG2");
    return e && e[0] == '0';
  }();
  return v;
}

bool bres_disabled() {  // A/B switch for measurements (EVO_GEMM_BRES=0)
  const char* e = getenv("EVO_GEMM_BRES");
  return e && e[0] == '0';
}

int forced_bn() {  // tile-width sweeps (tools/gemm_sweep.py): EVO_GEMM_BN=64|128
  static const int v = [] {
    const char* e = getenv("EVO_GEMM_BN");
    return e ? atoi(e) : 0;
  }();
  return v == 64 || v == 128 ? v : 0;
}

bool tc_gemm_disabled() {
  static const bool v = [] {
    const char* e = getenv("EVO_DISABLE_TC_GEMM");
    return e && e[0] == '1';
  }();
  return v;
}

}  // namespace

// Split-K workspace of the stream's slot (nullptr before the first non-capturing
// GEMM) and its close-out; shared with the CUDA-core GEMM (gemm_simt.cu).
float* gemm_split_ws(cudaStream_t s, size_t* bytes) {
  SplitWs& w = split_ws(s);
  *bytes = w.bytes;
  return w.ptr;
}

void splitk_reduce(const float* ws, int splits, int64_t M, int64_t N, void* D, int64_t ldd, const void* Cin,
                   int64_t ldc, float alpha, float beta, const float* bias, int relu, int d_dtype, cudaStream_t s) {
  EVO_REQUIRE(N % 4 == 0, EVO_ERR_ARG, "split-K reduce: N % 4 != 0");
  // thread per quad when that alone fills the GPU (each thread then keeps up to
  // eight split loads in flight); the split-parallel layout for few outputs
  const bool wide = splits >= 8 && M * (N / 4) < (int64_t)num_sms() * 128;
  const int64_t blocks = wide ? M * ((N + 127) / 128) : (M * (N / 4) + 255) / 256;
  EVO_REQUIRE(blocks < (1ll << 31), EVO_ERR_ARG, "split-K reduce: bad extents");
#define EVO_SPLITK(KERN, T) \
  KERN<T><<<(unsigned)blocks, 256, 0, s>>>(ws, splits, M, N, (T*)D, ldd, (const T*)Cin, ldc, alpha, beta, bias, relu)
  if (d_dtype == EVO_F32) {
    if (wide) EVO_SPLITK(splitk_reduce_wide_kernel, float); else EVO_SPLITK(splitk_reduce_quad_kernel, float);
  } else {
    if (wide) EVO_SPLITK(splitk_reduce_wide_kernel, bf16); else EVO_SPLITK(splitk_reduce_quad_kernel, bf16);
  }
#undef EVO_SPLITK
  EVO_LAUNCH_CHECK();
  count_launch(1);
}

// Row-major D[b] = act(alpha * op(A[b]) op(B[b]) + bias) + beta * C[b] on the
// tensor cores; A, B bf16; D and C (may alias D) of dtype d_dtype.  Returns
// false (caller uses the SIMT kernel) when TMA cannot address an operand.
namespace {
// OPM output layouts of gemm_tc_impl (k = 32 only)
struct OpmOut {
  int mode;          // 1 = outn, 2 = dnum
  const float* rec;  // outn: [NI*R] by (i, j); dnum: [NI*R] by the GEMM row
  int64_t R, NI;
};

// 4-D views of the OPM outputs for TMA stores of [2][32][32] bf16 boxes,
// 64-byte swizzled (inner extent 64 B):
//   outn [NI*R, k*k]:  (q, p, j, i), strides (1, k, k*k, R*k*k)
//   dnum [NI*k, R*k]:  (q, j, p, i), strides (1, k, R*k, k*R*k)
bool opm_map(CUtensorMap* m, void* base, const OpmOut& o) {
  auto enc = tmap_encoder();
  if (!enc || ((uintptr_t)base & 15)) return false;
  const cuuint64_t k = 32, R = (cuuint64_t)o.R, NI = (cuuint64_t)o.NI;
  cuuint64_t dims[4], strides[3];
  if (o.mode == 1) {
    dims[0] = k, dims[1] = k, dims[2] = R, dims[3] = NI;
    strides[0] = k * 2, strides[1] = k * k * 2, strides[2] = R * k * k * 2;
  } else {
    dims[0] = k, dims[1] = R, dims[2] = k, dims[3] = NI;
    strides[0] = k * 2, strides[1] = R * k * 2, strides[2] = k * R * k * 2;
  }
  cuuint32_t box[4] = {32, 32, 2, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}
}  // namespace

static bool gemm_tc_impl(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int ta, int64_t sa,
                         const void* B, int64_t ldb, int tb, int64_t sb, void* D, int64_t ldd, int64_t sd, int batch,
                         float alpha, float beta, const void* Cin, int64_t ldc, const float* bias, int relu,
                         int d_dtype, cudaStream_t s, const OpmOut* opm, int cmask = 0, float* csum = nullptr);

bool gemm_tc(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int ta, int64_t sa, const void* B,
             int64_t ldb, int tb, int64_t sb, void* D, int64_t ldd, int64_t sd, int batch, float alpha,
             float beta, const void* Cin, int64_t ldc, const float* bias, int relu, int d_dtype, cudaStream_t s) {
  return gemm_tc_impl(M, N, K, A, lda, ta, sa, B, ldb, tb, sb, D, ldd, sd, batch, alpha, beta, Cin, ldc, bias, relu,
                      d_dtype, s, nullptr);
}

// The OPM contractions with the normalisation and re-layout in the epilogue
// (src/model.py:366-378):
//   outn[i*R + j, p*k + q] = rec[i*R + j] * sum_s a[s, i*k + p] c[s, j*k + q]      (mode 1)
//   dnum[i*k + p, j*k + q] = rec[i*R + j] * sum_c d[(i, j), c] w_out[p*k + q, c]   (mode 2)
bool gemm_tc_opm(int mode, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int ta, const void* B,
                 int64_t ldb, int tb, void* D, const float* rec, int64_t R, int64_t NI, cudaStream_t s) {
  if (mode == 1 && (M != NI * 32 || N != R * 32)) return false;
  if (mode == 2 && (M != NI * R || N != 32 * 32 || R % BM)) return false;
  const OpmOut o{mode, rec, R, NI};
  return gemm_tc_impl(M, N, K, A, lda, ta, 0, B, ldb, tb, 0, D, N, 0, 1, 1.f, 0.f, nullptr, 0, nullptr, 0, EVO_BF16, s,
                      &o);
}

// D = (h > 0) ? op(A) op(B) : 0 -- the ReLU backward in the epilogue of the
// d(hidden) GEMM (h: the saved ReLU output, [M, N] like D)
int64_t gemm_tc_relu_mask_ws(int64_t M, int64_t N) { return ((M + BM - 1) / BM) * 4 * N * 4; }

bool gemm_tc_relu_mask(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int ta, const void* B,
                       int64_t ldb, int tb, const void* h, void* D, int d_dtype, cudaStream_t s, float* colsum,
                       int accumulate, void* ws) {
  float* part = colsum ? partial_buffer(ws, (size_t)gemm_tc_relu_mask_ws(M, N)) : nullptr;
  if (!gemm_tc_impl(M, N, K, A, lda, ta, 0, B, ldb, tb, 0, D, N, 0, 1, 1.f, 0.f, h, N, nullptr, 0, d_dtype, s,
                    nullptr, 1, part))
    return false;
  if (colsum) finalize_partials(part, (int)(((M + BM - 1) / BM) * 4), N, colsum, accumulate, s);
  return true;
}

static bool gemm_tc_impl(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int ta, int64_t sa,
                         const void* B, int64_t ldb, int tb, int64_t sb, void* D, int64_t ldd, int64_t sd, int batch,
                         float alpha, float beta, const void* Cin, int64_t ldc, const float* bias, int relu,
                         int d_dtype, cudaStream_t s, const OpmOut* opm, int cmask, float* csum) {
  if (tc_gemm_disabled()) return false;
  if (csum && (d_dtype != EVO_BF16 || batch != 1)) return false;
  if (M <= 0 || N <= 0 || K <= 0 || batch < 1) return false;
  if (M > (1ll << 31) - BM || N > (1ll << 31) - 256 || K > (1ll << 31) - BK) return false;
  const bool f32 = d_dtype == EVO_F32;
  const bool has_res = Cin != nullptr && (beta != 0.f || cmask);
  int BN = N <= 64 ? 64 : (N <= 128 ? 128 : 256);
  // split-K problems (few output tiles, long K): 128-wide tiles give twice
  // the tiles per split and halve each CTA's B stream (measured faster on
  // every weight-gradient shape of the block)
  // -- unless CTA pairs take them (cta_group::2, 256 x 256 per pair, each CTA
  // streaming only half of B: half the L2->SM bytes per output of 128 x 128
  // tiles, which is what bounds these GEMMs)
  // Off by default: 5% faster in isolation, but in the two-stream step the
  // CTA pairs (two co-scheduled SMs) measured 0.5 ms slower (EVO_GEMM_CG2_SPLIT=1 enables)
  static const bool cg2_split = [] {
    const char* e = getenv("EVO_GEMM_CG2_SPLIT");
    return e && e[0] == '1';
  }();
  // (measured: 256x1024 and 1024x256 weight gradients 5% faster; with fewer
  // than 8 pair-halves per split, e.g. 256x256, slower -- tools/splitk_sweep.py)
  const bool pair_split = cg2_split && !opm && !cmask && batch == 1 && (M + BM - 1) / BM >= 2 &&
                          ((M + BM - 1) / BM) * ((N + 255) / 256) >= 8 && !cg2_disabled();
  // (EVO_GEMM_SPLIT_BN=0: 256-wide tiles with >= 2 M-tiles and >= 8 256-wide
  // tiles -- 256x1024 / 1024x256 dW 24.5 -> 22.7 / 24.6 -> 23.2 us in
  // isolation, but the bench step measured 101.8 vs 101.6 ms, so off; =256:
  // always 256-wide)
  static const int split_bn = [] {
    const char* e = getenv("EVO_GEMM_SPLIT_BN");
    return e ? atoi(e) : 128;
  }();
  const int64_t mt = (M + BM - 1) / BM, nt256 = (N + 255) / 256;
  const bool wide_split = split_bn == 256 || (split_bn == 0 && mt >= 2 && mt * nt256 >= 8);
  if (BN == 256 && batch == 1 && mt * nt256 < num_sms() && (K + BK - 1) / BK >= 16 && !pair_split && !wide_split)
    BN = 128;
  if (const int f = forced_bn(); f && f < BN) BN = f;
  Params p{};
  p.M = (int)M;
  p.N = (int)N;
  p.K = (int)K;
  p.batch = batch;
  p.n_mt = (int)((M + BM - 1) / BM);
  p.n_nt = (int)((N + BN - 1) / BN);
  p.kblocks = (int)((K + BK - 1) / BK);
  p.a_mn = ta ? 1 : 0;
  p.b_mn = tb ? 0 : 1;
  p.alpha = alpha;
  p.beta = beta;
  p.bias = bias;
  p.relu = relu;
  p.has_res = has_res ? 1 : 0;
  p.cmask = cmask;
  p.csum = csum;
  const int nsm = num_sms();
  const int64_t base = (int64_t)batch * p.n_mt * p.n_nt;
  if (base > (1ll << 30)) return false;
  // split K when the output tiles cannot fill the SMs and K is long
  int splits = 1;
  if (!opm && !cmask && !csum && batch == 1 && base < nsm && p.kblocks >= 16 && N % 4 == 0) {
    // >= 8 k-blocks (K >= 512) per split; at most 64 partial planes; the
    // split tiles must fit one wave of the persistent grid (a second, mostly
    // idle wave doubles the kernel time)
    splits = (int)(nsm / base);
    if (splits > p.kblocks / 8) splits = p.kblocks / 8;
    if (splits > 64) splits = 64;
    if (const char* e = getenv("EVO_GEMM_SPLITS")) {  // tuning sweeps (tools/splitk_sweep.py)
      const int f = atoi(e);
      if (f > 0) splits = f < p.kblocks ? f : p.kblocks;
    }
    SplitWs& ws = split_ws(s);
    while (splits > 1 && (size_t)splits * M * N * 4 > ws.bytes) --splits;
    if (!ws.ptr) splits = 1;
  }
  p.kb_per_split = (p.kblocks + splits - 1) / splits;
  splits = (p.kblocks + p.kb_per_split - 1) / p.kb_per_split;
  p.partial = splits > 1 ? 1 : 0;
  p.tiles = (int)(base * splits);
  // B resident: short K, several M-tiles per CTA; the grid is a multiple of
  // the N-tile count so each CTA keeps one N-tile (tile t -> n = t % n_nt)
  const bool bres = !p.partial && BN >= 128 && p.kblocks <= KB_RES && p.n_nt <= nsm &&
                    p.tiles >= 2 * nsm && !bres_disabled();
  // otherwise CTA pairs (tcgen05 cta_group::2, 256 x BN per pair, each CTA
  // receiving half the B bytes per k-block) for the 256-wide, K >= 512,
  // unsplit problems: measured 5-9% faster there (tools/gemm_shapes.py),
  // neutral-to-slower for 128-wide tiles, short K and split-K partials
  static const int cg2_minkb = [] {  // sweeps: EVO_GEMM_CG2_MINKB
    const char* e = getenv("EVO_GEMM_CG2_MINKB");
    return e ? atoi(e) : 8;
  }();
  const bool cg2 = !bres && BN == 256 && (!p.partial || pair_split) && p.kblocks >= cg2_minkb && p.n_mt >= 2 &&
                   !cg2_disabled();
  if (cg2) p.tiles = (int)((int64_t)batch * ((p.n_mt + 1) / 2) * p.n_nt * splits);

  CUtensorMap ma, mb, md, mc;
  // A: K-major [M, K] (lda) or MN-major [K, M]
  if (!ta) {
    if (!make_map(&ma, A, false, K, M, lda, sa, batch, 64, BM)) return false;
  } else if (!make_map(&ma, A, false, M, K, lda, sa, batch, 64, BK)) {
    return false;
  }
  if (tb) {
    if (!make_map(&mb, B, false, K, N, ldb, sb, batch, 64, cg2 ? BN / 2 : BN)) return false;
  } else if (!make_map(&mb, B, false, N, K, ldb, sb, batch, 64, BK)) {
    return false;
  }
  float* wsp = nullptr;
  if (opm) {
    p.pmode = opm->mode;
    p.rec = opm->rec;
    p.R = (int)opm->R;
    if (!opm_map(&md, D, *opm)) return false;
  } else if (p.partial) {
    wsp = split_ws(s).ptr;
    if (!make_map(&md, wsp, true, N, M, N, M * N, splits, 32, 32)) return false;
  } else if (!make_map(&md, D, f32, N, M, ldd, sd, batch, f32 ? 32 : 64, 32)) {
    return false;
  }
  if (has_res && !p.partial) {
    if (!make_map(&mc, Cin, f32, N, M, ldc, sd, batch, f32 ? 32 : 64, 32)) return false;
  } else {
    mc = md;
    p.has_res = 0;
  }
  int grid = (int)(p.tiles < nsm ? p.tiles : nsm);
  const bool out32 = p.partial || f32;
  if (bres) grid = (nsm / p.n_nt) * p.n_nt;
  if (cg2) grid = 2 * (p.tiles < nsm / 2 ? p.tiles : nsm / 2);
#define EVO_GL(BNV, BR, C2) \
  (out32 ? launch<BNV, true, BR, C2>(ma, mb, md, mc, p, grid, s) : launch<BNV, false, BR, C2>(ma, mb, md, mc, p, grid, s))
  if (BN == 256) {
    if (bres) EVO_GL(256, true, false);
    else if (cg2) EVO_GL(256, false, true);
    else EVO_GL(256, false, false);
  } else if (BN == 128) {
    if (bres) EVO_GL(128, true, false);
    else if (cg2) EVO_GL(128, false, true);
    else EVO_GL(128, false, false);
  } else {
    EVO_GL(64, false, false);
  }
#undef EVO_GL
  if (p.partial) splitk_reduce(wsp, splits, M, N, D, ldd, has_res ? Cin : nullptr, ldc, alpha, beta, bias, relu,
                               d_dtype, s);
  return true;
}

}  // namespace evo

extern "C" int64_t evo_gemm_tc_launches(void) { return evo::g_tc_gemms; }

#ifdef EVO_GEMM_TRACE
extern "C" int evo_gemm_trace_read(long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, evo::g_gemm_trace, sizeof(long long) * n);
}
#endif
