// tcgen05 engines (TF32x3, F16x3) of the two ICNNM contractions: shared
// host/device declarations.  See icnnm_tc.cu for the kernel design.
#pragma once
#include <cuda.h>  // CUtensorMap (types only; encoded through the runtime's driver entry point)

#include <cstddef>
#include <cstdint>

#include "icnnm_kernels.cuh"

namespace icnnm_dev {
namespace tc {

constexpr int KC = 16;                         // K per chunk (tf32: 2 MMA K-steps of 8; f16: 1 of 16)
constexpr int SA = 16;                         // TMEM A stages (max; runtime a.sa); tf32: 2*KC
                                               // columns each, f16: KC columns (2 halves / column)
constexpr int NSC = 8;                         // F16x3 forward: per-brick scale ring
constexpr int SB = 16;                         // SMEM B stages (max; runtime a.sb)
constexpr int WS = 8;                          // SMEM W stages (max; runtime a.ws, even)
constexpr int W_STAGE_BYTES = 128 * KC * 4;    // adjoint: 8 KB W chunk, 16 columns x 128 rows
constexpr int WO_STAGE_BYTES = 128 * 32 * 4;   // forward: 16 KB W group, 32 columns x 128 rows
constexpr int NTMAX = 208;                     // max accumulator width (N per tile)
constexpr int B_STAGE_BYTES = 256 * KC * 4 * 2;    // hi + lo, up to 256 rows = 32 KB (tf32;
                                                   // also the packed-block stride in global)
constexpr int B_STAGE_F16 = 256 * KC * 2 * 2;      // f16 hi + lo: 16 KB SMEM stage
constexpr int BAR_BYTES = 1024;  // mbarriers + scale ring + halo maxima + halo barriers
static_assert((2 * SA + 2 * SB + 4 + 2 * WS + NSC) * 8 + NSC * 4 + 16 * 4 + 2 * 4 * 8 <= BAR_BYTES,
              "barrier block overflows BAR_BYTES");
constexpr int NPREP = 4;  // forward: halo-preparation warps
constexpr int NHB_MAX = 4;  // forward: halo buffers (max; runtime a.nhb)
// CTA pairs hold half of every B tile (N split across the pair)
inline int b_stage_bytes(bool f16, bool pair = false) {
  return f16 ? (pair ? B_STAGE_F16 / 2 : B_STAGE_F16) : B_STAGE_BYTES;
}

constexpr int TAPMAX = 4096;  // taps (the C ABI's kernel-size limit), padded to 32

struct alignas(64) TcArgs {
  // CTA pairs (F16x3): 2-D views (rows of 32 B) of the packed B tiles for
  // cp.async.bulk.tensor .cta_group::2 -- each CTA's half-tile copy signals
  // the leader's B_full directly; [0]: box of wbase/2 rows, [1]: nlast/2 rows
  CUtensorMap tmB[2];
  int tma_pair;          // 1: pair B halves via tmB (no relay); 0: bulk copies + relay
  Geo g;                 // kp = ktp = roundup(k, 32)
  const float* src;      // forward: L~ (natural [H,W,T] layout, slab halo rows first)
  const float* Win;      // adjoint: W in this engine's layout
  float* Wout;           // forward: W (read-modify-write in mode 1)
  const float* Bpk;      // pre-packed B tiles [nt][kc][hi|lo][q][n/8][2][8][4]
  const float* cvec;     // shrink factors (mode 1)
  float* adj;            // adjoint output (natural layout, slab halo rows first)
  double* norm2;         // forward: column norms^2 accumulator
  const IterState* st;
  int mode;              // 0: plain operator, 1: ADMM iteration
  int ntn;               // N-tiles per brick
  int nkc;               // K-chunks per N-tile
  int nlast;             // width of the last N-tile (multiple of 16)
  int wbase;             // width of the other N-tiles (multiple of 16, <= NTMAX)
  int accw;              // TMEM accumulator width (= wbase): acc0 @0, acc1 @accw, A @2*accw
  int sa;                // A stages used (<= SA, limited by TMEM)
  int64_t nbricks;
  unsigned long long* dbg;  // optional: per-role wait cycles (see DBG_*), or null
  int skip;                 // timing experiments only: 1 = no build work, 2 = no epilogue work
  int sb;                   // B stages used (<= SB)
  int ws;                   // adjoint W stages used (<= WS)
  int bsplit;               // A build: 0 = the two 4-warp groups own alternate K-chunks
                            // (16 columns each); 1 = both groups split every chunk (TF32x3)
  float bunscale;           // F16x3: 2^-eB, the inverse of the power-of-2 scale of B
  float amax;               // F16x3 adjoint, mode 0: bound on |W| (mode 1: st->adj_amax)
  int bpair;                // builders hand over owned chunks in pairs (one wait::st)
  int grp;                  // N-tiles per tile group sharing each built A chunk (1 or 2)
  int skew;                 // tile-group schedule skew D (chunks), see tg_seq
  int cs;                   // 2: CTA pairs (cta_group::2, M = 256, B split by N); 1: single CTAs
  int mcb;                  // F16x3 single CTAs in 2-CTA clusters sharing one multicast B stream
  int ehalf;                // adjoint: epilogue halves in use (1 or 2; 4 warps and 4 output
                            // bricks each -- 2 when the extra output bricks fit in SMEM)
  int nsplit;               // CTA roles per brick (1: a CTA does whole bricks); forward: N-tile
                            // ranges, adjoint: K-chunk ranges (single CTAs only)
  int bres;                 // 1: the role's B tiles are resident in SMEM (one load per launch)
  int bres_stride;          // resident B: bytes per (tile, chunk) block
  int bres_bytes;           // resident B: SMEM bytes of the role's resident blocks
  int bmix;                 // 1: mixed residency -- only the role's first nresblk (tile, chunk)
                            // blocks are resident, the rest stream through the sb-stage ring
                            // (whole bricks per CTA: A built once per brick, B half-streamed)
  int nresblk;              // mixed residency: resident blocks, in (tile, chunk) order
  // deterministic reductions (null: fp32 / fp64 atomics as before)
  float2* adjq;             // adjoint (mode 1): {hi, lo} fixed-grid output pairs, adj's layout
  double* npart;            // forward: per-CTA column partials [grid][kp] (mode 2: [grid])
  int nhb;                  // forward: halo buffers (2..NHB_MAX; the prep warps run nhb-2 ahead)
  int bstride;              // F16x3 single CTAs: B ring stage stride in bytes (0: B_STAGE_F16)
  int warr;                 // 1: one mbarrier arrival per warp (lane 0 after __syncwarp); 0: per thread
  // Tap table: minus the byte offset of tap s inside the halo / output box, in
  // this kernel's tap order (forward: t fastest; adjoint: the N order of its B
  // tiles).  In the parameters so that the warp-uniform index reads go through
  // the constant bank into uniform registers (tc_fill_taps).
  alignas(16) int tapn[TAPMAX];
};
void tc_fill_taps(TcArgs& a, bool fwd);

// dbg slots (cycles summed over CTAs)
enum { DBG_BUILD_WAIT = 0, DBG_BUILD_WORK, DBG_MMA_WAIT_A, DBG_MMA_WAIT_B, DBG_MMA_WAIT_ACC,
       DBG_EPI_WAIT, DBG_EPI_WORK, DBG_LOAD_WAIT, DBG_TOTAL, DBG_BUILD_PREP, DBG_SLOTS };

template <bool FWD, bool F16>
__global__ void icnnm_tc_kernel(TcArgs a);

void* fwd_kernel_ptr(bool f16, bool pair = false);
void* adj_kernel_ptr(bool f16, bool pair = false);

// 8 builder + 8 epilogue + MMA + B loader + W loader warps (both kernels);
// the forward adds NPREP halo-preparation warps
inline int threads(bool fwd) { return fwd ? 608 + 32 * NPREP : 608; }

inline size_t smem_bytes(const Geo& g, bool fwd, int sb, int ws, bool f16, bool pair = false,
                         int ehalf = 1, int bres_bytes = 0, int nhb = 2, int bstride = 0,
                         bool bmix = false) {
  const size_t nob = static_cast<size_t>(g.HH) * g.HW * g.HT;
  const size_t nobp = ((nob + 3) / 4) * 4;
  const size_t stage = bstride > 0 ? static_cast<size_t>(bstride) : b_stage_bytes(f16, pair);
  size_t b = static_cast<size_t>(bres_bytes) +
             ((bres_bytes > 0 && !bmix) ? 0 : static_cast<size_t>(sb) * stage) +
             static_cast<size_t>(ws) * (fwd ? WO_STAGE_BYTES : W_STAGE_BYTES) + BAR_BYTES + 16;
  b += ((g.ktp * 4 + 15) / 16) * 16;
  b += ((g.kp * 4 + 15) / 16) * 16;
  if (fwd)
    b += static_cast<size_t>(nhb) * nobp * 4 + static_cast<size_t>(g.kp) * 8;
  else
    b += static_cast<size_t>(4 * ehalf) * (nobp + 32) * 4;
  return b;
}

}  // namespace tc
}  // namespace icnnm_dev
