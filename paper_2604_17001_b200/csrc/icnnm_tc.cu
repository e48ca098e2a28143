// ICNNM forward / adjoint contractions on the 5th-gen tensor cores (sm_100a).
//
// Each fp32 GEMM is computed from a hi/lo split of both operands with fp32
// accumulation in TMEM, three MMAs per K-step:
//     D += A_hi B_hi + A_lo B_hi + A_hi B_lo
// Engine ICNNM_ENGINE_TF32X3: x_hi = rna_tf32(x), x_lo = x - x_hi,
//   tcgen05.mma kind::tf32 (K = 8 per MMA).
// Engine ICNNM_ENGINE_F16X3: x_hi = rn_f16(s x), x_lo = rn_f16(s x - x_hi) with a
//   power-of-2 scale s that puts max|x| below 2^14, tcgen05.mma kind::f16
//   (K = 16 per MMA at the same cycle cost: half the MMA time).  Both keep
//   ~22 mantissa bits of every product.  Scales: B (the basis)
//   once on the host; forward A per brick from the max of the brick's halo
//   (builders -> epilogue through a ring of mbarrier-guarded slots); adjoint A
//   from the bound |W_vj c_j| <= min(n_j, 1/theta) computed by the coef kernel.
//
// Kernel shape (persistent, one CTA per SM, 576 (forward) / 480 (adjoint) threads):
//   warps 0-7  builders : im2col / scaled-W rows -> hi/lo split -> tcgen05.st
//                         into a TMEM A-stage (row = TMEM lane = voxel); the two
//                         4-warp groups own alternate K-chunks
//   warps 8..  epilogue : tcgen05.ld the accumulator; forward: W update +
//                         column norms; adjoint: col2im into per-warp SMEM
//                         output bricks, flushed with one atomic per entry
//   next warp  MMA      : one elected thread issues tcgen05.mma (A from TMEM,
//                         B from SMEM via a SWIZZLE_NONE K-major descriptor)
//   next warp  loader   : cp.async.bulk of host-pre-packed B tiles (UMMA
//                         canonical layout) into an SMEM ring; the adjoint has
//                         one more warp streaming W chunks
// TMEM: two accumulators of accw <= 208 columns (epilogue of tile i overlaps
// the MMAs of tile i+1) + sa A stages (tf32: 2*KC columns, f16: KC columns).
//
// Forward  (a)+(b): D[v, j] = sum_s L~[v - s] K[s, j]          (N = columns j)
// Adjoint  (c)    : D[v, s] = sum_j W[v, j] c_j K[s, j]        (N = taps s)
// W layout (this engine): [brick][j][row] (column-major per brick), so
// epilogue/builder threads (one per row) access it coalesced and any column
// range of a brick is one contiguous block.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "icnnm_kernels.cuh"
#include "icnnm_tc.cuh"

namespace icnnm_dev {
namespace tc {

// Work-skipping timing switches (TcArgs::skip) exist only in the experiments
// build (make EXPERIMENTS=1); the shipped kernels compile them out.
// So do the in-kernel pipeline counters (TcArgs::dbg) and the per-thread
// barrier arrivals (TcArgs::warr = 0): in the shipped kernels every role's
// chunk loop is short enough that these checks showed up in its time.
#ifdef ICNNM_EXPERIMENTS
#define TC_SKIP(a) ((a).skip)
#define TC_DBG(a) ((a).dbg)
#define TC_WARR(a) ((a).warr != 0)
#define TC_BPAIR(a) ((a).bpair != 0)
#else
#define TC_SKIP(a) 0
#define TC_DBG(a) (static_cast<unsigned long long*>(nullptr))
#define TC_WARR(a) true
#define TC_BPAIR(a) false
#endif

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#ifdef ICNNM_WAIT_HINT
  // A/B: suspend-time hint (ns) -- a waiting warp sleeps longer per probe and
  // takes fewer issue slots from the working warps
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(static_cast<uint32_t>(ICNNM_WAIT_HINT))
      : "memory");
#else
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#endif
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Multicast bulk copy: the bytes land at the same shared-memory offset in every
// CTA of ctaMask, each of whose mbarrier at the same offset gets complete_tx.
__device__ __forceinline__ void bulk_g2s_mc(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
// 2-SM tensor copy: box at (0, row) of a 2-D tensor map into this CTA's
// shared memory, complete_tx signalled on `bar_cluster` -- with .cta_group::2
// the barrier may live in the peer CTA of the pair (the leader's B_full).
__device__ __forceinline__ void tma2d_pair(void* dst, const CUtensorMap* map, int row,
                                           uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.cta_group::2 "
      "[%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(row), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
// Issued by one elected lane of a converged warp (the warp-uniform operands
// stay in uniform registers; no per-MMA divergence).
__device__ __forceinline__ void tc_mma_ts_elect(uint32_t d, uint32_t a, uint64_t bdesc,
                                                uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tc_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}
// ---- CTA-pair (cta_group::2) primitives ----
// The address of the same shared-memory object in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa_u32(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// Arrive on a (possibly remote) mbarrier.  Default (CTA-scope) semantics, as
// CUTLASS's ClusterBarrier::arrive(cta_id): what these arrivals publish is TMEM
// state ordered by tcgen05.wait::{st,ld} + tcgen05.fence::before_thread_sync,
// or a TMA completion already observed through the local barrier.  The
// .release.cluster form compiled to MEMBAR.ALL.GPU + ERRBAR per arrive (22% of
// the pair forward's stall samples, profiles/ab_r1/pairs_skip/).
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}
// Wait whose acquire covers arrivals released by the peer CTA.
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// One F16x3 K-chunk of a CTA pair (M = 256: 128 rows from each CTA's TMEM A
// stage, B split by N between the two CTAs' shared memory), issued by the
// leader; commits are multicast to the barrier at the same offset in both CTAs.
__device__ __forceinline__ void tc_chunk_f16_pair(uint32_t d, uint32_t a, uint32_t alo, uint64_t dh,
                                                  uint64_t dl, uint32_t idesc, uint32_t accum,
                                                  uint32_t bar_b, uint32_t bar_a, uint32_t bar_acc,
                                                  uint32_t flags) {
  asm volatile(
      "{\n"
      ".reg .pred e, p, t, qa, qc;\n"
      ".reg .b32 f;\n"
      ".reg .b16 m;\n"
      "mov.b16 m, 3;\n"
      "setp.ne.b32 p, %6, 0;\n"
      "setp.eq.b32 t, %6, %6;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "and.b32 f, %10, 1;\n"
      "setp.ne.b32 qa, f, 0;\n"
      "and.b32 f, %10, 2;\n"
      "setp.ne.b32 qc, f, 0;\n"
      "and.pred qa, qa, e;\n"
      "and.pred qc, qc, e;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %3, %5, p;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%2], %3, %5, t;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %4, %5, t;\n"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%7], m;\n"
      "@qa tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%8], m;\n"
      "@qc tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%9], m;\n"
      "}\n" ::"r"(d),
      "r"(a), "r"(alo), "l"(dh), "l"(dl), "r"(idesc), "r"(accum), "r"(bar_b), "r"(bar_a),
      "r"(bar_acc), "r"(flags)
      : "memory");
}
// kind::f16 instruction descriptor for M = 256 (CTA pair): D f32, A/B f16, K-major.
__device__ __forceinline__ uint32_t idesc_f16_m256(int n) {
  return (1u << 4) | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(256 >> 4) << 24);
}
__device__ __forceinline__ void tc_mma_f16_elect(uint32_t d, uint32_t a, uint64_t bdesc,
                                                 uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
// One F16x3 K-chunk, issued by one elected lane of the converged MMA warp in a
// single block: D += A_hi B_hi + A_lo B_hi + A_hi B_lo, then the commits (B
// stage always; A stage on its last use; accumulator when the tile is done).
// One elect and one operand hand-off to the uniform datapath per chunk instead
// of one per instruction (the per-instruction form made the issue loop, not
// the tensor pipe, the limiter: ~770 cycles per 312-cycle chunk).
__device__ __forceinline__ void tc_chunk_f16(uint32_t d, uint32_t a, uint32_t alo, uint64_t dh,
                                             uint64_t dl, uint32_t idesc, uint32_t accum,
                                             uint32_t bar_b, uint32_t bar_a, uint32_t bar_acc,
                                             uint32_t flags) {
  asm volatile(
      "{\n"
      ".reg .pred e, p, t, qa, qc;\n"
      ".reg .b32 f;\n"
      "setp.ne.b32 p, %6, 0;\n"
      "setp.eq.b32 t, %6, %6;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "and.b32 f, %10, 1;\n"
      "setp.ne.b32 qa, f, 0;\n"
      "and.b32 f, %10, 2;\n"
      "setp.ne.b32 qc, f, 0;\n"
      "and.pred qa, qa, e;\n"
      "and.pred qc, qc, e;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %3, %5, p;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %3, %5, t;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %4, %5, t;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%7];\n"
      "@qa tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%8];\n"
      "@qc tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%9];\n"
      "}\n" ::"r"(d),
      "r"(a), "r"(alo), "l"(dh), "l"(dl), "r"(idesc), "r"(accum), "r"(bar_b), "r"(bar_a),
      "r"(bar_acc), "r"(flags)
      : "memory");
}
// Lean form of tc_chunk_f16 for the product path (single CTAs): the B
// descriptors arrive as their low words (the high word -- SBO 256 B, version 1,
// SWIZZLE_NONE -- is a constant), the lo tile's descriptor is the hi tile's plus
// a word offset, and the B-stage commit is optional (flags bit 2; resident
// blocks release nothing).  flags: 1 = release the A stage, 2 = accumulator
// complete, 4 = release the B stage.
__device__ __forceinline__ void tc_chunk_f16_lean(uint32_t d, uint32_t a, uint32_t blo,
                                                  uint32_t lo_off, uint32_t idesc, uint32_t accum,
                                                  uint32_t bar_b, uint32_t bar_a, uint32_t bar_acc,
                                                  uint32_t flags) {
  asm volatile(
      "{\n"
      ".reg .pred e, p, t, qa, qc, qb;\n"
      ".reg .b32 f, l2, a2;\n"
      ".reg .b64 dh, dl;\n"
      "setp.ne.b32 p, %5, 0;\n"
      "setp.eq.b32 t, %5, %5;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "and.b32 f, %9, 1;\n"
      "setp.ne.b32 qa, f, 0;\n"
      "and.b32 f, %9, 2;\n"
      "setp.ne.b32 qc, f, 0;\n"
      "and.b32 f, %9, 4;\n"
      "setp.ne.b32 qb, f, 0;\n"
      "and.pred qa, qa, e;\n"
      "and.pred qc, qc, e;\n"
      "and.pred qb, qb, e;\n"
      "add.u32 l2, %2, %3;\n"
      "add.u32 a2, %1, %10;\n"
      "mov.b64 dh, {%2, %11};\n"
      "mov.b64 dl, {l2, %11};\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], dh, %4, p;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], dh, %4, t;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], dl, %4, t;\n"
      "@qb tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%6];\n"
      "@qa tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%7];\n"
      "@qc tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%8];\n"
      "}\n" ::"r"(d),
      "r"(a), "r"(blo), "r"(lo_off), "r"(idesc), "r"(accum), "r"(bar_b), "r"(bar_a), "r"(bar_acc),
      "r"(flags), "r"(static_cast<uint32_t>(KC / 2)), "r"(0x4010u)
      : "memory");
}
// The same for the leader of a CTA pair (cta_group::2, M = 256: 128 rows from
// each CTA's TMEM A stage, B halves from both CTAs' shared memory); commits are
// multicast to the barrier at the same offset in both CTAs.  Resident B only
// (no B-stage release).  flags: 1 = release the A stage, 2 = accumulator done.
__device__ __forceinline__ void tc_chunk_f16_lean_pair(uint32_t d, uint32_t a, uint32_t blo,
                                                       uint32_t lo_off, uint32_t idesc,
                                                       uint32_t accum, uint32_t bar_a,
                                                       uint32_t bar_acc, uint32_t flags) {
  asm volatile(
      "{\n"
      ".reg .pred e, p, t, qa, qc;\n"
      ".reg .b32 f, l2, a2;\n"
      ".reg .b64 dh, dl;\n"
      ".reg .b16 m;\n"
      "mov.b16 m, 3;\n"
      "setp.ne.b32 p, %5, 0;\n"
      "setp.eq.b32 t, %5, %5;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "and.b32 f, %8, 1;\n"
      "setp.ne.b32 qa, f, 0;\n"
      "and.b32 f, %8, 2;\n"
      "setp.ne.b32 qc, f, 0;\n"
      "and.pred qa, qa, e;\n"
      "and.pred qc, qc, e;\n"
      "add.u32 l2, %2, %3;\n"
      "add.u32 a2, %1, %9;\n"
      "mov.b64 dh, {%2, %10};\n"
      "mov.b64 dl, {l2, %10};\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], dh, %4, p;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a2], dh, %4, t;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], dl, %4, t;\n"
      "@qa tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%6], m;\n"
      "@qc tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%7], m;\n"
      "}\n" ::"r"(d),
      "r"(a), "r"(blo), "r"(lo_off), "r"(idesc), "r"(accum), "r"(bar_a), "r"(bar_acc), "r"(flags),
      "r"(static_cast<uint32_t>(KC / 2)), "r"(0x4010u)
      : "memory");
}
// tc_chunk_f16 for B-multicast clusters: the B-stage release is committed to
// the barrier at the same offset in both CTAs of the 2-CTA cluster (the stage
// is refilled, for both, only after both CTAs' MMAs have read it).
__device__ __forceinline__ void tc_chunk_f16_mcb(uint32_t d, uint32_t a, uint32_t alo, uint64_t dh,
                                                 uint64_t dl, uint32_t idesc, uint32_t accum,
                                                 uint32_t bar_b, uint32_t bar_a, uint32_t bar_acc,
                                                 uint32_t flags) {
  asm volatile(
      "{\n"
      ".reg .pred e, p, t, qa, qc;\n"
      ".reg .b32 f;\n"
      ".reg .b16 m;\n"
      "mov.b16 m, 3;\n"
      "setp.ne.b32 p, %6, 0;\n"
      "setp.eq.b32 t, %6, %6;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "and.b32 f, %10, 1;\n"
      "setp.ne.b32 qa, f, 0;\n"
      "and.b32 f, %10, 2;\n"
      "setp.ne.b32 qc, f, 0;\n"
      "and.pred qa, qa, e;\n"
      "and.pred qc, qc, e;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %3, %5, p;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %3, %5, t;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %4, %5, t;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%7], m;\n"
      "@qa tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%8];\n"
      "@qc tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%9];\n"
      "}\n" ::"r"(d),
      "r"(a), "r"(alo), "l"(dh), "l"(dl), "r"(idesc), "r"(accum), "r"(bar_b), "r"(bar_a),
      "r"(bar_acc), "r"(flags)
      : "memory");
}
// {lo16 = rn_f16(x0), hi16 = rn_f16(x1)}: element 2i in the low half
__device__ __forceinline__ uint32_t pack_f16x2(float x0, float x1) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;\n" : "=r"(r) : "f"(x1), "f"(x0));
  return r;
}
__device__ __forceinline__ void unpack_f16x2(uint32_t h, float& x0, float& x1) {
  asm("{\n.reg .f16 a, b;\nmov.b32 {a, b}, %2;\ncvt.f32.f16 %0, a;\ncvt.f32.f16 %1, b;\n}\n"
      : "=f"(x0), "=f"(x1)
      : "r"(h));
}
// Packed fp32 pairs (sm_100 FMUL2 / FADD2): one instruction per two products /
// differences of the adjoint's operand build.
__device__ __forceinline__ void mul_f32x2(float& a0, float& a1, float b0, float b1) {
  asm("{\n.reg .b64 a, b;\nmov.b64 a, {%0, %1};\nmov.b64 b, {%2, %3};\nmul.rn.f32x2 a, a, b;\n"
      "mov.b64 {%0, %1}, a;\n}\n"
      : "+f"(a0), "+f"(a1)
      : "f"(b0), "f"(b1));
}
__device__ __forceinline__ void sub_f32x2(float& a0, float& a1, float b0, float b1) {
  asm("{\n.reg .b64 a, b;\nmov.b64 a, {%0, %1};\nmov.b64 b, {%2, %3};\nsub.rn.f32x2 a, a, b;\n"
      "mov.b64 {%0, %1}, a;\n}\n"
      : "+f"(a0), "+f"(a1)
      : "f"(b0), "f"(b1));
}
// Power-of-2 scale putting values of magnitude <= amax below 2^14 (f16 max 65504).
__device__ __forceinline__ float f16_scale(float amax) {
  if (!(amax > 0.f) || !(amax < 3.0e38f)) return 1.f;
  int ex;
  frexpf(amax, &ex);  // amax < 2^ex
  int e = 14 - ex;
  e = e > 126 ? 126 : e;
  return ldexpf(1.f, e);
}
__device__ __forceinline__ uint32_t f2tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return r;
}

#define R8(i) "r"(v[i]), "r"(v[i + 1]), "r"(v[i + 2]), "r"(v[i + 3]), "r"(v[i + 4]), "r"(v[i + 5]), "r"(v[i + 6]), "r"(v[i + 7])
#define W8(i) "=r"(v[i]), "=r"(v[i + 1]), "=r"(v[i + 2]), "=r"(v[i + 3]), "=r"(v[i + 4]), "=r"(v[i + 5]), "=r"(v[i + 6]), "=r"(v[i + 7])

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
      "%29, %30, %31, %32};\n" ::"r"(taddr),
      R8(0), R8(8), R8(16), R8(24)
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
      "%29, %30, %31}, [%32];\n"
      : W8(0), W8(8), W8(16), W8(24)
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// SWIZZLE_NONE K-major shared-memory matrix descriptor: core matrices of
// 8 rows x 16 B; LBO = 128 B (next 16 B along K), SBO = 256 B (next 8 rows).
__device__ __forceinline__ uint64_t bdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(128 >> 4) << 16;
  d |= static_cast<uint64_t>(256 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version (sm_100)
  return d;                            // base_offset 0, lbo_mode 0, SWIZZLE_NONE
}
// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major, M=128.
__device__ __forceinline__ uint32_t idesc_tf32(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(128 >> 4) << 24);
}
// kind::f16 instruction descriptor: D f32, A/B f16, both K-major, M=128.
__device__ __forceinline__ uint32_t idesc_f16(int n) {
  return (1u << 4) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(128 >> 4) << 24);
}

__device__ __forceinline__ long long clk() { return clock64(); }
struct Dbg {
  unsigned long long* p;
  long long acc[2] = {0, 0};
  __device__ explicit Dbg(unsigned long long* q) : p(q) {}
  __device__ void flush(int s0, int s1) {
    if (p) {
      atomicAdd(p + s0, static_cast<unsigned long long>(acc[0]));
      if (s1 >= 0) atomicAdd(p + s1, static_cast<unsigned long long>(acc[1]));
    }
  }
};

__device__ __forceinline__ int wrapi(int x, int n) {
  int r = x % n;
  return r < 0 ? r + n : r;
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(taddr),
      R8(0)
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};\n" ::"r"(taddr),
      R8(0), R8(8)
      : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}
__device__ __forceinline__ int tile_width(const TcArgs& a, int nt) {
  const int w = a.g.kp - nt * a.wbase;
  return w < a.wbase ? w : a.wbase;
}

// Tile-group MMA schedule.  The A operand of a K-chunk depends only on
// (brick, chunk), so the MMAs of a group of gsz (1 or 2) N-tiles share each
// built A stage: the builders build every chunk once per group instead of once
// per tile.  The two tiles of a group accumulate in acc0/acc1 at the same
// time, so the schedule is skewed to keep the epilogue overlapped: the first
// D chunks go to tile 0 alone (tile 1's accumulator is still being drained by
// the epilogue of the previous group), then tile 1 catches up on them, the body
// alternates (0,c),(1,c), and the last D chunks again go to tile 0 first so
// that its accumulator completes D chunk periods before tile 1's.  A stage of
// chunk c is released after its last use; D <= sa keeps the ring live.
__device__ __forceinline__ void tg_seq(int i, int gsz, int nkc, int D, int& t, int& c) {
  if (gsz == 1) {
    t = 0;
    c = i;
    return;
  }
  if (i < D) {
    t = 0;
    c = i;
    return;
  }
  if (i < 2 * D) {
    t = 1;
    c = i - D;
    return;
  }
  int j = i - 2 * D;
  const int nb = 2 * (nkc - 2 * D);
  if (j < nb) {
    t = j & 1;
    c = D + (j >> 1);
    return;
  }
  j -= nb;
  t = j < D ? 0 : 1;
  c = nkc - D + (j < D ? j : j - D);
}

// ---------------------------------------------------------------------------
// The kernel (FWD = forward implicit GEMM, !FWD = adjoint)
//   warps [0, 8)            builders (two per TMEM lane quadrant, 16 K each)
//   warps [8, 8 + NEPI)     epilogue (NEPI = 8 forward, 4 adjoint)
//   warp  8 + NEPI          MMA issuer
//   warp  9 + NEPI          B loader
// ---------------------------------------------------------------------------
template <bool FWD, bool F16, bool PAIR>
__global__ void __launch_bounds__(608 + 32 * NPREP, 1)
icnnm_tc_kernel(const __grid_constant__ TcArgs a) {
  constexpr int ASC = F16 ? KC : 2 * KC;  // TMEM columns per A stage
  constexpr int ALO = ASC / 2;            // column offset of the lo half
  constexpr int NB = 8;                  // builder warps
  constexpr int NEPI = 8;                // epilogue warps (adjoint: 4 * a.ehalf active)
  constexpr int WMMA = NB + NEPI;        // MMA warp
  constexpr int WLOAD = NB + NEPI + 1;   // B loader warp; W loader warp after it
  constexpr int WPREP = WLOAD + 2;       // forward: NPREP halo-preparation warps
  // B stage stride: the widest tile's hi/lo bytes when the host packs the
  // ring tightly (a.bstride, F16x3 single CTAs), else the fixed stage size
  const int BSTG = (F16 && !PAIR && a.bstride > 0)
                       ? a.bstride
                       : (F16 ? (PAIR ? B_STAGE_F16 / 2 : B_STAGE_F16) : B_STAGE_BYTES);
  const Geo& g = a.g;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* p = smem;
  const int sbn = a.sb, wsn = a.ws, san = a.sa;
  const uint32_t a_col0 = 2u * static_cast<uint32_t>(a.accw);
  // resident B blocks (a.bres) first, then the stage ring (absent when every
  // block of the CTA's role is resident)
  float* Bst = reinterpret_cast<float*>(p);
  uint8_t* Bring = p + (a.bres ? a.bres_bytes : 0);
  p = Bring + ((a.bres && !a.bmix) ? 0 : sbn * BSTG);
  float* Wst = reinterpret_cast<float*>(p);   // adjoint: W-chunk ring; forward: W-group ring
  p += wsn * (FWD ? WO_STAGE_BYTES : W_STAGE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(p);
  uint64_t* A_full = bars;
  uint64_t* A_empty = bars + SA;
  uint64_t* B_full = bars + 2 * SA;
  uint64_t* B_empty = bars + 2 * SA + SB;
  uint64_t* ACC_full = bars + 2 * SA + 2 * SB;
  uint64_t* ACC_empty = ACC_full + 2;
  uint64_t* W_full = ACC_empty + 2;
  uint64_t* W_empty = W_full + WS;
  uint64_t* SC_full = W_empty + WS;   // F16x3 forward: per-brick scale slots
  float* sc_ring = reinterpret_cast<float*>(SC_full + NSC);
  float* wmax = sc_ring + NSC;        // 2 x 8 halo-warp maxima
  uint64_t* HALO_full = reinterpret_cast<uint64_t*>(wmax + 16);  // forward: halo buffer ready
  uint64_t* HALO_empty = HALO_full + NHB_MAX;                     // forward: halo buffer read
  const int nhb = a.nhb >= 2 ? a.nhb : 2;                         // forward: halo buffers
  p += BAR_BYTES;  // 2*SA + 2*SB + 4 + 2*WS + NSC mbarriers, NSC scales, 16 maxima
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p);
  p += 16;
  // (ktp words kept in the carve-up: smem_bytes() is shared with the host)
  p += ((g.ktp * 4 + 15) / 16) * 16;
  float* cs = reinterpret_cast<float*>(p);
  p += ((g.kp * 4 + 15) / 16) * 16;
  const int nob = g.HH * g.HW * g.HT;
  const int nobp = ((nob + 3) / 4) * 4;
  // FWD: halo[nhb] (nhb x nobp) | nrm (kp doubles)
  // ADJ: 4 * ehalf output bricks (nobp + 32 each)
  float* halo = reinterpret_cast<float*>(p);
  double* nrm = reinterpret_cast<double*>(halo + (FWD ? nhb : 2) * nobp);
  float* ob = reinterpret_cast<float*>(p);

  const int tid = threadIdx.x;
  // adjoint epilogue: active 4-warp halves, each with its own 4 output bricks
  // (two halves take alternate 32-column blocks of every accumulator)
  const int ehalf = FWD ? 2 : (a.ehalf > 1 ? 2 : 1);
  // B multicast: a 2-CTA cluster of independent CTAs (own bricks, own M = 128
  // MMAs) consuming one B stream; each CTA loads half of every B stage and
  // multicasts it to both, so the L2 -> SM traffic of the basis halves
  const bool MCB = !PAIR && F16 && a.mcb != 0;
  const bool CL2 = PAIR || MCB;  // launched as 2-CTA clusters
  const int nepi_act = 4 * ehalf;
  // CTA pairs / B multicast: barriers completed by the peer (remote arrives,
  // multicast commits) are waited on with the default CTA-scope wait, as
  // CUTLASS's 2-SM pipelines do (the .acquire.cluster form adds a CCTL.IVALL --
  // an L1 invalidation -- after every wait: 25% of the pair adjoint's stall
  // samples); skip bit 64 restores it (A/B)
  auto pwait = [&](uint64_t* b, uint32_t ph) {
    if (TC_SKIP(a) & 64)
      mbar_wait_cluster(b, ph);
    else
      mbar_wait(b, ph);
  };
  // warp index through a shuffle: provably warp-uniform, so role branches are
  // uniform and the MMA issuer's counters can live in uniform registers
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;

  // consumer / producer hand-over arrive of a whole warp: lane 0 after a warp
  // sync (a.warr), or every lane
  const bool warr = TC_WARR(a);
  auto warp_arrive = [&](uint64_t* b) {
    if (warr) {
      __syncwarp();
      if (lane == 0) mbar_arrive(b);
    } else {
      mbar_arrive(b);
    }
  };
  auto warp_arrive2 = [&](uint64_t* b0, uint64_t* b1) {  // b1 may be null
    if (warr) {
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(b0);
        if (b1) mbar_arrive(b1);
      }
    } else {
      mbar_arrive(b0);
      if (b1) mbar_arrive(b1);
    }
  };
  if (warp == WMMA) {
    if (PAIR) {  // both CTAs' warp WMMA: 512 columns in each CTA of the pair
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
          smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
          smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
  }
  if (tid == 0) {
    // arrivals per barrier phase: one per warp (a.warr: the warp's lane 0 after
    // __syncwarp; 128 single-lane arrives on one mbarrier serialise in the
    // shared-memory atomic unit) or one per thread
    const int per = TC_WARR(a) ? 1 : 32;
    const int nbuild = ((a.bsplit && !F16) ? NB : NB / 2) * per;  // builder arrivals / chunk
    // PAIR: the leader's A_full / ACC_empty count one arrival per warp of both
    // CTAs; its B_full the local expect_tx plus the peer's relayed arrival
    for (int i = 0; i < SA; ++i) {
      mbar_init(A_full + i, PAIR ? 2 * (NB / 2) : nbuild);
      mbar_init(A_empty + i, 1);
    }
    for (int i = 0; i < SB; ++i) {
      mbar_init(B_full + i, (PAIR && !a.tma_pair && !a.bres && (blockIdx.x & 1u) == 0) ? 2 : 1);
      mbar_init(B_empty + i, MCB ? 2 : 1);  // MCB: released by both CTAs' MMAs
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(ACC_full + i, 1);
      mbar_init(ACC_empty + i, PAIR ? 2 * nepi_act : nepi_act * per);
    }
    for (int i = 0; i < WS; ++i) {
      mbar_init(W_full + i, 1);
      mbar_init(W_empty + i, FWD ? 4 * per : nbuild);  // forward: the half's 4 epilogue warps
    }
    for (int i = 0; i < NSC; ++i) mbar_init(SC_full + i, 1);
    for (int i = 0; i < NHB_MAX; ++i) {
      mbar_init(HALO_full + i, 1);             // the prep warps' leader, after their barrier
      mbar_init(HALO_empty + i, NB * per);     // every builder warp / thread, after the brick
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // (tap offsets: a.tapn, negative byte offsets filled by the host -- read
  // through the constant bank with warp-uniform indices, so gathers and
  // scatters address shared memory as [thread base + uniform offset])
  // everything above reads only the launch parameters: with PDL it overlaps
  // the predecessor kernel; from here on the predecessor's writes are read
  pdl_wait();
  pdl_trigger();
  // iteration state: a finished solve's replays are no-ops (uniform over the grid)
  float rr = 0.f;
  {
    bool quit = false;
    if (a.mode == 1) {
      if (!a.st->active)
        quit = true;
      else if (FWD && a.st->it >= a.st->max_iters - 1)
        quit = true;
      else
        rr = static_cast<float>(a.st->r);
    }
    if (a.mode == 2 && !a.st->active) quit = true;  // forward on L_{t+1}: exact residual only
    if (quit) {
      tc_fence_before();
      if (CL2)
        cluster_sync_all();
      else
        __syncthreads();
      tc_fence_after();
      if (warp == WMMA) {
        if (PAIR)
          asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(*tmem_slot));
        else
          asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(*tmem_slot));
      }
      return;
    }
  }
  // cs[j]: forward mode 1: r c_j (the W_old weight); mode 2: c_j; adjoint:
  // c_j (mode 1) or 1, times the F16x3 operand scale
  const float fscale_adj =
      (F16 && !FWD) ? f16_scale(a.mode >= 1 ? static_cast<float>(a.st->adj_amax) : a.amax) : 1.f;
  for (int j = tid; j < g.kp; j += blockDim.x) {
    float c = 1.f;
    if (a.mode >= 1) c = a.cvec[j];
    if (FWD && a.mode == 1) c *= rr;
    if (!FWD) c *= fscale_adj;
    cs[j] = (j < g.k) ? c : 0.f;
  }
  if (FWD) {
    for (int j = tid; j < g.kp; j += blockDim.x) nrm[j] = 0.0;
  } else {
    for (int e = tid; e < nepi_act * (nobp + 32); e += blockDim.x) ob[e] = 0.f;
  }
  tc_fence_before();
  if (CL2)
    cluster_sync_all();  // the peer's barriers are initialised before any remote arrive / commit
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  const int nbr = static_cast<int>(a.nbricks);
  const int ntn = a.ntn;
  const int nkc = a.nkc;
  // Split mode (a.nsplit > 1, single CTAs only): CTA role = blockIdx % nsplit
  // owns a range of the N-tiles of every brick -- forward: its columns j of
  // W; adjoint: its taps s, whose col2im partial output brick is summed with
  // the other roles' by the flush -- so that the role's B tiles fit in shared
  // memory and stay resident (a.bres: loaded once per launch instead of once
  // per brick).  Each role builds the brick's A operand itself (the adjoint's
  // builders idle ~80% of the time).  The K-chunk range
  // [kcb, kce) is the whole basis (kept general for the loops below).
  const int nsp = a.nsplit > 1 ? a.nsplit : 1;
  const int role = nsp > 1 ? static_cast<int>(blockIdx.x % static_cast<unsigned>(nsp)) : 0;
  const int ntb = nsp > 1 ? role * ntn / nsp : 0;
  const int nte = nsp > 1 ? (role + 1) * ntn / nsp : ntn;
  const int kcb = 0;
  const int kce = nkc;
  const int nkr = kce - kcb;                   // K-chunks per tile in this CTA
  const int grp = a.grp > 1 ? 2 : 1;          // N-tiles sharing each A chunk
  const int ngrp = (nte - ntb + grp - 1) / grp;
  // resident B: SMEM offset of tile nt's chunk kc (tiles of the role's range,
  // chunks of its K range, a.bres_stride bytes each)
  auto bres_off = [&](int nt, int kc) {
    return static_cast<uint32_t>(((nt - ntb) * nkr + (kc - kcb)) * a.bres_stride);
  };
  // mixed residency (a.bmix): only the role's first a.nresblk (tile, chunk)
  // blocks are resident, the others stream through the ring
  auto is_res = [&](int nt, int kc) {
    return a.bres && (!a.bmix || (nt - ntb) * nkr + (kc - kcb) < a.nresblk);
  };
  uint64_t* const BRES_full = B_full + (SB - 1);   // resident fill (one phase per launch)
  int skew = a.skew < nkr / 2 ? a.skew : nkr / 2;
  skew = skew < san ? skew : san;
  skew = skew < 0 ? 0 : skew;
  // Bricks by cluster slot: CTA `crank` of a cs-CTA cluster takes brick
  // cs*s + crank of slot s, so both CTAs of a pair walk the same number of
  // slots (they consume one multicast B stream in lockstep); a pair's odd
  // tail brick is a dummy (brick nbr-1 re-read, nothing written).
  const int ncta = CL2 ? 2 : 1;
  const int crank = ncta > 1 ? static_cast<int>(blockIdx.x & 1u) : 0;
  const int sfirst = static_cast<int>(blockIdx.x) / (ncta * nsp);
  const int sstep = static_cast<int>(gridDim.x) / (ncta * nsp);
  const int nslot = (nbr + ncta - 1) / ncta;
  auto brick_of = [&](int sl) {
    const int bb = sl * ncta + crank;
    return bb < nbr ? bb : nbr - 1;
  };
  auto real_slot = [&](int sl) { return sl * ncta + crank < nbr; };
  // Brick coordinates (t fastest) of this CTA's slots, advanced by sstep in
  // mixed radix for single CTAs (three integer divisions per brick and thread
  // otherwise: 3-4% of either kernel's instructions at k = 245); clusters
  // (clamped dummy tail brick) divide.
  struct BrickIt {
    int bt, bw, bh;
  };
  const int bs_t = sstep % g.nbt, bs_w = (sstep / g.nbt) % g.nbw, bs_h = sstep / (g.nbt * g.nbw);
  auto brick_at = [&](int b) {
    BrickIt x;
    x.bt = b % g.nbt;
    const int q = b / g.nbt;
    x.bw = q % g.nbw;
    x.bh = q / g.nbw;
    return x;
  };
  auto brick_next = [&](BrickIt& x, int sl_next) {
    if (ncta > 1) {
      x = brick_at(brick_of(sl_next));
      return;
    }
    x.bt += bs_t;
    int cy = x.bt >= g.nbt ? 1 : 0;
    x.bt -= cy * g.nbt;
    x.bw += bs_w + cy;
    cy = x.bw >= g.nbw ? 1 : 0;
    x.bw -= cy * g.nbw;
    x.bh += bs_h + cy;
  };

  if (warp < NB && !(TC_SKIP(a) & 8)) {
    // ===================== builders =====================
    const int quad = warp & 3, half = warp >> 2;
    const int row = 32 * quad + lane;
    const int bt_tid = tid;                       // 0..255
    const int vt = row % g.bt;
    const int vw = g.vmap ? row / (g.bt * g.bh) : (row / g.bt) % g.bw;
    const int vh = g.vmap ? (row / g.bt) % g.bh : row / (g.bt * g.bw);
    const int hidx = ((vh + g.kh - 1) * g.HW + (vw + g.kw - 1)) * g.HT + (vt + g.kt - 1);
    const uint32_t lane_base = static_cast<uint32_t>(32 * quad) << 16;
    uint32_t cnt = 0;
    Dbg dbg(lane == 0 ? TC_DBG(a) : nullptr);
    // F16x3 operand scale: forward per brick (the halo is prescaled in place);
    // adjoint: folded into cs
    // (the held chunk c and the next owned chunk c+2 must use different A and
    // W stages: sa >= 3 always; the adjoint's W ring needs 4)
    const bool pair = TC_BPAIR(a) && !PAIR && (F16 || !a.bsplit) && san >= 3 && (FWD || wsn >= 4);
    const uint32_t lead_afull = PAIR ? mapa_u32(smem_u32(A_full), 0) : 0u;
    int pend_sa = -1, pend_wsi = 0;
    int iter = 0;
    int st_sa = 0, st_ws = 0;
    uint32_t st_ph = 0, st_wph = 0;
    // A / W stage (index, parity) advanced by n <= 2 chunks (rings of >= 2 stages)
    auto adv_stage = [&](int n) {
      st_sa += n;
      if (st_sa >= san) {
        st_sa -= san;
        st_ph ^= 1u;
      }
      st_ws += n;
      if (st_ws >= wsn) {
        st_ws -= wsn;
        st_wph ^= 1u;
      }
    };
    // bsplit = 0: group `half` owns the chunks with cnt % 2 == half and builds
    // all KC columns, so each warp has two chunk periods of MMA time to cover
    // its TMEM-store round trip; the loop visits only the owned chunks
    const int nchunk = ngrp * nkr;
    const int cstep = (F16 || !a.bsplit) ? 2 : 1;

    long long prep = 0;
    int f = cstep == 2 ? half : 0;  // my next chunk, relative to the current brick
    adv_stage(f);
    int kc = kcb + f;
    if (kc >= kce) kc -= nkr;
    for (int sl = sfirst; sl < nslot; sl += sstep, ++iter) {
      const int hbuf = iter % nhb;
      float* hcur = halo + hbuf * nobp;
      // this thread's halo element, as a byte pointer (tap offsets are in bytes)
      const char* const hb = reinterpret_cast<const char*>(hcur + hidx);
      const long long tp0 = dbg.p ? clk() : 0;
      // forward: this brick's halo (prescaled / pre-split for F16x3) is
      // prepared by the prep warps while the previous brick is built
      if (FWD) mbar_wait(HALO_full + hbuf, static_cast<uint32_t>(iter / nhb) & 1u);
      if (dbg.p) prep += clk() - tp0;
      {
        // (this group's chunks are every cstep-th of the global chunk sequence:
        // its stage iterator, kc and brick-local index f simply advance by
        // cstep, across bricks too)
        for (; f < nchunk; f += cstep) {
          // A / W stage (index, parity) of this chunk, advanced incrementally
          // (cnt % san and cnt / san were a 32-bit division per chunk)
          const int sa = st_sa;
          const uint32_t ph = st_ph;
          const int wsi = st_ws;
          const uint32_t wph = st_wph;
          long long t0c = dbg.p ? clk() : 0;
          if (PAIR)
            pwait(A_empty + sa, ph ^ 1);  // released by the leader's MMAs
          else
            mbar_wait(A_empty + sa, ph ^ 1);
          if (!FWD) mbar_wait(W_full + wsi, wph);
          tc_fence_after();
          long long t1c = dbg.p ? clk() : 0;
          if (!(TC_SKIP(a) & 1)) {
            const uint32_t col = a_col0 + sa * ASC;
            // the chunk's 16 tap offsets (forward) or c_j factors (adjoint), 4 vector loads
            int tq[KC];
            float cq[KC];
#pragma unroll
            for (int v4 = 0; v4 < KC / 4; ++v4) {
              if (FWD) {
                const int4 t4 = reinterpret_cast<const int4*>(a.tapn + kc * KC)[v4];
                tq[4 * v4] = t4.x; tq[4 * v4 + 1] = t4.y; tq[4 * v4 + 2] = t4.z; tq[4 * v4 + 3] = t4.w;
              } else {
                const float4 c4 = reinterpret_cast<const float4*>(cs + kc * KC)[v4];
                cq[4 * v4] = c4.x; cq[4 * v4 + 1] = c4.y; cq[4 * v4 + 2] = c4.z; cq[4 * v4 + 3] = c4.w;
              }
            }
            if (F16 && FWD) {
              // pre-split halo words {hi, lo}: hi pair = low halves, lo pair = high halves
              uint32_t hi[8], lo[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const uint32_t w0 = *reinterpret_cast<const uint32_t*>(hb + tq[2 * i]);
                const uint32_t w1 = *reinterpret_cast<const uint32_t*>(hb + tq[2 * i + 1]);
                hi[i] = __byte_perm(w0, w1, 0x5410);
                lo[i] = __byte_perm(w0, w1, 0x7632);
              }
              tmem_st8(tbase + lane_base + col, hi);
              tmem_st8(tbase + lane_base + col + ALO, lo);
            } else if (F16) {
              // 16 K values -> 8 f16x2 words hi | 8 words lo (element 2i in the low half)
              uint32_t hi[8], lo[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                float x[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                  x[u] = FWD ? *reinterpret_cast<const float*>(hb + tq[2 * i + u])
                             : Wst[wsi * (W_STAGE_BYTES / 4) + (2 * i + u) * 128 + row];
                }
                if (!FWD) mul_f32x2(x[0], x[1], cq[2 * i], cq[2 * i + 1]);
                hi[i] = pack_f16x2(x[0], x[1]);
                float h0, h1;
                unpack_f16x2(hi[i], h0, h1);
                sub_f32x2(x[0], x[1], h0, h1);
                lo[i] = pack_f16x2(x[0], x[1]);
              }
              tmem_st8(tbase + lane_base + col, hi);
              tmem_st8(tbase + lane_base + col + ALO, lo);
            } else if (a.bsplit) {
              uint32_t hi[8], lo[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int q = kc * KC + 8 * half + i;
                const float x = FWD ? *reinterpret_cast<const float*>(hb + a.tapn[q])
                                    : Wst[wsi * (W_STAGE_BYTES / 4) + (8 * half + i) * 128 + row] * cs[q];
                const uint32_t h = f2tf32(x);
                hi[i] = h;
                lo[i] = __float_as_uint(x - __uint_as_float(h));
              }
              tmem_st8(tbase + lane_base + col + 8 * half, hi);
              tmem_st8(tbase + lane_base + col + 8 * half + KC, lo);
            } else {
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {  // two 8-column halves, one wait::st
                uint32_t hi[8], lo[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  const float x = FWD ? *reinterpret_cast<const float*>(hb + tq[8 * hh + i])
                                      : Wst[wsi * (W_STAGE_BYTES / 4) + (8 * hh + i) * 128 + row] * cq[8 * hh + i];
                  const uint32_t h = f2tf32(x);
                  hi[i] = h;
                  lo[i] = __float_as_uint(x - __uint_as_float(h));
                }
                tmem_st8(tbase + lane_base + col + 8 * hh, hi);
                tmem_st8(tbase + lane_base + col + 8 * hh + KC, lo);
              }
            }
            if (!pair) tmem_wait_st();
          }
          if (pair) {
            // pairing: hand over the previous owned chunk together with this
            // one after a single wait::st (its store latency overlapped this
            // chunk's gathers); the last chunk of a brick is flushed below
            if (pend_sa >= 0) {
              if (!(TC_SKIP(a) & 1)) tmem_wait_st();
              tc_fence_before();
              warp_arrive2(A_full + pend_sa, FWD ? nullptr : W_empty + pend_wsi);
              warp_arrive2(A_full + sa, FWD ? nullptr : W_empty + wsi);
              pend_sa = -1;
            } else {
              pend_sa = sa;
              pend_wsi = wsi;
            }
          } else if (PAIR) {
            // one arrival per warp on the leader's A_full (after the warp's wait::st)
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(lead_afull + 8u * static_cast<uint32_t>(sa));
            if (!FWD) warp_arrive(W_empty + wsi);
          } else {
            tc_fence_before();
            if constexpr (FWD) {
              warp_arrive(A_full + sa);
            } else {  // one warp sync, both arrivals from lane 0
              if (warr) {
                __syncwarp();
                if (lane == 0) {
                  mbar_arrive(A_full + sa);
                  mbar_arrive(W_empty + wsi);
                }
              } else {
                mbar_arrive(A_full + sa);
                mbar_arrive(W_empty + wsi);
              }
            }
          }
          if (dbg.p) {
            long long t2c = clk();
            dbg.acc[0] += t1c - t0c;
            dbg.acc[1] += t2c - t1c;
          }
          adv_stage(cstep);
          kc += cstep;
          if (kc >= kce) kc -= nkr;
        }
      }
      cnt += static_cast<uint32_t>(nchunk);
      f -= nchunk;
      if (pair && pend_sa >= 0) {  // flush the brick's last owned chunk
        if (!(TC_SKIP(a) & 1)) tmem_wait_st();
        tc_fence_before();
        warp_arrive2(A_full + pend_sa, FWD ? nullptr : W_empty + pend_wsi);
        pend_sa = -1;
      }
      if (FWD) warp_arrive(HALO_empty + hbuf);  // this warp's reads of the halo are done
    }
    dbg.flush(DBG_BUILD_WAIT, DBG_BUILD_WORK);
    if (dbg.p) atomicAdd(dbg.p + DBG_BUILD_PREP, static_cast<unsigned long long>(prep));
  } else if (FWD && warp >= WPREP && warp < WPREP + NPREP) {
    // ===================== halo preparation (forward) =====================
    // Brick i's halo box (periodic L~ gather) into halo[i % nhb], its max|x|,
    // the F16x3 operand scale (published to the epilogue's scale ring), and
    // the in-place prescale / hi-lo pre-split -- off the builders' critical
    // path (the all-builder barrier phase this replaces took ~25-33% of the
    // builders' time at brick transitions, profiles/README_r2.md)
    const int pt = tid - WPREP * 32;  // 0 .. 32*NPREP-1
    const int pw = warp - WPREP;
    // software pipeline over nhb halo buffers: the gather of brick i is issued
    // (cp.async group i) LAG bricks before its scale / split pass, so its
    // L2/HBM latency overlaps the preparation of the bricks before it
    const int LAG = nhb - 2 >= 1 ? (nhb - 2 > 2 ? 2 : nhb - 2) : 0;
    // halo element e = (aa*HW + bb)*HT + c of this thread: decomposed once,
    // then advanced by NPREP*32 in mixed radix (no divisions per element)
    // Copies are vw = 4, 2 or 1 consecutive frames wide (16 / 8 / 4 bytes): a
    // box row's frames are contiguous in L~ between wraps, and groups of vw
    // stay aligned and never straddle a wrap when vw divides T, bt, kt - 1
    // (then also HT = bt + kt - 1 and every brick's first halo frame)
    constexpr int PSTEP = NPREP * 32;
    const int vw = ((g.T | g.bt | (g.kt - 1)) & 3) == 0 ? 4 : (((g.T | g.bt | (g.kt - 1)) & 1) == 0 ? 2 : 1);
    const int nc = g.HT / vw, ngrp_h = nob / vw;   // groups per box row / per box
    const int dc = PSTEP % nc, dbb = (PSTEP / nc) % g.HW, daa = PSTEP / (nc * g.HW);
    const int c0 = pt % nc, bb0 = (pt / nc) % g.HW, aa0 = pt / (nc * g.HW);
    // one conditional wrap suffices unless a dimension is smaller than its halo
    auto wrap1 = [](int x, int n) {
      x = x < 0 ? x + n : x;
      x = x >= n ? x - n : x;
      return (static_cast<unsigned>(x) < static_cast<unsigned>(n)) ? x : wrapi(x, n);
    };
    BrickIt pk = brick_at(brick_of(sfirst < nslot ? sfirst : 0));
    auto issue = [&](int i, int sl) {
      const int buf = i % nhb;
      float* hdst = halo + buf * nobp;
      // (timing experiments without builders: nobody releases the buffers)
      if (!(TC_SKIP(a) & 8)) mbar_wait(HALO_empty + buf, (static_cast<uint32_t>(i / nhb) & 1u) ^ 1u);
      // (issue() is called for this CTA's slots in order: pk is slot sl's brick)
      const int hb0 = pk.bh * g.bh - (g.kh - 1) + g.hoff, wb0 = pk.bw * g.bw - (g.kw - 1),
                tb0 = pk.bt * g.bt - (g.kt - 1);
      brick_next(pk, sl + sstep);
      int c = c0, bb = bb0, aa = aa0;
      for (int e = pt; e < ngrp_h; e += PSTEP) {
        int hs = hb0 + aa;
        hs = g.wrapH ? wrap1(hs, g.Hsrc) : (hs < 0 ? 0 : (hs >= g.Hsrc ? g.Hsrc - 1 : hs));
        const int ws = wrap1(wb0 + bb, g.W);
        const int ts = wrap1(tb0 + c * vw, g.T);
        const float* src = a.src + (static_cast<size_t>(hs) * g.W + ws) * g.T + ts;
        if (vw == 4)
          cp_async16(hdst + 4 * e, src);
        else if (vw == 2)
          cp_async8(hdst + 2 * e, src);
        else
          cp_async4(hdst + e, src);
        c += dc;
        int cy = c >= nc ? 1 : 0;
        c -= cy * nc;
        bb += dbb + cy;
        cy = bb >= g.HW ? 1 : 0;
        bb -= cy * g.HW;
        aa += daa + cy;
      }
      cp_async_commit();
    };
    auto finish = [&](int i, int pending) {
      const int buf = i % nhb;
      float* hcur = halo + buf * nobp;
      if (pending >= 2)
        asm volatile("cp.async.wait_group 2;\n" ::: "memory");
      else if (pending == 1)
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
      else
        cp_async_wait_all();
      named_sync(5, NPREP * 32);  // brick i's halo landed (every prep thread's copies)
      if (F16) {
        float mx = 0.f;
        for (int e = pt; e < nob; e += NPREP * 32) mx = fmaxf(mx, fabsf(hcur[e]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0) wmax[(i & 1) * 8 + pw] = mx;
        named_sync(5, NPREP * 32);
        float bm = 0.f;
#pragma unroll
        for (int w = 0; w < NPREP; ++w) bm = fmaxf(bm, wmax[(i & 1) * 8 + w]);
        const float fscale = f16_scale(bm);
        // prescale and pre-split in place: word = rn_f16(x) | rn_f16(x - hi) << 16,
        // so each chunk's build is gathers + byte permutes (same bits as
        // splitting per chunk, once per halo element instead of once per tap)
        uint32_t* hw = reinterpret_cast<uint32_t*>(hcur);
        for (int e = pt; e < nob; e += NPREP * 32) {
          const float x = hcur[e] * fscale;
          const float xh = __half2float(__float2half_rn(x));
          hw[e] = pack_f16x2(x, x - xh);
        }
        if (pt == 0) {  // the epilogue unscales this brick by 2^-(eA + eB)
          sc_ring[i % NSC] = a.bunscale / fscale;
          mbar_arrive(SC_full + i % NSC);
        }
        named_sync(5, NPREP * 32);  // halo scaled
      }
      if (pt == 0) mbar_arrive(HALO_full + buf);
    };
    const int nmine = sfirst < nslot ? (nslot - sfirst + sstep - 1) / sstep : 0;
    for (int i = 0; i < nmine + LAG; ++i) {
      if (i < nmine) issue(i, sfirst + i * sstep);
      if (i >= LAG) {
        const int j = i - LAG;
        const int pend = (i < nmine ? LAG : LAG - (i - nmine) - 1);
        finish(j, pend < 0 ? 0 : pend);
      }
    }
  } else if (warp < NB) {
  } else if (warp < NB + nepi_act && !(TC_SKIP(a) & 32)) {
    // ===================== epilogue =====================
    const int ew = warp - NB;
    const int quad = ew & 3, half = ew >> 2;     // half in {0} (adjoint) or {0,1} (forward)
    const int row = 32 * quad + lane;
    const uint32_t lane_base = static_cast<uint32_t>(32 * quad) << 16;
    const int vt = row % g.bt;
    const int vw = g.vmap ? row / (g.bt * g.bh) : (row / g.bt) % g.bw;
    const int vh = g.vmap ? (row / g.bt) % g.bh : row / (g.bt * g.bw);
    const int hidx = ((vh + g.kh - 1) * g.HW + (vw + g.kw - 1)) * g.HT + (vt + g.kt - 1);
    const int obs = nobp + 32;             // output-brick stride (+32 scratch)
    float* myob = ob + (FWD ? quad : ew) * obs;  // adjoint: one output brick per warp
    const int NHALF = ehalf;
    uint32_t gbase = 0;  // forward: W-group ring slot of the current tile's first group
    int ep_ws = half;    // forward: this half's next W-group ring slot and its parity
    uint32_t ep_wph = 0;
    float gacc = 0.f;  // mode 2: this thread's share of ||(1-c)W - A(L)K||^2
    uint32_t tcount = 0;
    Dbg dbg(lane == 0 ? TC_DBG(a) : nullptr);
    float us_adj = 1.f;  // F16x3 adjoint: 2^-(eA + eB)
    if (F16 && !FWD)
      us_adj = a.bunscale / f16_scale(a.mode >= 1 ? static_cast<float>(a.st->adj_amax) : a.amax);
    uint32_t biter = 0;
    // adjoint flush: this thread's first output-box element and its step
    const int FSTEP = nepi_act * 32, fe0 = ew * 32 + lane;
    const int fl_c0 = fe0 % g.HT, fl_bb0 = (fe0 / g.HT) % g.HW, fl_aa0 = fe0 / (g.HT * g.HW);
    const int fl_dc = FSTEP % g.HT, fl_dbb = (FSTEP / g.HT) % g.HW, fl_daa = FSTEP / (g.HT * g.HW);
    // the same in groups of 4 frames (HT % 4 == 0): fv_nc groups per box row
    const int fv_nc = g.HT >> 2 > 0 ? g.HT >> 2 : 1;
    const int fv_c0 = fe0 % fv_nc, fv_bb0 = (fe0 / fv_nc) % g.HW, fv_aa0 = fe0 / (fv_nc * g.HW);
    const int fv_dc = FSTEP % fv_nc, fv_dbb = (FSTEP / fv_nc) % g.HW, fv_daa = FSTEP / (fv_nc * g.HW);
    // one conditional wrap suffices unless a dimension is smaller than its halo
    auto wrap1 = [](int x, int n) {
      x = x < 0 ? x + n : x;
      x = x >= n ? x - n : x;
      return (static_cast<unsigned>(x) < static_cast<unsigned>(n)) ? x : wrapi(x, n);
    };
    // deterministic adjoint flush: the {hi, lo} grids of this launch
    const AdjGrid qg = adj_grid((!FWD && a.adjq != nullptr) ? a.st->adj_amax : 0.0, g.k);
    const uint32_t lead_accempty = PAIR ? mapa_u32(smem_u32(ACC_empty), 0) : 0u;
    BrickIt bk = brick_at(brick_of(sfirst < nslot ? sfirst : 0));
    for (int sl = sfirst; sl < nslot; sl += sstep, ++biter, brick_next(bk, sl)) {
      const int b = brick_of(sl);
      const bool breal = real_slot(sl);  // false: the pair's dummy tail brick, nothing written
      const int h0 = bk.bh * g.bh, w0 = bk.bw * g.bw, t0 = bk.bt * g.bt;
      const bool valid = breal && (h0 + vh < g.H) && (w0 + vw < g.W) && (t0 + vt < g.T);
      const bool bfull = (h0 + g.bh <= g.H) && (w0 + g.bw <= g.W) && (t0 + g.bt <= g.T);
      float us = us_adj;
      if (F16 && FWD) {  // this brick's scale, published by the builders
        mbar_wait(SC_full + biter % NSC, (biter / NSC) & 1);
        us = sc_ring[biter % NSC];
      }
      for (int nt = ntb; nt < nte; ++nt, ++tcount) {
        const int acc = tcount & 1;
        const uint32_t ph = (tcount >> 1) & 1;
        const int wn = tile_width(a, nt);
        long long t0c = dbg.p ? clk() : 0;
        mbar_wait(ACC_full + acc, ph);
        tc_fence_after();
        long long t1c = dbg.p ? clk() : 0;
        if (FWD) {
          // forward: the W group (32 columns x 128 rows) is staged in SMEM by
          // the W loader (mode 1/2: W_old), updated in place, reduced for the
          // column norms and written back with one bulk store
          const int ng = (wn + 31) / 32, ngp = ng + (ng & 1);  // even: one half per stage
          for (int gq = half; gq < ngp; gq += 2) {
            // this half's ring slot: two groups further every visit (even ring)
            const int wsl = ep_ws;
            mbar_wait(W_full + wsl, ep_wph);
            ep_ws += 2;
            if (ep_ws >= wsn) {
              ep_ws -= wsn;
              ep_wph ^= 1u;
            }
            if (gq < ng && !(TC_SKIP(a) & 2)) {
              const int c0 = 32 * gq;
              const int ncol = (wn - c0) < 32 ? (wn - c0) : 32;
              const int j0 = nt * a.wbase + c0;
              float* st = Wst + wsl * (WO_STAGE_BYTES / 4);
              uint32_t u[32];
              tmem_ld32(tbase + lane_base + acc * a.accw + c0, u);
              tmem_wait_ld();
              auto accv = [&](int i) {
                return F16 ? __uint_as_float(u[i]) * us : __uint_as_float(u[i]);
              };
              if (a.mode == 2) {
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                  const float gap = (1.f - cs[j0 + i]) * st[i * 128 + row] - accv(i);
                  gacc = (i < ncol && valid) ? fmaf(gap, gap, gacc) : gacc;
                }
              } else {
                if (ncol == 32 && bfull) {
                  const float4* c4 = reinterpret_cast<const float4*>(cs + j0);
#pragma unroll
                  for (int q = 0; q < 8; ++q) {
                    const float4 cc = c4[q];
                    const float cq[4] = {cc.x, cc.y, cc.z, cc.w};
#pragma unroll
                    for (int r4 = 0; r4 < 4; ++r4) {
                      const int i = 4 * q + r4;
                      float w = accv(i);
                      if (a.mode == 1) w = fmaf(cq[r4], st[i * 128 + row], w);
                      st[i * 128 + row] = w;
                    }
                  }
                } else {
#pragma unroll
                  for (int i = 0; i < 32; ++i) {
                    float w = accv(i);
                    if (a.mode == 1) w = fmaf(cs[j0 + i], st[i * 128 + row], w);
                    st[i * 128 + row] = (valid && i < ncol) ? w : 0.f;
                  }
                }
                fence_proxy_async_smem();   // the bulk store reads these writes
                named_sync(3 + half, 128);
                // column norms: warp `quad` owns columns 8 quad .. 8 quad + 7, four
                // lanes per column, each over 32 of the 128 rows (float4 index
                // rotated by lane & 7: conflict-free within every quarter-warp),
                // combined with two shuffles; one thread per column of the CTA
                // then adds into nrm without an atomic (the columns of a group
                // belong to one half, and a half's warps own disjoint columns)
                const int cl = 8 * quad + (lane >> 2);
                const float* colp = st + cl * 128 + (lane & 3) * 32;
                float sq = 0.f;
#pragma unroll
                for (int k4 = 0; k4 < 8; ++k4) {
                  const float4 v = *reinterpret_cast<const float4*>(colp + ((k4 + lane) & 7) * 4);
                  sq = fmaf(v.x, v.x, sq);
                  sq = fmaf(v.y, v.y, sq);
                  sq = fmaf(v.z, v.z, sq);
                  sq = fmaf(v.w, v.w, sq);
                }
                sq += __shfl_xor_sync(0xffffffffu, sq, 1);
                sq += __shfl_xor_sync(0xffffffffu, sq, 2);
                if (breal && (lane & 3) == 0 && cl < ncol) nrm[j0 + cl] += static_cast<double>(sq);
                const int t = quad * 32 + lane;
                if (t == 0 && breal) {
                  bulk_s2g(a.Wout + (static_cast<size_t>(b) * g.kp + j0) * 128, st,
                           static_cast<uint32_t>(ncol) * 512u);
                  bulk_wait_read();  // the stage may be refilled after this
                }
              }
            }
            warp_arrive(W_empty + wsl);
          }
          gbase += static_cast<uint32_t>(ngp);
        } else {
          for (int c0 = 32 * half; c0 < wn && !(TC_SKIP(a) & 2); c0 += 32 * NHALF) {
            uint32_t u[32];
            tmem_ld32(tbase + lane_base + acc * a.accw + c0, u);
            tmem_wait_ld();
            const int ncol = (wn - c0) < 32 ? (wn - c0) : 32;
            auto accv = [&](int i) {
              return F16 ? __uint_as_float(u[i]) * us : __uint_as_float(u[i]);
            };
            const int s0 = nt * a.wbase + c0;
            if ((g.vmap ? g.kw : g.kh) >= 4 && ncol == 32 && s0 + 32 <= g.k) {
              // full block of real taps: the 4 tap offsets of a batch in one
              // broadcast 128-bit load, no per-column predicates
              char* const obase = reinterpret_cast<char*>(myob + hidx);
#pragma unroll
              for (int i = 0; i < 32; i += 4) {
                const int4 t4 = *reinterpret_cast<const int4*>(a.tapn + s0 + i);
                float* const o0 = reinterpret_cast<float*>(obase + t4.x);
                float* const o1 = reinterpret_cast<float*>(obase + t4.y);
                float* const o2 = reinterpret_cast<float*>(obase + t4.z);
                float* const o3 = reinterpret_cast<float*>(obase + t4.w);
                const float x0 = *o0, x1 = *o1, x2 = *o2, x3 = *o3;
                if (F16) {
                  *o0 = fmaf(__uint_as_float(u[i]), us, x0);
                  *o1 = fmaf(__uint_as_float(u[i + 1]), us, x1);
                  *o2 = fmaf(__uint_as_float(u[i + 2]), us, x2);
                  *o3 = fmaf(__uint_as_float(u[i + 3]), us, x3);
                } else {
                  *o0 = x0 + __uint_as_float(u[i]);
                  *o1 = x1 + __uint_as_float(u[i + 1]);
                  *o2 = x2 + __uint_as_float(u[i + 2]);
                  *o3 = x3 + __uint_as_float(u[i + 3]);
                }
                __syncwarp();
              }
            } else if ((g.vmap ? g.kw : g.kh) >= 4) {
              // batches of 4 consecutive N columns = 4 distinct sh (vmap 0) or
              // sw (vmap 1), the coordinate the warp's rows share: no hazards
#pragma unroll
              for (int i = 0; i < 32; i += 4) {
                float* o[4];
                float v[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const int sidx = s0 + i + q;
                  const bool ok = (i + q < ncol) && sidx < g.k;
                  o[q] = myob + (ok ? hidx + (a.tapn[sidx] >> 2) : nobp + lane);  // per-lane scratch
                  v[q] = ok ? __uint_as_float(u[i + q]) : 0.f;
                }
                float x[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) x[q] = *o[q];
#pragma unroll
                for (int q = 0; q < 4; ++q) *o[q] = F16 ? fmaf(v[q], us, x[q]) : x[q] + v[q];
                __syncwarp();
              }
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const int sidx = s0 + i;
                if (i < ncol && sidx < g.k) {
                  float* o = myob + (hidx + (a.tapn[sidx] >> 2));
                  *o += accv(i);
                }
                __syncwarp();
              }
            }
          }
        }
        tc_fence_before();
        if (PAIR) {  // one arrival per warp on the leader's ACC_empty
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(lead_accempty + 8u * static_cast<uint32_t>(acc));
        } else {
          warp_arrive(ACC_empty + acc);
        }
        if (dbg.p) {
          long long t2c = clk();
          dbg.acc[0] += t1c - t0c;
          dbg.acc[1] += t2c - t1c;
        }
      }
      if (!FWD && !(TC_SKIP(a) & 128)) {
        named_sync(2, nepi_act * 32);
        // flush: element e = (aa*HW + bb)*HT + c of the output box, advanced by
        // the step in mixed radix (no per-element divisions)
        const int hbase = h0 - (g.kh - 1) + g.hoff, wbase = w0 - (g.kw - 1), tbase_ = t0 - (g.kt - 1);
        auto emit = [&](float sv, int hs, int ws, int cc) {
          if (sv == 0.f) return;
          const int ts = wrap1(tbase_ + cc, g.T);
          const size_t oi = (static_cast<size_t>(hs) * g.W + ws) * g.T + ts;
          if (a.adjq != nullptr) {
            // deterministic: the brick's partial sum (fixed order within the
            // CTA) goes out as a {hi, lo} pair on fixed fp32 grids -- every
            // add is exact, so the flush order across CTAs does not matter
            // (adj_grid, icnnm_kernels.cuh); icnnm_adj_q2f folds the pairs
            const float hi = rintf(sv * qg.inv_qh) * qg.qh;
            const float lo = rintf((sv - hi) * qg.inv_ql) * qg.ql;
            asm volatile("red.global.add.v2.f32 [%0], {%1, %2};\n" ::"l"(a.adjq + oi), "f"(hi),
                         "f"(lo)
                         : "memory");
          } else {
            atomicAdd(a.adj + oi, sv);
          }
        };
        // deterministic flush, two frames per atomic: an even first frame and an
        // even T keep each frame pair contiguous, 16-byte aligned and on one
        // side of the periodic wrap (red.global.add.v4.f32: half the atomics)
        const bool pair_ok = a.adjq != nullptr && (((tbase_ | g.T) & 1) == 0);
        auto emit2 = [&](float s0, float s1, int hs, int ws, int cc) {
          if (s0 == 0.f && s1 == 0.f) return;
          const int ts = wrap1(tbase_ + cc, g.T);
          const size_t oi = (static_cast<size_t>(hs) * g.W + ws) * g.T + ts;
          const float h0 = rintf(s0 * qg.inv_qh) * qg.qh;
          const float l0 = rintf((s0 - h0) * qg.inv_ql) * qg.ql;
          const float h1 = rintf(s1 * qg.inv_qh) * qg.qh;
          const float l1 = rintf((s1 - h1) * qg.inv_ql) * qg.ql;
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"l"(a.adjq + oi), "f"(h0),
                       "f"(l0), "f"(h1), "f"(l1)
                       : "memory");
        };
        if ((g.HT & 3) == 0) {
          // four consecutive frames of one (aa, bb) box row per step: the
          // nepi_act per-warp copies are read and cleared with 128-bit accesses
          int c = fv_c0, bb = fv_bb0, aa = fv_aa0;
          const int ng4 = nob >> 2;
          for (int gq = ew * 32 + lane; gq < ng4; gq += nepi_act * 32) {
            float4 sv = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int q = 0; q < nepi_act; ++q) {
              float4* pq = reinterpret_cast<float4*>(ob + q * obs) + gq;
              const float4 v = *pq;
              sv.x += v.x; sv.y += v.y; sv.z += v.z; sv.w += v.w;
              *pq = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            const int ce = 4 * c, bbe = bb, aae = aa;
            c += fv_dc;
            int cy = c >= fv_nc ? 1 : 0;
            c -= cy * fv_nc;
            bb += fv_dbb + cy;
            cy = bb >= g.HW ? 1 : 0;
            bb -= cy * g.HW;
            aa += fv_daa + cy;
            if (!breal) continue;  // dummy brick: output bricks cleared, nothing written
            int hs = hbase + aae;
            if (g.wrapH) hs = wrap1(hs, g.Hsrc);
            if (hs < 0 || hs >= g.Hsrc) continue;
            const int ws = wrap1(wbase + bbe, g.W);
            if (pair_ok) {
              emit2(sv.x, sv.y, hs, ws, ce);
              emit2(sv.z, sv.w, hs, ws, ce + 2);
            } else {
              emit(sv.x, hs, ws, ce);
              emit(sv.y, hs, ws, ce + 1);
              emit(sv.z, hs, ws, ce + 2);
              emit(sv.w, hs, ws, ce + 3);
            }
          }
        } else {
          int c = fl_c0, bb = fl_bb0, aa = fl_aa0;
          for (int e = ew * 32 + lane; e < nob; e += nepi_act * 32) {
            float sv = 0.f;
            for (int q = 0; q < nepi_act; ++q) {
              sv += ob[q * obs + e];
              ob[q * obs + e] = 0.f;
            }
            const int ce = c, bbe = bb, aae = aa;
            c += fl_dc;
            int cy = c >= g.HT ? 1 : 0;
            c -= cy * g.HT;
            bb += fl_dbb + cy;
            cy = bb >= g.HW ? 1 : 0;
            bb -= cy * g.HW;
            aa += fl_daa + cy;
            if (!breal) continue;  // dummy brick: output bricks cleared, nothing written
            int hs = hbase + aae;
            if (g.wrapH) hs = wrap1(hs, g.Hsrc);
            if (hs < 0 || hs >= g.Hsrc) continue;
            emit(sv, hs, wrap1(wbase + bbe, g.W), ce);
          }
        }
        named_sync(2, nepi_act * 32);
      }
    }
    dbg.flush(DBG_EPI_WAIT, DBG_EPI_WORK);
    if (FWD && quad == 0 && lane == 0) bulk_wait_all();  // W stores complete before exit
    if (FWD && a.mode == 2) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) gacc += __shfl_xor_sync(0xffffffffu, gacc, o);
      if (a.npart != nullptr) {
        // deterministic: the CTA's partial (warps summed in a fixed order)
        if (lane == 0) nrm[ew] = static_cast<double>(gacc);
        named_sync(2, NEPI * 32);
        if (ew == 0 && lane == 0) {
          double t = 0.0;
          for (int w = 0; w < NEPI; ++w) t += nrm[w];
          a.npart[blockIdx.x] = t;
        }
      } else if (lane == 0) {
        atomicAdd(a.norm2, static_cast<double>(gacc));
      }
    } else if (FWD && a.npart != nullptr) {
      // deterministic: the CTA's column partials (its bricks, its columns;
      // zeros elsewhere) in its own row, summed over the rows in a fixed
      // order by the coefficient / fold kernel
      named_sync(2, NEPI * 32);
      for (int j = ew * 32 + lane; j < g.kp; j += NEPI * 32)
        a.npart[static_cast<size_t>(blockIdx.x) * g.kp + j] = nrm[j];
    } else if (FWD && a.norm2 != nullptr) {
      named_sync(2, NEPI * 32);
      for (int j = ew * 32 + lane; j < g.kp; j += NEPI * 32)
        if (nrm[j] != 0.0) atomicAdd(a.norm2 + j, nrm[j]);
    }
  } else if (warp < NB + NEPI) {
  } else if (warp == WMMA) {
    // ===================== MMA issuer (converged warp, elected lane issues) =====================
    if (PAIR && crank != 0) {
      // peer CTA of a pair: the leader issues the pair's MMAs; without tma_pair
      // this warp relays "my half of B stage sb landed" to the leader's B_full
      if (lane == 0 && a.bres && sfirst < nslot) {
        // resident B: one relay per launch -- "my half of every tile landed"
        mbar_wait(BRES_full, 0);
        mbar_arrive_cluster(mapa_u32(smem_u32(B_full + (SB - 2)), 0));
      } else if (lane == 0 && !(TC_SKIP(a) & 16) && !a.tma_pair) {
        const uint32_t lead_bfull = mapa_u32(smem_u32(B_full), 0);
        int sb = 0;
        uint32_t bph = 0;
        const int nfill = ((nslot - sfirst + sstep - 1) / sstep) * ntn * nkc;
        for (int f = 0; f < nfill; ++f) {
          mbar_wait(B_full + sb, bph);
          mbar_arrive_cluster(lead_bfull + 8u * static_cast<uint32_t>(sb));
          if (++sb == sbn) {
            sb = 0;
            bph ^= 1u;
          }
        }
      }
    } else {
      uint32_t cnt = 0, tcount = 0;
      int sb = 0;
      uint32_t bph = 0;
      const uint32_t bs0 = smem_u32(Bst), br0 = smem_u32(Bring);
      const uint32_t bar_af = smem_u32(A_full), bar_ae = smem_u32(A_empty);
      const uint32_t bar_bf = smem_u32(B_full), bar_be = smem_u32(B_empty);
      const uint32_t bar_accf = smem_u32(ACC_full);
      long long wa = 0, wb = 0, wacc = 0, tstart = TC_DBG(a) ? clk() : 0;
      uint32_t idesc_t[2], dcol_t[2];
      int wn_t[2];
      // MMAs of chunk kc (A stage sa, parity aph) into tile t of the current group
      int cur_nt0 = 0;  // first N-tile of the current group
      bool bres_ready = false;
      auto issue = [&](int t, int kc, int sa, uint32_t aph, bool first_use, bool last_use) {
        if (kc == kcb) {
          const uint32_t tci = tcount + static_cast<uint32_t>(t);
          long long q0 = TC_DBG(a) ? clk() : 0;
          if (!(TC_SKIP(a) & 32)) {
            if (PAIR)
              pwait(ACC_empty + (tci & 1), ((tci >> 1) & 1) ^ 1);
            else
              mbar_wait(ACC_empty + (tci & 1), ((tci >> 1) & 1) ^ 1);
          }
          if (TC_DBG(a)) wacc += clk() - q0;
        }
        long long q1 = TC_DBG(a) ? clk() : 0;
        if (first_use && !(TC_SKIP(a) & 8)) {
          if (PAIR)
            pwait(A_full + sa, aph);
          else
            mbar_wait(A_full + sa, aph);
        }
        long long q2 = TC_DBG(a) ? clk() : 0;
        const bool res = is_res(cur_nt0 + t, kc);
        if (res) {
          if (!bres_ready) {
            mbar_wait(BRES_full, 0);  // resident B: one fill per launch (phase 0)
            if (PAIR) pwait(B_full + (SB - 2), 0);  // ... and the peer's half (its relay)
            bres_ready = true;
          }
        } else if (!(TC_SKIP(a) & 16)) {
          if (PAIR)
            pwait(B_full + sb, bph);
          else
            mbar_wait(B_full + sb, bph);
        }
        if (TC_DBG(a)) {
          long long q3 = clk();
          wa += q2 - q1;
          wb += q3 - q2;
        }
        tc_fence_after();
        const uint32_t acol = tbase + a_col0 + sa * ASC;
        const uint32_t bhi = res ? bs0 + bres_off(cur_nt0 + t, kc) : br0 + sb * BSTG;
        // resident blocks release no stage: their commit goes to a barrier nobody waits on
        const uint32_t bar_b = bar_be + 8u * static_cast<uint32_t>(res ? SB - 1 : sb);
        const uint32_t dcol = dcol_t[t], idesc = idesc_t[t];
        const int wn = wn_t[t];
        const bool acc_done = kc == kce - 1 && !(TC_SKIP(a) & 32);
        if (PAIR) {
          // this CTA's half of B: hi rows [0, wn/2) then lo rows (wn/2 x 32 B each)
          tc_chunk_f16_pair(dcol, acol, acol + ALO, bdesc(bhi), bdesc(bhi + (wn / 2) * 32), idesc,
                            kc == kcb ? 0u : 1u, bar_b, bar_ae + 8u * sa,
                            bar_accf + 8u * ((tcount + static_cast<uint32_t>(t)) & 1),
                            (last_use ? 1u : 0u) | (acc_done ? 2u : 0u));
        } else if (MCB && !(TC_SKIP(a) & 24)) {
          tc_chunk_f16_mcb(dcol, acol, acol + ALO, bdesc(bhi), bdesc(bhi + wn * 32), idesc,
                           kc == kcb ? 0u : 1u, bar_b, bar_ae + 8u * sa,
                           bar_accf + 8u * ((tcount + static_cast<uint32_t>(t)) & 1),
                           (last_use ? 1u : 0u) | (acc_done ? 2u : 0u));
        } else if (F16 && !(TC_SKIP(a) & 24)) {
          tc_chunk_f16(dcol, acol, acol + ALO, bdesc(bhi), bdesc(bhi + wn * 32), idesc,
                       kc == kcb ? 0u : 1u, bar_b, bar_ae + 8u * sa,
                       bar_accf + 8u * ((tcount + static_cast<uint32_t>(t)) & 1),
                       (last_use ? 1u : 0u) | (acc_done ? 2u : 0u));
        } else {
          if (F16) {
            const uint64_t dh = bdesc(bhi);
            const uint64_t dl = bdesc(bhi + wn * 32);
            tc_mma_f16_elect(dcol, acol, dh, idesc, kc == kcb ? 0u : 1u);
            tc_mma_f16_elect(dcol, acol + ALO, dh, idesc, 1u);
            tc_mma_f16_elect(dcol, acol, dl, idesc, 1u);
          } else {
            const uint32_t blo = bhi + wn * (KC / 8) * 32;
#pragma unroll
            for (int q = 0; q < KC / 8; ++q) {
              const uint64_t dh = bdesc(bhi + q * wn * 32);
              const uint64_t dl = bdesc(blo + q * wn * 32);
              const uint32_t first = (kc == kcb && q == 0) ? 0u : 1u;
              tc_mma_ts_elect(dcol, acol + q * 8, dh, idesc, first);
              tc_mma_ts_elect(dcol, acol + ALO + q * 8, dh, idesc, 1u);
              tc_mma_ts_elect(dcol, acol + q * 8, dl, idesc, 1u);
            }
          }
          if (last_use && !(TC_SKIP(a) & 8)) tc_commit_elect(A_empty + sa);
          if (!(TC_SKIP(a) & 16) && !res) tc_commit_elect(B_empty + sb);
          if (acc_done) tc_commit_elect(ACC_full + ((tcount + static_cast<uint32_t>(t)) & 1));
        }
        if (!res && ++sb == sbn) {
          sb = 0;
          bph ^= 1u;
        }
      };
      (void)bar_af;
      (void)bar_bf;

      // A-stage (index, parity) of chunk ci, advanced incrementally within a phase
      struct StageIt {
        int s;
        uint32_t ph;
      };
      auto stage_of = [&](uint32_t ci) {
        return StageIt{static_cast<int>(ci % static_cast<uint32_t>(san)), (ci / san) & 1u};
      };
      auto next = [&](StageIt& x) {
        if (++x.s == san) {
          x.s = 0;
          x.ph ^= 1u;
        }
      };
      // Product fast path (F16x3 single CTAs, no counters): the per-chunk issue
      // sequence was the serial bottleneck of both kernels -- ~70 instructions
      // and ~370 non-waiting cycles per 192-cycle chunk at k = 245
      // (profiles/r2/README.md) -- so this loop keeps every launch parameter in
      // registers, advances descriptors / stages incrementally and commits
      // nothing for resident B blocks.
      bool lean = false;
      if constexpr (F16)
        lean = !MCB && (TC_SKIP(a) & ~(1 | 2 | 128 | 256)) == 0 &&  // (counters: MMA waits read 0)
               (!PAIR || (a.bres && !a.bmix));  // pairs: resident B only
      if (lean) {
        const uint32_t a0 = tbase + a_col0;
        const int bres = a.bres, bmix = a.bmix, nresblk = a.nresblk;
        const uint32_t res_lo0 = ((bs0 >> 4) & 0x3FFFu) | 0x80000u;   // LBO 128 B
        const uint32_t ring_lo0 = ((br0 >> 4) & 0x3FFFu) | 0x80000u;
        const uint32_t res_step = static_cast<uint32_t>(a.bres_stride) >> 4;
        const uint32_t ring_step = static_cast<uint32_t>(BSTG) >> 4;
        const uint32_t accw = static_cast<uint32_t>(a.accw);
        // one K-chunk of tile t of the current group from A stage (sa, aph)
        auto chunk = [&](int t, int c, int sa, uint32_t aph, bool first_use, bool last_use) {
          const uint32_t tci = tcount + static_cast<uint32_t>(t);
          if (c == 0) mbar_wait(ACC_empty + (tci & 1), ((tci >> 1) & 1) ^ 1);
          if (first_use) mbar_wait(A_full + sa, aph);
          const int blk = (cur_nt0 + t - ntb) * nkr + c;
          uint32_t blo, fl = (last_use ? 1u : 0u) | (c == nkr - 1 ? 2u : 0u);
          if (bres && (!bmix || blk < nresblk)) {
            if (!bres_ready) {
              mbar_wait(BRES_full, 0);
              if (PAIR) mbar_wait(B_full + (SB - 2), 0);  // the peer's half (its relay)
              bres_ready = true;
            }
            blo = res_lo0 + static_cast<uint32_t>(blk) * res_step;
          } else {
            mbar_wait(B_full + sb, bph);
            blo = ring_lo0 + static_cast<uint32_t>(sb) * ring_step;
            fl |= 4u;
          }
          tc_fence_after();
          if constexpr (PAIR)  // this CTA's half: hi rows, then lo rows (wn / 2 x 32 B each)
            tc_chunk_f16_lean_pair(tbase + (tci & 1) * accw, a0 + sa * ASC, blo,
                                   static_cast<uint32_t>(wn_t[t]), idesc_t[t], c == 0 ? 0u : 1u,
                                   bar_ae + 8u * sa, bar_accf + 8u * (tci & 1), fl);
          else
            tc_chunk_f16_lean(tbase + (tci & 1) * accw, a0 + sa * ASC, blo,
                              static_cast<uint32_t>(wn_t[t]) * 2u, idesc_t[t], c == 0 ? 0u : 1u,
                              bar_be + 8u * sb, bar_ae + 8u * sa, bar_accf + 8u * (tci & 1), fl);
          if ((fl & 4u) && ++sb == sbn) {
            sb = 0;
            bph ^= 1u;
          }
        };
        int sa = 0;        // A stage of the next chunk (chunks are consumed in build order)
        uint32_t aph = 0;
        for (int sl = sfirst; sl < nslot; sl += sstep) {
          for (int gi = 0; gi < ngrp; ++gi) {
            const int nt0 = ntb + gi * grp;
            const int gsz = (nte - nt0) < grp ? (nte - nt0) : grp;
            cur_nt0 = nt0;
            for (int t = 0; t < gsz; ++t) {
              wn_t[t] = tile_width(a, nt0 + t);
              idesc_t[t] = PAIR ? idesc_f16_m256(wn_t[t]) : idesc_f16(wn_t[t]);
            }
            auto adv = [&](int& s_, uint32_t& p_) {
              if (++s_ == san) {
                s_ = 0;
                p_ ^= 1u;
              }
            };
            if (gsz == 1) {
              for (int c = 0; c < nkr; ++c) {
                chunk(0, c, sa, aph, true, true);
                adv(sa, aph);
              }
            } else {  // the tg_seq order, phase by phase (A stage iterators x, y)
              int xs = sa;
              uint32_t xp = aph;
              for (int c = 0; c < skew; ++c, adv(xs, xp)) chunk(0, c, xs, xp, true, false);
              xs = sa;
              xp = aph;
              for (int c = 0; c < skew; ++c, adv(xs, xp)) chunk(1, c, xs, xp, false, true);
              for (int c = skew; c < nkr - skew; ++c, adv(xs, xp)) {
                chunk(0, c, xs, xp, true, false);
                chunk(1, c, xs, xp, false, true);
              }
              const int ys = xs;
              const uint32_t yp = xp;
              for (int c = nkr - skew; c < nkr; ++c, adv(xs, xp)) chunk(0, c, xs, xp, true, false);
              xs = ys;
              xp = yp;
              for (int c = nkr - skew; c < nkr; ++c, adv(xs, xp)) chunk(1, c, xs, xp, false, true);
              sa = xs;
              aph = xp;
            }
            tcount += static_cast<uint32_t>(gsz);
          }
        }
      } else
      for (int sl = sfirst; sl < nslot; sl += sstep) {
        for (int gi = 0; gi < ngrp; ++gi) {
          const int nt0 = ntb + gi * grp;
          const int gsz = (nte - nt0) < grp ? (nte - nt0) : grp;
          cur_nt0 = nt0;
          for (int t = 0; t < gsz; ++t) {
            wn_t[t] = tile_width(a, nt0 + t);
            idesc_t[t] = PAIR ? idesc_f16_m256(wn_t[t]) : (F16 ? idesc_f16(wn_t[t]) : idesc_tf32(wn_t[t]));
            dcol_t[t] = tbase + ((tcount + t) & 1) * a.accw;
          }
          if (gsz == 1) {
            StageIt x = stage_of(cnt);
            for (int kc = kcb; kc < kce; ++kc, next(x)) issue(0, kc, x.s, x.ph, true, true);
          } else {  // the tg_seq order, phase by phase
            StageIt x = stage_of(cnt);
            for (int kc = kcb; kc < kcb + skew; ++kc, next(x)) issue(0, kc, x.s, x.ph, true, false);
            x = stage_of(cnt);
            for (int kc = kcb; kc < kcb + skew; ++kc, next(x)) issue(1, kc, x.s, x.ph, false, true);
            for (int kc = kcb + skew; kc < kce - skew; ++kc, next(x)) {
              issue(0, kc, x.s, x.ph, true, false);
              issue(1, kc, x.s, x.ph, false, true);
            }
            const StageIt y = x;
            for (int kc = kce - skew; kc < kce; ++kc, next(x)) issue(0, kc, x.s, x.ph, true, false);
            x = y;
            for (int kc = kce - skew; kc < kce; ++kc, next(x)) issue(1, kc, x.s, x.ph, false, true);
          }
          cnt += static_cast<uint32_t>(nkr);
          tcount += static_cast<uint32_t>(gsz);
        }
      }
      if (TC_DBG(a) && lane == 0) {
        atomicAdd(TC_DBG(a) + DBG_MMA_WAIT_A, static_cast<unsigned long long>(wa));
        atomicAdd(TC_DBG(a) + DBG_MMA_WAIT_B, static_cast<unsigned long long>(wb));
        atomicAdd(TC_DBG(a) + DBG_MMA_WAIT_ACC, static_cast<unsigned long long>(wacc));
        atomicAdd(TC_DBG(a) + DBG_TOTAL, static_cast<unsigned long long>(clk() - tstart));
      }
    }
    __syncwarp();
  } else if (warp == WLOAD) {
    // ===================== B loader =====================
    if (lane == 0 && a.bres && sfirst < nslot) {
      // resident B: this CTA's (tile, chunk) blocks -- all of them, or the first
      // a.nresblk (mixed residency) -- loaded once (one barrier phase) and read
      // by every brick's MMAs; only when the CTA has a brick (its MMA warp then
      // waits for the fill before the CTA can exit)
      // (CTA pairs hold their half of every tile's N rows: hi half, then lo half)
      uint32_t total = 0;
      for (int nt = ntb; nt < nte; ++nt)
        for (int kc = kcb; kc < kce; ++kc)
          if (is_res(nt, kc))
            total += static_cast<uint32_t>(tile_width(a, nt) * KC * (F16 ? 4 : 8)) / (PAIR ? 2u : 1u);
      mbar_arrive_expect_tx(BRES_full, total);
      for (int nt = ntb; nt < nte; ++nt) {
        const uint32_t bytes = static_cast<uint32_t>(tile_width(a, nt)) * KC * (F16 ? 4 : 8);
        for (int kc = kcb; kc < kce; ++kc) {
          if (!is_res(nt, kc)) continue;
          uint8_t* dst = reinterpret_cast<uint8_t*>(Bst) + bres_off(nt, kc);
          const float* src = a.Bpk + (static_cast<size_t>(nt) * nkc + kc) * (B_STAGE_BYTES / 4);
          if (PAIR) {
            const uint32_t hb = bytes / 4;  // half of the rows of the hi (or lo) tile
            const uint8_t* s8 = reinterpret_cast<const uint8_t*>(src);
            bulk_g2s(dst, s8 + crank * hb, hb, BRES_full);
            bulk_g2s(dst + hb, s8 + bytes / 2 + crank * hb, hb, BRES_full);
          } else {
            bulk_g2s(dst, src, bytes, BRES_full);
          }
        }
      }
    }
    if (lane == 0 && (!a.bres || a.bmix) && !CL2 && TC_SKIP(a) == 0) {
      // Single CTAs, product path: the ring is fed by ONE thread, so its
      // instruction count per stage bounds the B stream (the general loop
      // below -- two 32-bit divisions for the ring slot and parity plus the
      // tile-group sequence decode per stage -- kept this thread busy 80% of
      // the time with the MMA warp waiting on B half of its time at k = 405:
      // profiles/r2/README.md).  Ring slot, parity and the tile-group order
      // advance incrementally here.
      int sb = 0;
      uint32_t bwph = 1;  // parity of B_empty to wait on
      const size_t blkf = B_STAGE_BYTES / 4;  // floats per packed (tile, chunk) block
      auto put = [&](int nt, int kc, uint32_t bytes) {
        if (is_res(nt, kc)) return;  // resident block: no stage
        mbar_wait(B_empty + sb, bwph);
        mbar_arrive_expect_tx(B_full + sb, bytes);
        bulk_g2s(Bring + sb * BSTG, a.Bpk + (static_cast<size_t>(nt) * nkc + kc) * blkf, bytes,
                 B_full + sb);
        if (++sb == sbn) {
          sb = 0;
          bwph ^= 1u;
        }
      };
      for (int sl = sfirst; sl < nslot; sl += sstep) {
        for (int gi = 0; gi < ngrp; ++gi) {
          const int nt0 = ntb + gi * grp;
          const int gsz = (nte - nt0) < grp ? (nte - nt0) : grp;
          const uint32_t by0 = static_cast<uint32_t>(tile_width(a, nt0)) * KC * (F16 ? 4 : 8);
          if (gsz == 1) {
            for (int kc = kcb; kc < kce; ++kc) put(nt0, kc, by0);
          } else {  // the tg_seq order, phase by phase (as the MMA warp consumes it)
            const uint32_t by1 = static_cast<uint32_t>(tile_width(a, nt0 + 1)) * KC * (F16 ? 4 : 8);
            for (int kc = kcb; kc < kcb + skew; ++kc) put(nt0, kc, by0);
            for (int kc = kcb; kc < kcb + skew; ++kc) put(nt0 + 1, kc, by1);
            for (int kc = kcb + skew; kc < kce - skew; ++kc) {
              put(nt0, kc, by0);
              put(nt0 + 1, kc, by1);
            }
            for (int kc = kce - skew; kc < kce; ++kc) put(nt0, kc, by0);
            for (int kc = kce - skew; kc < kce; ++kc) put(nt0 + 1, kc, by1);
          }
        }
      }
    } else if (lane == 0 && (!a.bres || a.bmix) && !(TC_SKIP(a) & 16)) {
      uint32_t bcnt = 0;
      long long wl = 0;
      for (int sl = sfirst; sl < nslot; sl += sstep) {
        for (int gi = 0; gi < ngrp; ++gi) {
          const int nt0 = ntb + gi * grp;
          const int gsz = (nte - nt0) < grp ? (nte - nt0) : grp;
          for (int i = 0; i < gsz * nkr; ++i) {
            int t, kc;
            tg_seq(i, gsz, nkr, skew, t, kc);
            kc += kcb;
            const int nt = nt0 + t;
            if (is_res(nt, kc)) continue;  // resident block: no stage
            const int wn = tile_width(a, nt);
            const uint32_t bytes = static_cast<uint32_t>(wn) * KC * (F16 ? 4 : 8);
            const int sb = bcnt % sbn;
            long long q0 = TC_DBG(a) ? clk() : 0;
            if (CL2)
              pwait(B_empty + sb, ((bcnt / sbn) & 1) ^ 1);
            else
              mbar_wait(B_empty + sb, ((bcnt / sbn) & 1) ^ 1);
            ++bcnt;
            if (TC_DBG(a)) wl += clk() - q0;
            if (TC_SKIP(a) & 4) {
              mbar_arrive(B_full + sb);  // timing experiment: no B traffic
              continue;
            }
            const float* src = a.Bpk + (static_cast<size_t>(nt) * nkc + kc) * (B_STAGE_BYTES / 4);
            uint8_t* dst = Bring + sb * BSTG;
            if (PAIR && a.tma_pair) {
              // this CTA's half of the N rows (hi, then lo) as two 2-SM tensor
              // copies that complete_tx on the leader's B_full, which expects
              // the whole stage (both CTAs' halves)
              const uint32_t hb = static_cast<uint32_t>(wn / 2) * 32u;
              const CUtensorMap* map = &a.tmB[wn == a.wbase ? 0 : 1];
              const int row0 = (nt * nkc + kc) * (B_STAGE_BYTES / 32);
              const uint32_t lead_bar = mapa_u32(smem_u32(B_full + sb), 0);
              if (crank == 0) mbar_arrive_expect_tx(B_full + sb, 4u * hb);
              tma2d_pair(dst, map, row0 + crank * (wn / 2), lead_bar);
              tma2d_pair(dst + hb, map, row0 + wn + crank * (wn / 2), lead_bar);
            } else if (PAIR) {
              // this CTA's half of the N rows, hi then lo (the canonical layout
              // keeps each half of the rows contiguous: 8-row core-matrix groups)
              const uint32_t hb = static_cast<uint32_t>(wn / 2) * 32u;
              const uint8_t* sb8 = reinterpret_cast<const uint8_t*>(src);
              mbar_arrive_expect_tx(B_full + sb, 2u * hb);
              bulk_g2s(dst, sb8 + crank * hb, hb, B_full + sb);
              bulk_g2s(dst + hb, sb8 + static_cast<uint32_t>(wn) * 32u + crank * hb, hb, B_full + sb);
            } else if (MCB) {
              // this CTA's half of the stage, multicast to both CTAs; the
              // local B_full expects the whole stage (both halves)
              const uint32_t h0 = ((bytes / 2) + 15u) & ~15u;
              const uint32_t mine = crank == 0 ? h0 : bytes - h0;
              const uint32_t off = crank == 0 ? 0u : h0;
              mbar_arrive_expect_tx(B_full + sb, bytes);
              bulk_g2s_mc(dst + off, reinterpret_cast<const uint8_t*>(src) + off, mine, B_full + sb,
                          static_cast<uint16_t>(3));
            } else {
              mbar_arrive_expect_tx(B_full + sb, bytes);
              bulk_g2s(dst, src, bytes, B_full + sb);
            }
          }
        }
      }
      // drain: every stage released by the MMAs that signal into this CTA
      // (the leader's, or both CTAs' under MCB) before the final cluster sync
      if (CL2)
        for (int q = 0; q < sbn; ++q, ++bcnt)
          pwait(B_empty + bcnt % sbn, ((bcnt / sbn) & 1) ^ 1);
      if (TC_DBG(a)) atomicAdd(TC_DBG(a) + DBG_LOAD_WAIT, static_cast<unsigned long long>(wl));
    }
    __syncwarp();
  } else if (FWD && warp == WLOAD + 1) {
    if (lane == 0) {
      // forward: stream W groups (32 columns x 128 rows, 16 KB contiguous in
      // the [brick][j][row] layout) into the ring ahead of the epilogue; mode 0
      // has no W_old (the slot is only handed over).  Tiles are padded to an
      // even number of groups so that each stage serves one epilogue half.
      int wsl_it = 0;        // ring slot and parity, advanced incrementally (one thread
      uint32_t wwph = 1;     // feeds the ring: no per-group divisions)
      for (int sl = sfirst; sl < nslot; sl += sstep) {
        const int b = brick_of(sl);
        for (int nt = ntb; nt < nte; ++nt) {
          const int wn = tile_width(a, nt);
          const int ng = (wn + 31) / 32, ngp = ng + (ng & 1);
          for (int gq = 0; gq < ngp; ++gq) {
            const int wsl = wsl_it;
            mbar_wait(W_empty + wsl, wwph);
            if (++wsl_it == wsn) {
              wsl_it = 0;
              wwph ^= 1u;
            }
            if (gq < ng && a.mode >= 1 && !(TC_SKIP(a) & 2)) {
              const int ncol = (wn - 32 * gq) < 32 ? (wn - 32 * gq) : 32;
              const uint32_t bytes = static_cast<uint32_t>(ncol) * 512u;
              mbar_arrive_expect_tx(W_full + wsl, bytes);
              bulk_g2s(reinterpret_cast<uint8_t*>(Wst) + wsl * WO_STAGE_BYTES,
                       a.Wout + (static_cast<size_t>(b) * g.kp + nt * a.wbase + 32 * gq) * 128,
                       bytes, W_full + wsl);
            } else {
              mbar_arrive(W_full + wsl);
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (!FWD && warp == WLOAD + 1) {
    if (lane == 0) {
      // adjoint: stream W chunks (16 columns x 128 rows, 8 KB contiguous in the
      // [brick][j][row] layout) ahead of the builders
      int wsi_it = 0;        // ring slot and parity, advanced incrementally
      uint32_t wwph = 1;
      for (int sl = sfirst; sl < nslot; sl += sstep) {
        const int b = brick_of(sl);
        for (int gi = 0; gi < ngrp; ++gi) {
          for (int kc = kcb; kc < kce; ++kc) {
            const int wsi = wsi_it;
            mbar_wait(W_empty + wsi, wwph);
            if (++wsi_it == wsn) {
              wsi_it = 0;
              wwph ^= 1u;
            }
            if (TC_SKIP(a) & 256) {  // timing experiment: no W traffic
              mbar_arrive(W_full + wsi);
              continue;
            }
            mbar_arrive_expect_tx(W_full + wsi, W_STAGE_BYTES);
            const float* src = a.Win + (static_cast<size_t>(b) * g.kp + kc * KC) * 128;
            bulk_g2s(reinterpret_cast<uint8_t*>(Wst) + wsi * W_STAGE_BYTES, src, W_STAGE_BYTES,
                     W_full + wsi);
          }
        }
      }
    }
    __syncwarp();
  }

  tc_fence_before();
  if (CL2)
    cluster_sync_all();  // no CTA leaves while its peer can still signal into it
  else
    __syncthreads();
  tc_fence_after();
  if (warp == WMMA) {
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
  }
}

template __global__ void icnnm_tc_kernel<true, false, false>(const __grid_constant__ TcArgs);
template __global__ void icnnm_tc_kernel<false, false, false>(const __grid_constant__ TcArgs);
template __global__ void icnnm_tc_kernel<true, true, false>(const __grid_constant__ TcArgs);
template __global__ void icnnm_tc_kernel<false, true, false>(const __grid_constant__ TcArgs);
template __global__ void icnnm_tc_kernel<true, true, true>(const __grid_constant__ TcArgs);
template __global__ void icnnm_tc_kernel<false, true, true>(const __grid_constant__ TcArgs);

void* fwd_kernel_ptr(bool f16, bool pair) {
  if (f16 && pair) return reinterpret_cast<void*>(&icnnm_tc_kernel<true, true, true>);
  return f16 ? reinterpret_cast<void*>(&icnnm_tc_kernel<true, true, false>)
             : reinterpret_cast<void*>(&icnnm_tc_kernel<true, false, false>);
}
void* adj_kernel_ptr(bool f16, bool pair) {
  if (f16 && pair) return reinterpret_cast<void*>(&icnnm_tc_kernel<false, true, true>);
  return f16 ? reinterpret_cast<void*>(&icnnm_tc_kernel<false, true, false>)
             : reinterpret_cast<void*>(&icnnm_tc_kernel<false, false, false>);
}

}  // namespace tc
}  // namespace icnnm_dev

namespace icnnm_dev {
namespace tc {
// Host: the tap table of one kernel (TcArgs::tapn) from its geometry.
void tc_fill_taps(TcArgs& a, bool fwd) {
  const Geo& g = a.g;
  for (int s = 0; s < TAPMAX; ++s) {
    int off = 0;
    if (s < g.k) {
      int st, sw, sh;
      if (fwd) {
        st = s % g.kt;
        const int q = s / g.kt;
        sw = q % g.kw;
        sh = q / g.kw;
      } else if (g.vmap) {
        // adjoint N order (host adj_tap): vmap 1 -- the warp's rows share vw, sw fastest
        sw = s % g.kw;
        const int q = s / g.kw;
        st = q % g.kt;
        sh = q / g.kt;
      } else {
        // vmap 0 -- sh fastest: within a warp the 32 rows share vh, so taps
        // with different sh never hit the same output cell and the col2im
        // scatter can batch them hazard-free
        sh = s % g.kh;
        const int q = s / g.kh;
        st = q % g.kt;
        sw = q / g.kt;
      }
      off = (sh * g.HW + sw) * g.HT + st;
    }
    a.tapn[s] = -4 * off;
  }
}
}  // namespace tc
}  // namespace icnnm_dev
