// Compile-time tuning switches of the product library.
//
// The shipped build reads no environment variables: every kernel-selection and schedule choice
// below is fixed at compile time to the measured default (DESIGN.md section 4 records the A/B
// measurements behind each).  Experiment builds override them with -D flags through
// tools/build_variant.py (e.g. `python tools/build_variant.py nopdl -DMCP_CFG_PDL=0`), never in
// the product .so.  The one per-context run-time option (the fused reduce+finish, used by the
// bitwise fused-vs-unfused test) is set through mcp_set_option().
#pragma once

// programmatic dependent launch along the kernel chains
#ifndef MCP_CFG_PDL
#define MCP_CFG_PDL 1
#endif
// host evaluations: x pulled from mapped pinned memory by a kernel (0) or copy-engine memcpys (1)
#ifndef MCP_CFG_HOST_MEMCPY
#define MCP_CFG_HOST_MEMCPY 0
#endif
// K1Z: FP64 evaluations with r <= 32, n <= 512 and at most MCP_CFG_K1Z_MAX_ROWS rows per SM
// run as ONE cooperative launch (csrc/k1z_small.cuh) where the general chain would be the
// 4-6 launch prep -> K1 -> reduce -> tail.  Measured crossover against that chain
// (tools/sweep_small.py, profiles/r02/sweep_small_k1z.txt): 140-290 rows per CTA.
#ifndef MCP_CFG_K1Z
#define MCP_CFG_K1Z 1
#endif
#ifndef MCP_CFG_K1Z_MAX_ROWS
#define MCP_CFG_K1Z_MAX_ROWS 128
#endif
// K1Z launch: cooperative (every CTA resident by contract: the grid barrier cannot deadlock
// against other kernels) or a plain launch (experiment builds, timing only)
#ifndef MCP_CFG_K1Z_COOP
#define MCP_CFG_K1Z_COOP 1
#endif
// K1Z launched cooperatively AND with programmatic stream serialization (its launch latency
// hides under the predecessor; probed once per process).  Works, and back-to-back evaluations
// gain 7% (16.4 -> 15.2 us), but the device Adam loses (batch 100: 24.7 vs 21.3 us per
// iteration, batch 1000: 30.2 vs 25.6 -- profiles/r02/ab_k1z_pdl.txt), so off
#ifndef MCP_CFG_K1Z_PDL
#define MCP_CFG_K1Z_PDL 0
#endif
#ifndef MCP_CFG_K1Z_MAXG
#define MCP_CFG_K1Z_MAXG 0         // cap on K1Z's CTAs (0: one per SM)
#endif
#ifndef MCP_K1Z_PROF
#define MCP_K1Z_PROF 0             // per-phase clock stamps printed by three CTAs (experiment builds)
#endif
#ifndef MCP_K1Z_KO
#define MCP_K1Z_KO 0               // timing knockouts (wrong results), experiment builds only
#endif
// stochastic path: Adam iterations per replayed graph (1: one graph launch per iteration)
#ifndef MCP_CFG_ADAM_ITER_CHUNK
#define MCP_CFG_ADAM_ITER_CHUNK 128
#endif
// stochastic path: the Adam update runs inside K1Z's finish when the mini-batch plans to K1Z
#ifndef MCP_CFG_ADAM_FUSED_STEP
#define MCP_CFG_ADAM_FUSED_STEP 1
#endif
// device L-BFGS: the host polls each round's record count in mapped memory instead of
// synchronising the stream after every evaluation
#ifndef MCP_CFG_LBFGS_POLL
#define MCP_CFG_LBFGS_POLL 1
#endif
// device L-BFGS: up to 256 variables (one block per run, e.g. c1) the round prologue (pull, save,
// accept, direction, trial) is one kernel instead of five launches
#ifndef MCP_CFG_LBFGS_FUSED_SMALL
#define MCP_CFG_LBFGS_FUSED_SMALL 1
#endif
// FP64 K1 family for n <= 128: K1Q (warp-specialised pairs), then K1P, then K1S fallbacks
#ifndef MCP_CFG_K1Q
#define MCP_CFG_K1Q 1
#endif
#ifndef MCP_CFG_K1P
#define MCP_CFG_K1P 1
#endif
#ifndef MCP_CFG_K1S
#define MCP_CFG_K1S 1
#endif
// r mod 8 in 1..2 runs as DFMA tail columns (0: pad to DMMA-only columns, measured 22% slower)
#ifndef MCP_CFG_DFMA_TAIL
#define MCP_CFG_DFMA_TAIL 1
#endif
// K1R warp triads (experiment, 5% slower than K1Q at c2): not compiled into the product build
#ifndef MCP_WITH_K1R
#define MCP_WITH_K1R 0
#endif
#ifndef MCP_CFG_K1X
#define MCP_CFG_K1X 1              // K1X (16 warps, double-buffered tiles) for 384 < n <= 512
#endif
// K1X's n <= 1024 shape (T = 16, RB = 8) for 768 < n <= 1024 instead of K1G: measured 770 ms at
// c5 vs 617 ms for K1G (two row blocks per 16-row tile: the P waits and the 256-thread merge
// barrier cost twice as much per DMMA as at T = 32), so experiment builds only
#ifndef MCP_CFG_K1X_1024
#define MCP_CFG_K1X_1024 0
#endif
// K1G (Y partial in L2) for large n when K1's register-bound column block is <= 1/4 of K1G's
#ifndef MCP_CFG_K1G
#define MCP_CFG_K1G 1
#endif
// K1GT: K1G with the Y partial in TMEM (no L2 read-modify-write) when n_chunks * 16 <= 512
#ifndef MCP_CFG_K1GT
#define MCP_CFG_K1GT 1
#endif
// K1GT with 16 warps (column halves per warp, 128 TMEM columns per thread) for RB = 32 and
// n <= 1024: measured 664 ms at c5 vs 643 ms with 8 warps (half the DMMA chains per warp, V
// fragments loaded twice), so experiment builds only
// K1GT at RB = 64 with chunks beyond TMEM's 256 columns per thread kept in L2 (n <= 1024)
#ifndef MCP_CFG_K1GT_HALF
#define MCP_CFG_K1GT_HALF 1
#endif
#ifndef MCP_CFG_K1GT_NW
#define MCP_CFG_K1GT_NW 8
#endif
#ifndef MCP_CFG_FORCE_K1G
#define MCP_CFG_FORCE_K1G 0
#endif
// ||X||^2 on fp64 sets: K53 (TMA ring, no CTA barrier) instead of K52 (cp.async chunks)
#ifndef MCP_CFG_K53
#define MCP_CFG_K53 1
#endif
// K53 with each tile pair split in two 64-row halves (8 warps, two CTAs per SM)
#ifndef MCP_CFG_K53_HALF
#define MCP_CFG_K53_HALF 1
#endif
#ifndef MCP_CFG_K53_TI
#define MCP_CFG_K53_TI 64          // I-tile rows per CTA when split: 64 (2 CTAs / SM) or 32
#endif
// fast mode: K1T2 (precomputed V_lo) unless 1 -> the in-kernel split K1T
#ifndef MCP_CFG_K1T_V1
#define MCP_CFG_K1T_V1 0
#endif
// fast mode: V_lo formed in shared memory by splitter warps (no V_lo copy in HBM)
#ifndef MCP_CFG_K1T2_INSPLIT
#define MCP_CFG_K1T2_INSPLIT 1
#endif
// fast mode: up to two GEMM2 m-tiles accumulate in Z's TMEM columns and drain every tile, so
// the column block can stay 64 where the persistent Y would not fit (c5)
#ifndef MCP_CFG_K1T2_TRANSIENT
#define MCP_CFG_K1T2_TRANSIENT 1
#endif
#ifndef MCP_CFG_K1T2_TRWIDE
// one wide transient m-tile so every GEMM2 m-tile is wide (c3): measured 5.77 vs 5.09 ms with
// the per-element RED drain and 5.16-5.17 vs 5.10-5.13 ms with the bulk tensor reduce-add drain
#define MCP_CFG_K1T2_TRWIDE 0
#endif
#ifndef MCP_CFG_K1T2_SERIAL
#define MCP_CFG_K1T2_SERIAL 1
#endif
#ifndef MCP_CFG_K1T2_HINT
#define MCP_CFG_K1T2_HINT 1
#endif
#ifndef MCP_CFG_K1T2_FLUSH
#define MCP_CFG_K1T2_FLUSH 16
#endif
#ifndef MCP_CFG_K1T2_RB
#define MCP_CFG_K1T2_RB 0          // 0: widest column block TMEM allows
#endif
#ifndef MCP_CFG_K1T2_WIDE
#define MCP_CFG_K1T2_WIDE 1
#endif
#ifndef MCP_CFG_K1T2_G2_3D
#define MCP_CFG_K1T2_G2_3D 1
#endif
#ifndef MCP_CFG_K1T_ZCAT
#define MCP_CFG_K1T_ZCAT 1
#endif
// GEMM2 as V P_hi with round-to-nearest P_hi (8-9% faster, error up to 7e-5 normwise): off
#ifndef MCP_CFG_K1T2_G2X2
#define MCP_CFG_K1T2_G2X2 0
#endif
