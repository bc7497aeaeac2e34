/*
 * mpbjac_order.h — the row-tile plan and the fixed reduction order shared by
 * the CUDA kernels (paper_2407_15973_b200/csrc) and the CPU oracle's
 * "device order" mode (oracle/mpbjac_oracle.c).
 *
 * Why this exists: the reference (pkg/src/mpcg/kernels_numba.py:18-34) sums
 * dot products strictly left to right, which no GPU can do in parallel.
 * Every other operation on the PCG hot path (SpMV, block-Jacobi sweeps,
 * narrowing, axpys) is reproduced bit for bit by thread-per-row sequential
 * accumulation without FMA.  So the only freedom is the order of the fp64
 * dot/norm sums, and we FIX it here, independent of launch configuration and
 * SM count, so that (a) every GPU solve is bitwise reproducible and (b) the
 * oracle can replay the exact same order and match the GPU solve bit for bit
 * (x, trace, iteration count).
 *
 * Row-tile plan (computed on the host from the block partition):
 *   walk the partition's blocks in order; a block with more than
 *   MPB_TILE_MAX_ROWS rows closes the open tile and is cut into chunks of
 *   MPB_TILE_MAX_ROWS rows, one tile each ("large" partition); otherwise the
 *   block joins the open tile unless that would exceed MPB_TILE_MAX_ROWS rows
 *   or MPB_TILE_PACK_NNZ nonzeros, in which case the open tile is closed first.
 *   Tiles therefore hold whole blocks whenever blocks are small, which is what
 *   lets one CTA run all inner Jacobi sweeps of its blocks in shared memory.
 *
 * Tile sum of per-row values v[row] over rows [lo, hi):
 *   1. lane j in [0, MPB_TILE_THREADS): s_j = 0; s_j += v[lo + j + m*MPB_TILE_THREADS]
 *      for m = 0, 1, ... while the row is < hi (one rounding per add; with
 *      MPB_TILE_THREADS == MPB_TILE_MAX_ROWS every lane owns at most one row);
 *   2. each warp butterflies (xor 16, 8, 4, 2, 1) -> lane 0 holds W_w;
 *   3. warp 0 butterflies W_0..W_{nw-1} padded with +0.0 to 32 lanes.
 * Global sum of the tile partials P[0..T):
 *   T <= MPB_ONE_LEVEL_TILES: steps 1-3 with MPB_FIN_THREADS lanes over P.
 *   Larger T, two levels: chunk c = tiles [c*MPB_CHUNK_TILES,
 *     min(T, (c+1)*MPB_CHUNK_TILES)); C_c = steps 1-3 with MPB_CHUNK_TILES
 *     lanes over the chunk's partials (lane j holds P[c*MPB_CHUNK_TILES + j]
 *     or +0.0); total = steps 1-3 with MPB_FIN_THREADS lanes over the C_c.
 *   The chunks are summed while the kernel runs, by the CTA that claimed a
 *   chunk's last tile, so the kernel's final CTA adds T/256 values instead of
 *   T (C3: 65,536 partials, C5: 524,288).  Up to MPB_ONE_LEVEL_TILES the
 *   final CTA's one-level sum (two rounds of loads) is the faster one.
 * Multi-GPU: each rank's global sum is combined by an fp64 all-reduce.
 */
#ifndef MPBJAC_ORDER_H
#define MPBJAC_ORDER_H

#define MPB_TILE_THREADS   256
#define MPB_TILE_MAX_ROWS  256
#define MPB_TILE_PACK_NNZ  2048
#define MPB_FIN_THREADS    256
#define MPB_CHUNK_TILES    256
#define MPB_ONE_LEVEL_TILES 8192

#endif
