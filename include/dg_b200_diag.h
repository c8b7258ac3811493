/*
 * dg_b200_diag.h -- DIAGNOSTICS of the B200 densegraph library, built as a
 * separate shared object (paper_2311_04333_b200/libdg_b200_diag.so, linked
 * against libdg_b200.so): latency microbenchmarks that set the per-round and
 * per-batch floors quoted in DESIGN.md, and read-outs of the instrumented
 * (profiling) kernel variants.  Not part of the drop-in boundary; the
 * product library carries none of this code.
 */
#ifndef DG_B200_DIAG_H
#define DG_B200_DIAG_H

#include "dg_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Diagnostic latency floors (ns per op): 0 grid barrier (this library's),
 * 1 cooperative-groups grid.sync, 2 cluster barrier (8 CTAs), 3 CTA barrier
 * (1024 threads), 4 dependent L2 load, 5 shared atomicAdd per warp
 * instruction (spread addresses), 6 plain shared load+store per warp instr,
 * 7/8 dependent load over 64 MiB / 1 GiB, 9/10 cluster barrier (16 / 4 CTAs),
 * 11 shared atomic with the result used per warp instruction (spread), 12
 * spread shared load per warp instruction, 13 / 14 / 15 dependent shared
 * load / redux.sync / shared atomic chain (one warp, latency per op); 16 / 17
 * / 18 shared load / reduction / atomic with return at random addresses, 8 in
 * flight per thread (throughput per warp instruction); 100 + (11..18)
 * reports SM cycles per op (clock64) instead of ns. */
dg_status dg_microbench(int which, uint64_t iters, double* ns_per_op);
/* Diagnostic (instrumented launches only, see dg_peel_trace_arm): thread-0 SM
 * cycles of the last Greedy++ peel launch spent in S1 (min scan), S2 (batch
 * extraction), S3 (removal), its batch count, S3 cycles of single-vertex
 * batches, their count, #batches > 32, n, #batches on the table path. */
dg_status dg_peel_profile(uint64_t out[16]);
/* Diagnostic: launch the instrumented single-CTA peel (fills dg_peel_profile)
 * and record a per-warp timeline (SM cycles) of batches [first_batch,
 * first_batch + 8) of subsequent launches; 0xFFFFFFFF disarms.  Read it as
 * [8 batches][32 warps][12 stamps]: loop top, S1 done, S2 start, S2 done,
 * S3 start, S3 done, then kernel-specific S1 internals (candidate-list
 * kernel: list length read, list + key loads, warp min). */
dg_status dg_peel_trace_arm(uint32_t first_batch);
dg_status dg_peel_trace_read(uint64_t out[8 * 32 * 12]);
/* Diagnostic: block-0 cycles of the last coreness launch in level-advance min
 * scans, level-advance barriers, collects, expansion, flushes, expansion
 * barriers; #level advances; #overflow collects. */
#define DG_KCORE_PROFILE_WORDS (8 + 6 * 4096)
dg_status dg_kcore_profile(uint64_t out[DG_KCORE_PROFILE_WORDS]); /* + per-round and per-level traces */

#ifdef __cplusplus
}
#endif
#endif
