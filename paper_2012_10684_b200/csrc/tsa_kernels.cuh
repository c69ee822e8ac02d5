// tsa_kernels.cuh -- the libtsa kernels (sm_100a), one file per SURVEY.md §8(a) row:
//   a1 k_histogram.cuh   per-slice gray-level histogram
//   a2 k_tables.cuh      prefix tables of c and c^q (k_luts, k_scan, k_rtable)
//   a3 k_search.cuh      exhaustive tuple search, fp64
//   a4 k_finalize.cuh    argmax merge + phi(t*) recompute
//   f4 k_dp.cuh          exact O(k m^2) interval DP for the fold
//   a5 k_label.cuh       Algorithm 1 generalised to k classes
//   f2 k_hu.cuh          pre-processing fused into histogram / labels PAPER.md:514-516
//   f3 k_morph.cuh       disk opening / top-hat (streaming, 16-bit SIMD)
//   f1 k_tsallis2d.cuh   the paper's 2-D formulation (cluster per slice) PAPER.md:564-597
#pragma once
#include "k_histogram.cuh"
#include "k_tables.cuh"
#include "k_search.cuh"
#include "k_finalize.cuh"
#include "k_scan_seed.cuh"
#include "k_label.cuh"
#include "k_dp.cuh"
#include "k_tsallis2d.cuh"
#include "k_hu.cuh"
#include "k_morph.cuh"
