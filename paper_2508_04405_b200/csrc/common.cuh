// Shared definitions for the sm_100a W6Ax kernels.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/flexq.h"

namespace flexq {

// ---- error plumbing (host) ---------------------------------------------------
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);
#define FLEXQ_LAUNCH_CHECK(where)                               \
  do {                                                          \
    cudaError_t _e = cudaGetLastError();                        \
    if (_e != cudaSuccess) return ::flexq::cuda_status(_e, where); \
  } while (0)

// ---- geometry ------------------------------------------------------------------
constexpr int kChunkK = 128;   // packing.py:27 MMA_K, one FLXQ-P k-chunk
constexpr int kKStep = 32;     // mma.m16n8k32 contraction per instruction
constexpr int kStepsPerBlock = 4;  // one T6 k-block = 4 k-steps = 128 k-slots
constexpr int kRowTile = 16;   // mma M (weight rows per A fragment)
constexpr int kTokTile = 8;    // mma N (tokens per B fragment)

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Group-padded K geometry of the T6 layouts: every scale group occupies
// spg = ceil(group_size/32) k-steps, so a k-step never straddles two groups.
struct T6Geom {
  int64_t n, k, gs;
  int64_t ng;   // scale groups  ceil(k / gs)
  int64_t spg;  // k-steps per group
  int64_t ks;   // total k-steps = ng * spg
  int64_t kb;   // k-blocks = ceil(ks / 4)
  int64_t rt;   // row tiles = ceil(n / 16)
  __host__ __device__ T6Geom(int64_t n_, int64_t k_, int64_t gs_) : n(n_), k(k_), gs(gs_) {
    ng = cdiv(k, gs);
    spg = cdiv(gs < k ? gs : k, kKStep);  // a group holds at most min(gs, k) elements
    ks = ng * spg;
    kb = cdiv(ks, kStepsPerBlock);
    rt = cdiv(n, kRowTile);
  }
  // padded slot of logical column kk
  __host__ __device__ int64_t slot(int64_t kk) const {
    int64_t g = kk / gs, j = kk - g * gs;
    return g * spg * kKStep + j;
  }
};

}  // namespace flexq
