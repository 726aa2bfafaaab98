// Internal GEMM engines behind enks_gemm.
#pragma once
#include "common.cuh"

namespace enks {

int gemm_simt(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, float alpha,
              const float* A, int64_t lda, const float* B, int64_t ldb, float beta,
              const float* C0, int64_t ldc0, const float* bias, int64_t ld_bias, int bias_cols,
              float* C, int64_t ldc, int64_t tri_rows, int64_t tri_k, int split_k, void* ws,
              cudaStream_t st);

// tcgen05 3xTF32 engine for the NT contraction C = alpha * A B^T (+ beta C0 + bias).
bool tc_gemm_applicable(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, const float* A,
                        int64_t lda, const float* B, int64_t ldb, int64_t tri_rows);
int gemm_tc(int64_t M, int64_t N, int64_t K, float alpha, const float* A, int64_t lda,
            const float* B, int64_t ldb, float beta, const float* C0, int64_t ldc0,
            const float* bias, int64_t ld_bias, int bias_cols, float* C, int64_t ldc, int split_k,
            void* ws, cudaStream_t st);
int gemm_tc_presplit(int64_t M, int64_t N, int64_t K, float alpha, const float* A, int64_t lda,
                     const float* Bh, const float* Bl, int64_t ldb, float beta, const float* C0,
                     int64_t ldc0, float* C, int64_t ldc, int split, float* ws, cudaStream_t st);
int tc_choose_split(int64_t M, int64_t K);
int64_t tc_ws_bytes(int64_t M, int64_t N, int64_t K, int split);

}  // namespace enks
