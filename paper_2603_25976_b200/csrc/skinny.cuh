// Output-layer ("skinny", N or K = c <= 32) kernels: argument structs + launchers.
#pragma once
#include "internal.h"

namespace cv {

struct SkinnySeg {
  const __half* a_hi; const __half* a_lo; int64_t lda; const Scale* a_sc;  // A: rows x K row-major (split)
  const __half* b_hi; const __half* b_lo; int64_t ldb; const Scale* b_sc;  // B: K x c row-major (split)
  int K;
};

enum SkinnyPost : int { POST_LOGITS = 0, POST_HZ = 1 };

// out[m, :c] = post( sum_s A_s[m, :] @ B_s )
struct SkinnyRowsArgs {
  int rows, c, nseg;
  SkinnySeg seg[2];
  int post;               // SkinnyPost
  int loss;               // CV_LOSS_*
  const float* probs;     // rows x c (POST_HZ, ce)
  float scale;            // POST_HZ: 1/b_global
  float* out;             // rows x c
  float* out_amax;        // optional: max |out|
  const int* skip;
};

// G[m, n] = epi( sum_s U_s[m, :c] . W_s[n, :c] ),  W_s = n x c row-major (ld c)
struct SkinnyDxArgs {
  int rows, n, c, nseg;
  const float* U[2];
  const __half* w_hi[2]; const __half* w_lo[2]; const Scale* w_sc[2];
  Epilogue epi;           // split output; epi.bound covers c * amax(U_s) * amax(W_s)
  const int* skip;
};

// out[m, j] = sum_s sum_k A_s[k, m] U_s[k, j]   (m < M = n + 1, ld c)
struct SkinnyDwArgs {
  int rows, M, c, nseg, ksplit;
  const __half* a_hi[2]; const __half* a_lo[2]; int64_t lda[2]; const Scale* a_sc[2];
  const float* U[2];
  float* partial;   // ksplit x M x c
  float* out;       // M x c
  const int* skip;
};

void skinny_rows(cv_ctx* ctx, const SkinnyRowsArgs& a);
void skinny_dx(cv_ctx* ctx, const SkinnyDxArgs& a);
void skinny_dw(cv_ctx* ctx, SkinnyDwArgs a, float* ws, int64_t ws_elems);

}  // namespace cv
