// Exact-fp32 varlen attention on CUDA cores (UB_FP32): the tiny-shape path of BASELINE
// config 1 (4 sequences, 2 heads, head_dim 8).  Same contract as the tensor-core path
// (Eq. 1; packed layout P:302; dropout R4/R5), one thread per query (or key) row,
// fp32 throughout.  Launch-latency bound by design; the bf16 path is fmha_fwd_sm100.cu.
#include <cmath>

#include "sm100.cuh"
#include "ub_internal.h"

namespace ub {

constexpr int kSimtRows = 64;
constexpr int kMaxD = 128;

struct SimtArgs {
  const float* qkv; const int32_t* cu; float* out; float* lse; const float* dout; const float* o;
  float* dqkv; float* delta;
  int32_t H, D; int64_t T; float scale, p, rp; uint32_t thr, k0, k1, off;
};

__device__ __forceinline__ bool keep_elem(const SimtArgs& a, int64_t t, int h, int j) {
  if (a.thr == 0) return true;
  const U4 w = philox4x32_10((uint32_t)j >> 4, (uint32_t)t, (uint32_t)h, a.off, a.k0, a.k1);
  const int widx = (j & 15) >> 2;
  const uint32_t word = widx == 0 ? w.x : widx == 1 ? w.y : widx == 2 ? w.z : w.w;
  const uint32_t r8 = (word >> (8 * (j & 3))) & 0xFFu;
  return r8 >= a.thr;
}

__device__ __forceinline__ const float* row_ptr(const SimtArgs& a, int64_t t, int which, int h) {
  return a.qkv + ((t * 3 + which) * a.H + h) * (int64_t)a.D;
}

__global__ void simt_fwd_kernel(SimtArgs a) {
  const int b = blockIdx.z, h = blockIdx.y;
  const int i = blockIdx.x * kSimtRows + threadIdx.x;
  const int32_t c0 = a.cu[b], L = a.cu[b + 1] - c0;
  if (i >= L) return;
  const int64_t t = c0 + i;
  float q[kMaxD], acc[kMaxD];
  const float* qp = row_ptr(a, t, 0, h);
  for (int d = 0; d < a.D; ++d) { q[d] = qp[d]; acc[d] = 0.f; }
  float m = -INFINITY;
  for (int j = 0; j < L; ++j) {
    const float* kp = row_ptr(a, c0 + j, 1, h);
    float s = 0.f;
    for (int d = 0; d < a.D; ++d) s = fmaf(q[d], kp[d], s);
    m = fmaxf(m, s * a.scale);
  }
  float l = 0.f;
  for (int j = 0; j < L; ++j) {
    const float* kp = row_ptr(a, c0 + j, 1, h);
    float s = 0.f;
    for (int d = 0; d < a.D; ++d) s = fmaf(q[d], kp[d], s);
    const float pexp = expf(s * a.scale - m);
    l += pexp;
    if (keep_elem(a, t, h, j)) {
      const float* vp = row_ptr(a, c0 + j, 2, h);
      for (int d = 0; d < a.D; ++d) acc[d] = fmaf(pexp, vp[d], acc[d]);
    }
  }
  const float inv = a.rp / l;
  float* op = a.out + (t * a.H + h) * (int64_t)a.D;
  for (int d = 0; d < a.D; ++d) op[d] = acc[d] * inv;
  a.lse[(int64_t)h * a.T + t] = m + logf(l);
}

__global__ void simt_delta_kernel(SimtArgs a) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // over T*H
  if (idx >= a.T * a.H) return;
  const int64_t t = idx / a.H;
  const int h = (int)(idx % a.H);
  const float* o = a.o + (t * a.H + h) * (int64_t)a.D;
  const float* g = a.dout + (t * a.H + h) * (int64_t)a.D;
  float s = 0.f;
  for (int d = 0; d < a.D; ++d) s = fmaf(o[d], g[d], s);
  a.delta[(int64_t)h * a.T + t] = s;
}

// dQ_i = scale * sum_j dS_ij k_j,   dS_ij = P_ij (dP_ij - Delta_i)
__global__ void simt_dq_kernel(SimtArgs a) {
  const int b = blockIdx.z, h = blockIdx.y;
  const int i = blockIdx.x * kSimtRows + threadIdx.x;
  const int32_t c0 = a.cu[b], L = a.cu[b + 1] - c0;
  if (i >= L) return;
  const int64_t t = c0 + i;
  float q[kMaxD], g[kMaxD], acc[kMaxD];
  const float* qp = row_ptr(a, t, 0, h);
  const float* gp = a.dout + (t * a.H + h) * (int64_t)a.D;
  for (int d = 0; d < a.D; ++d) { q[d] = qp[d]; g[d] = gp[d]; acc[d] = 0.f; }
  const float lse = a.lse[(int64_t)h * a.T + t], dl = a.delta[(int64_t)h * a.T + t];
  const float rs = a.rp;
  for (int j = 0; j < L; ++j) {
    const float* kp = row_ptr(a, c0 + j, 1, h);
    const float* vp = row_ptr(a, c0 + j, 2, h);
    float s = 0.f, dp = 0.f;
    for (int d = 0; d < a.D; ++d) { s = fmaf(q[d], kp[d], s); dp = fmaf(g[d], vp[d], dp); }
    const float P = expf(s * a.scale - lse);
    dp = keep_elem(a, t, h, j) ? dp * rs : 0.f;
    const float ds = P * (dp - dl);
    for (int d = 0; d < a.D; ++d) acc[d] = fmaf(ds, kp[d], acc[d]);
  }
  float* dq = a.dqkv + ((t * 3 + 0) * a.H + h) * (int64_t)a.D;
  for (int d = 0; d < a.D; ++d) dq[d] = acc[d] * a.scale;
}

// dV_j = sum_i P~_ij dO_i ;  dK_j = scale * sum_i dS_ij q_i
__global__ void simt_dkdv_kernel(SimtArgs a) {
  const int b = blockIdx.z, h = blockIdx.y;
  const int j = blockIdx.x * kSimtRows + threadIdx.x;
  const int32_t c0 = a.cu[b], L = a.cu[b + 1] - c0;
  if (j >= L) return;
  const int64_t tj = c0 + j;
  float k[kMaxD], v[kMaxD], dk[kMaxD], dv[kMaxD];
  const float* kp = row_ptr(a, tj, 1, h);
  const float* vp = row_ptr(a, tj, 2, h);
  for (int d = 0; d < a.D; ++d) { k[d] = kp[d]; v[d] = vp[d]; dk[d] = 0.f; dv[d] = 0.f; }
  const float rs = a.rp;
  for (int i = 0; i < L; ++i) {
    const int64_t ti = c0 + i;
    const float* qp = row_ptr(a, ti, 0, h);
    const float* gp = a.dout + (ti * a.H + h) * (int64_t)a.D;
    float s = 0.f, dp = 0.f;
    for (int d = 0; d < a.D; ++d) { s = fmaf(qp[d], k[d], s); dp = fmaf(gp[d], v[d], dp); }
    const float P = expf(s * a.scale - a.lse[(int64_t)h * a.T + ti]);
    const bool kp_ = keep_elem(a, ti, h, j);
    const float pd = kp_ ? P * rs : 0.f;
    dp = kp_ ? dp * rs : 0.f;
    const float ds = P * (dp - a.delta[(int64_t)h * a.T + ti]);
    for (int d = 0; d < a.D; ++d) { dv[d] = fmaf(pd, gp[d], dv[d]); dk[d] = fmaf(ds, qp[d], dk[d]); }
  }
  float* dkp = a.dqkv + ((tj * 3 + 1) * a.H + h) * (int64_t)a.D;
  float* dvp = a.dqkv + ((tj * 3 + 2) * a.H + h) * (int64_t)a.D;
  for (int d = 0; d < a.D; ++d) { dkp[d] = dk[d] * a.scale; dvp[d] = dv[d]; }
}

static SimtArgs make_args(const ub_fmha_params& p) {
  SimtArgs a{};
  a.H = p.heads; a.D = p.head_dim; a.T = p.T; a.scale = p.scale; a.p = p.p_dropout;
  a.thr = p.p_dropout > 0.f ? (uint32_t)floor((double)p.p_dropout * 256.0) : 0u;   // R5: 8-bit decisions
  a.rp = 1.f / (1.f - (float)a.thr / 256.f);
  a.k0 = (uint32_t)(p.seed & 0xFFFFFFFFull); a.k1 = (uint32_t)(p.seed >> 32);
  a.off = (uint32_t)(p.offset & 0xFFFFFFFFull);
  return a;
}

ub_status fmha_fwd_simt(const ub_fmha_params& p, const float* qkv, const int32_t* d_cu, float* out, float* lse,
                        cudaStream_t s) {
  SimtArgs a = make_args(p);
  a.qkv = qkv; a.cu = d_cu; a.out = out; a.lse = lse;
  dim3 grid((p.max_seqlen + kSimtRows - 1) / kSimtRows, p.heads, p.B);
  simt_fwd_kernel<<<grid, kSimtRows, 0, s>>>(a);
  UB_CHECK_LAUNCH();
  return UB_OK;
}

ub_status fmha_bwd_simt(const ub_fmha_params& p, const float* qkv, const float* out, const float* lse,
                        const float* dout, const int32_t* d_cu, float* dqkv, float* delta, cudaStream_t s) {
  SimtArgs a = make_args(p);
  a.qkv = qkv; a.cu = d_cu; a.o = out; a.lse = const_cast<float*>(lse); a.dout = dout; a.dqkv = dqkv; a.delta = delta;
  const int64_t n = p.T * p.heads;
  simt_delta_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a);
  UB_CHECK_LAUNCH();
  dim3 grid((p.max_seqlen + kSimtRows - 1) / kSimtRows, p.heads, p.B);
  simt_dq_kernel<<<grid, kSimtRows, 0, s>>>(a);
  UB_CHECK_LAUNCH();
  simt_dkdv_kernel<<<grid, kSimtRows, 0, s>>>(a);
  UB_CHECK_LAUNCH();
  return UB_OK;
}

}  // namespace ub
