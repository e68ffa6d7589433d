// Attention-dropout keep mask of reading R5, materialised once as bits (an input-only
// operator: it depends on cu_seqlens, the seed and the offset only, so it can run while the
// batch is still being exchanged).  The forward and backward FMHA kernels then read
// 16 / 8 bytes per thread and step instead of running Philox4x32-10 for every 16 probabilities.
//
// R5: key = (seed lo, seed hi), counter = (j >> 4, t, h, offset lo) with t the packed query
// row and j the key index inside the sequence; byte (j & 3) of word ((j & 15) >> 2) >= thr
// keeps (query t, key j).
//
// Two layouts of 32-bit words, MT = ceil(max_seqlen / 128) key (or query) tiles per row, the
// packed row index innermost so that 32 consecutive rows' words are 128 contiguous bytes (the
// writes here and the loads in the kernels are coalesced):
//   query-major  mq[((h * MT + kt) * 4 + w) * T + t_q]: bit e = key kt*128 + 32w + e of query row t_q
//   key-major    mk[((h * MT + it) * 4 + c) * T + t_k]: bit e = query it*128 + 32c + e of key row t_k
// (the forward's softmax thread owns a query row, the backward's compute thread a key row).
// One warp computes a 32 x 32 block: lane l the 32 keep bits of query l (two Philox calls),
// then a five-step shuffle transpose hands lane l the 32 bits of key l.
#include "fmha_common.cuh"

namespace ub {

// One CTA per (sequence b, head h, 32-query chunk qc): its warps take the key chunks kc
// (<= 16 at max_seqlen 512), so the CTAs' work is even (one CTA per sequence would give the
// 512-token sequences 256 blocks and leave most SMs idle behind them).
__global__ void __launch_bounds__(256) dropout_mask_kernel(const int32_t* __restrict__ cu, int32_t H, int64_t T,
                                                           int32_t MT, int32_t MQ, uint32_t k0, uint32_t k1,
                                                           uint32_t off, uint32_t thr, uint32_t* __restrict__ mq,
                                                           uint32_t* __restrict__ mk) {
  pdl_launch_dependents();                        // the forward may be scheduled (it waits for us)
  const int32_t b = blockIdx.x / MQ, qc = blockIdx.x - b * MQ, h = blockIdx.y;
  const int32_t c0 = cu[b], L = cu[b + 1] - c0;
  const int32_t n = (L + 31) / 32;
  if (qc >= n) {
    pdl_wait();
    return;
  }
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  for (int32_t kc = (int32_t)warp; kc < n; kc += (int32_t)(blockDim.x >> 5)) {
    const int32_t q = qc * 32 + (int32_t)lane, j0 = kc * 32;
    const uint32_t t = (uint32_t)(c0 + q);
    uint32_t x = keep_bits16((uint32_t)j0, t, (uint32_t)h, off, k0, k1, thr) |
                 (keep_bits16((uint32_t)j0 + 16u, t, (uint32_t)h, off, k0, k1, thr) << 16);
    if (q < L) mq[((int64_t)h * MT * 4 + kc) * T + c0 + q] = x;          // kc = 4 kt + w
    // 32 x 32 bit transpose: row = lane (query), column = bit (key)  ->  row = key
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
      const uint32_t m = s == 16 ? 0x0000FFFFu : s == 8 ? 0x00FF00FFu : s == 4 ? 0x0F0F0F0Fu : s == 2 ? 0x33333333u
                                                                                                : 0x55555555u;
      const uint32_t y = __shfl_xor_sync(0xffffffffu, x, s);
      x = (lane & (uint32_t)s) ? ((x & ~m) | ((y >> s) & m)) : ((x & m) | ((y & m) << s));
    }
    const int32_t kk = j0 + (int32_t)lane;
    if (kk < L) mk[((int64_t)h * MT * 4 + qc) * T + c0 + kk] = x;        // qc = 4 it + c
  }
  // launched as an overlapping dependent (UB_MASK_OVERLAP_PREVIOUS): finish only after the
  // previous kernel, so that a kernel waiting for this one also waits for that one
  pdl_wait();
}

int32_t mask_tiles(const ub_fmha_params& p) { return (p.max_seqlen + kTile - 1) / kTile; }

size_t dropout_mask_bytes(const ub_fmha_params& p) {
  return 2 * align_up((size_t)p.heads * p.T * mask_tiles(p) * 16, 256);
}

uint32_t dropout_threshold(float p) { return p > 0.f ? (uint32_t)floor((double)p * 256.0) : 0u; }

ub_status launch_dropout_mask(const ub_fmha_params& p, const int32_t* d_cu, void* mask, cudaStream_t s,
                              bool overlap_previous) {
  const int32_t MT = mask_tiles(p);
  uint32_t* mq = static_cast<uint32_t*>(mask);
  uint32_t* mk = reinterpret_cast<uint32_t*>(static_cast<char*>(mask) + dropout_mask_bytes(p) / 2);
  const int32_t MQ = (p.max_seqlen + 31) / 32;
  const int64_t nx = (int64_t)p.B * MQ;
  UB_REQUIRE(nx < (1ll << 31), UB_ERR_UNSUPPORTED, "batch too large for the mask launch");
  const dim3 grid((unsigned)nx, (unsigned)p.heads);
  const uint32_t k0 = (uint32_t)(p.seed & 0xFFFFFFFFull), k1 = (uint32_t)(p.seed >> 32);
  const uint32_t off = (uint32_t)(p.offset & 0xFFFFFFFFull), thr = dropout_threshold(p.p_dropout);
  if (overlap_previous)   // the kernel never waits: it may run beside the previous kernel's tail
    launch_pdl(dropout_mask_kernel, grid, dim3(128), 0, s, d_cu, (int32_t)p.heads, (int64_t)p.T, MT, MQ, k0, k1, off, thr,
               mq, mk);
  else
    dropout_mask_kernel<<<grid, 128, 0, s>>>(d_cu, p.heads, p.T, MT, MQ, k0, k1, off, thr, mq, mk);
  UB_CHECK_LAUNCH();
  return UB_OK;
}

}  // namespace ub

using namespace ub;

extern "C" size_t ub_dropout_mask_bytes(const ub_fmha_params* p) {
  if (!p || p->B < 1 || p->T < 1 || p->heads < 1 || p->max_seqlen < 1) return 0;
  return dropout_mask_bytes(*p);
}

extern "C" ub_status ub_dropout_mask_ex(const ub_fmha_params* p, const int32_t* d_cu, void* d_mask, int32_t flags,
                                       void* stream) {
  clear_error();
  UB_REQUIRE((flags & ~UB_MASK_OVERLAP_PREVIOUS) == 0, UB_ERR_INVALID_ARG, "unknown flag bits 0x%x", flags);
  UB_REQUIRE(p && d_cu && d_mask, UB_ERR_INVALID_ARG, "null pointer");
  UB_REQUIRE(p->B >= 1 && p->T >= 1 && p->heads >= 1 && p->max_seqlen >= 1, UB_ERR_INVALID_ARG, "bad sizes");
  UB_REQUIRE(p->heads <= 65535, UB_ERR_UNSUPPORTED, "heads above 65535");
  UB_REQUIRE(p->p_dropout > 0.f && p->p_dropout < 1.f && dropout_threshold(p->p_dropout) >= 1, UB_ERR_INVALID_ARG,
             "p_dropout %g: the mask needs 1/256 <= p < 1", (double)p->p_dropout);
  UB_REQUIRE(((uintptr_t)d_mask & 15) == 0, UB_ERR_INVALID_ARG, "mask must be 16-B aligned");
  if (ub_status st = require_sm100(); st != UB_OK) return st;
  return launch_dropout_mask(*p, d_cu, d_mask, as_stream(stream), (flags & UB_MASK_OVERLAP_PREVIOUS) != 0);
}

extern "C" ub_status ub_dropout_mask(const ub_fmha_params* p, const int32_t* d_cu, void* d_mask, void* stream) {
  return ub_dropout_mask_ex(p, d_cu, d_mask, 0, stream);
}
