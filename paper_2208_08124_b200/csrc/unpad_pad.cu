// Unpad (gather) and pad (scatter) between padded [B, S, row] and packed
// [T, row] rows, plus the exchange copy kernel (P:355-359 redistribution).
//
// HBM-bound byte movers.  Every thread walks the PADDED index space (B*S rows x V vectors,
// V = row_bytes / elem) with a grid-stride loop: padded-side accesses are perfectly
// coalesced, packed-side accesses are contiguous within each row.  Row -> (b, i) uses
// multiply-high division (no integer divide on the hot loop).  16-B vectors when the
// row and both base pointers allow it.
#include <algorithm>
#include <cstdlib>

#include "sm100.cuh"
#include "ub_internal.h"

namespace ub {

struct FastDiv {  // q = n / d for 32-bit n (Granlund-Montgomery round-up method)
  uint32_t d, m, s;
  __host__ explicit FastDiv(uint32_t d_ = 1) : d(d_) {
    s = 0;
    while ((1ull << s) < d) ++s;
    m = (uint32_t)((((1ull << s) - d) << 32) / d + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    return (uint32_t)(((uint64_t)__umulhi(n, m) + n) >> s);
  }
};

template <typename Vec, bool kPad>
__global__ void __launch_bounds__(256) unpad_pad_kernel(const Vec* __restrict__ src, Vec* __restrict__ dst,
                                                         const int32_t* __restrict__ cu, const Vec* __restrict__ pad_row,
                                                         uint32_t n, FastDiv divV, FastDiv divS) {
  constexpr int U = 4;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x + threadIdx.x; base < n; base += stride * U) {
    Vec val[U];
    int64_t dst_idx[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t f = base + u * stride;
      dst_idx[u] = -1;
      if (f < n) {
        const uint32_t p = divV.div(f), v = f - p * divV.d;      // padded row p, vector v
        const uint32_t b = divS.div(p), i = p - b * divS.d;      // sequence b, position i
        const int32_t c0 = __ldg(cu + b), L = __ldg(cu + b + 1) - c0;
        const int64_t packed_idx = ((int64_t)c0 + i) * divV.d + v;
        if constexpr (kPad) {
          dst_idx[u] = f;
          if ((int32_t)i < L) val[u] = src[packed_idx];
          else if (pad_row) val[u] = __ldg(pad_row + v);
          else val[u] = Vec{};
        } else if ((int32_t)i < L) {
          val[u] = src[f];
          dst_idx[u] = packed_idx;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (dst_idx[u] >= 0) dst[dst_idx[u]] = val[u];
  }
}

// Contiguous-span form for 16-B-aligned rows.  Within sequence b the packed and padded
// layouts differ by a constant shift: packed vector q <-> padded vector q + delta_b with
// delta_b = (b*S - cu[b]) * V (V = 16-B vectors per row).  So unpad / pad are B contiguous
// copies, and pad's zero fill is B contiguous runs whose prefix offsets are the same delta_b.
// Each CTA takes a fixed span of the packed (or zero) vector space, finds its first
// sequence by one binary search, and streams 16-B vectors with several loads in flight.
#ifndef UB_SPAN_UNROLL
#define UB_SPAN_UNROLL 4
#endif
#ifndef UB_SPAN_ITERS
#define UB_SPAN_ITERS 1
#endif
#ifndef UB_SPAN_THREADS
#define UB_SPAN_THREADS 256
#endif
constexpr int kSpanThreads = UB_SPAN_THREADS;
constexpr int kSpanUnroll = UB_SPAN_UNROLL;           // 16-B loads in flight per thread
// 16 KB per CTA: measured on the config-2 hidden state (B200, 3 rotating buffer sets) against
// 64 KB per CTA: unpad 13.8 -> 12.1 us (0.75 of HBM; torch's own copy of the packed tensor:
// 12.4 us), pad 17.6 -> 16.1 us (0.84); 8 loads in flight or 512 threads per CTA were slower
constexpr int64_t kSpanVecs = (int64_t)kSpanThreads * kSpanUnroll * UB_SPAN_ITERS;   // 16-B vectors per CTA

__device__ __forceinline__ int32_t seq_of(const int32_t* __restrict__ cu, int32_t B, int64_t key, int64_t V, int32_t S,
                                          bool zero_space) {
  // largest b with start_b <= key; start_b = cu[b]*V (packed space) or (b*S - cu[b])*V (zero space)
  int32_t lo = 0, hi = B - 1;
  while (lo < hi) {
    const int32_t mid = (lo + hi + 1) >> 1;
    const int64_t st = zero_space ? ((int64_t)mid * S - __ldg(cu + mid)) * V : (int64_t)__ldg(cu + mid) * V;
    if (st <= key) lo = mid; else hi = mid - 1;
  }
  return lo;
}

template <bool kPad>
__global__ void __launch_bounds__(kSpanThreads) span_copy_kernel(const int4* __restrict__ src, int4* __restrict__ dst,
                                                                 const int32_t* __restrict__ cu, const int4* __restrict__ pad_row,
                                                                 int32_t B, int32_t S, int64_t V, int64_t n_copy,
                                                                 int64_t n_zero, int32_t copy_ctas) {
  pdl_launch_dependents();
  pdl_wait();                                      // the source rows may come from the previous kernel
  const bool zero = kPad && (int32_t)blockIdx.x >= copy_ctas;
  const int64_t n = zero ? n_zero : n_copy;
  const int64_t beg = (int64_t)(zero ? blockIdx.x - copy_ctas : blockIdx.x) * kSpanVecs;
  const int64_t end = min(beg + kSpanVecs, n);
  if (beg >= end) return;
  __shared__ int32_t s_b;
  if (threadIdx.x == 0) s_b = seq_of(cu, B, beg, V, S, zero);
  __syncthreads();
  int32_t b = s_b;
  int64_t q = beg;
  while (q < end) {
    // skip empty runs (zero-length sequence, or a full sequence in the zero space)
    int64_t seg_end, shift;
    const int64_t c0 = __ldg(cu + b), c1 = __ldg(cu + b + 1);
    if (!zero) {
      seg_end = min(end, c1 * V);
      shift = ((int64_t)b * S - c0) * V;                      // padded = packed + shift
    } else {
      seg_end = min(end, ((int64_t)(b + 1) * S - c1) * V);
      shift = ((int64_t)b * S + (c1 - c0)) * V - ((int64_t)b * S - c0) * V;   // padded = zero index + shift
    }
    for (int64_t i0 = q + threadIdx.x; i0 < seg_end; i0 += (int64_t)kSpanThreads * kSpanUnroll) {
      int4 v[kSpanUnroll];
#pragma unroll
      for (int u = 0; u < kSpanUnroll; ++u) {
        const int64_t i = i0 + (int64_t)u * kSpanThreads;
        if (i < seg_end) {
          if (zero) v[u] = pad_row ? __ldg(pad_row + (i + shift) % V) : make_int4(0, 0, 0, 0);
          else v[u] = kPad ? __ldcs(src + i) : __ldcs(src + i + shift);
        }
      }
#pragma unroll
      for (int u = 0; u < kSpanUnroll; ++u) {
        const int64_t i = i0 + (int64_t)u * kSpanThreads;
        if (i < seg_end) {
          if (zero || kPad) __stcs(dst + i + shift, v[u]);
          else __stcs(dst + i, v[u]);
        }
      }
    }
    q = seg_end;
    ++b;
  }
}

// TMA form of the span copy: a CTA moves one kBulkBytes chunk of the packed (or zero) byte
// space through shared memory with 1-D bulk copies -- one load per sequence segment in the
// chunk, completing on one mbarrier, then one store per segment -- so a handful of
// instructions keep 32 KB in flight per CTA (6 CTAs per SM).  Pad's zero space stores from a
// zeroed buffer.
#ifndef UB_BULK_BYTES
#define UB_BULK_BYTES 32768
#endif
constexpr int64_t kBulkBytes = UB_BULK_BYTES;
template <bool kPad>
__global__ void __launch_bounds__(128) span_bulk_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                                        const int32_t* __restrict__ cu, int32_t B, int32_t S, int64_t row,
                                                        int64_t n_copy, int64_t n_zero, int32_t copy_ctas) {
  __shared__ __align__(128) uint8_t buf[kBulkBytes];
  __shared__ uint64_t bar;
  pdl_launch_dependents();
  pdl_wait();                                      // the source rows may come from the previous kernel
  // CTAs [0, copy_ctas) walk the copy chunks, the others the zero chunks (pad), chunk-strided
  const bool zero = kPad && (int32_t)blockIdx.x >= copy_ctas;
  const int64_t n = zero ? n_zero : n_copy;
  const int64_t c0 = zero ? blockIdx.x - copy_ctas : blockIdx.x, dc = zero ? gridDim.x - copy_ctas : copy_ctas;
  if (c0 * kBulkBytes >= n) return;
  if (zero) {
    for (int64_t i = threadIdx.x * 16; i < kBulkBytes; i += 128 * 16) st_shared_v4(smem_u32(buf + i), 0, 0, 0, 0);
    fence_proxy_async_smem();
  } else if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t it = 0;
  for (int64_t c = c0; c * kBulkBytes < n; c += dc, ++it) {
    const int64_t beg = c * kBulkBytes, end = min(beg + kBulkBytes, n);
    // segments of [beg, end) per sequence: packed bytes of b are [cu[b], cu[b+1]) * row, its
    // zero bytes [(b S - cu[b]), ((b+1) S - cu[b+1])) * row; padded = space index + shift
    const int32_t b0 = seq_of(cu, B, beg / 16, row / 16, S, zero);
    if (!zero) {
      bulk_wait_group_read0();                     // the previous chunk's stores have read buf
      mbar_expect_tx(&bar, (uint32_t)(end - beg));
      for (int64_t q = beg, bb = b0; q < end; ++bb) {
        const int64_t x0 = __ldg(cu + bb), x1 = __ldg(cu + bb + 1);
        const int64_t seg_end = min(end, x1 * row);
        if (seg_end > q) bulk_load_1d(buf + (q - beg), src + (kPad ? q : q + (bb * S - x0) * row), (uint32_t)(seg_end - q), &bar);
        q = max(q, seg_end);
      }
      mbar_wait(&bar, it & 1);
    }
    for (int64_t q = beg, bb = b0; q < end; ++bb) {
      const int64_t x0 = __ldg(cu + bb), x1 = __ldg(cu + bb + 1);
      int64_t seg_end, shift;
      if (!zero) {
        seg_end = min(end, x1 * row);
        shift = (bb * S - x0) * row;
      } else {
        seg_end = min(end, ((bb + 1) * S - x1) * row);
        shift = (bb * S + (x1 - x0)) * row - (bb * S - x0) * row;
      }
      if (seg_end > q)
        bulk_store_1d(dst + ((zero || kPad) ? q + shift : q), buf + (zero ? 0 : q - beg), (uint32_t)(seg_end - q));
      q = max(q, seg_end);
    }
    bulk_commit_group();
  }
  bulk_wait_group_read0();                         // smem must outlive the stores' reads
}

static ub_status launch_span(bool pad, const void* src, void* dst, const int32_t* d_cu, const void* pad_row, int32_t B,
                             int32_t S, int64_t T, int64_t row_bytes, cudaStream_t s) {
  const int64_t V = row_bytes / 16;
  const int64_t n_copy = T * V, n_zero = pad ? ((int64_t)B * S - T) * V : 0;
  const int64_t cc = (n_copy + kSpanVecs - 1) / kSpanVecs, zc = (n_zero + kSpanVecs - 1) / kSpanVecs;
  UB_REQUIRE(cc + zc < (1ll << 31), UB_ERR_UNSUPPORTED, "tensor too large for one launch");
  if (cc + zc == 0) return UB_OK;
  const int pk = pad ? kProfPad : kProfUnpad;
  // TMA bulk copies unless a pad row pattern is given (or UB_SPAN_BULK=0 selects the vector
  // kernel, kept as the measured alternative): config-2 hidden state back to back, unpad
  // 12.2 -> 11.8 us (0.77 of HBM), pad 16.1 -> 14.9 us (0.91)
  static const bool bulk = [] { const char* e = std::getenv("UB_SPAN_BULK"); return !(e && e[0] == '0'); }();
  if (bulk && !pad_row) {
    const int64_t nb = T * row_bytes, zb = pad ? ((int64_t)B * S - T) * row_bytes : 0;
    // one chunk per CTA (a grid of at most one wave with each CTA striding over several
    // chunks measured slower: unpad 11.8 -> 12.1 us, pad 14.9 -> 18.1 us -- a CTA's chunks
    // serialise on its one buffer)
    const int64_t bc = (nb + kBulkBytes - 1) / kBulkBytes, bz = (zb + kBulkBytes - 1) / kBulkBytes;
    prof_record(pk, 0, s);
    if (pad)
      launch_pdl(span_bulk_kernel<true>, dim3((unsigned)(bc + bz)), dim3(128), 0, s, static_cast<const uint8_t*>(src),
                 static_cast<uint8_t*>(dst), d_cu, B, S, row_bytes, nb, zb, (int32_t)bc);
    else
      launch_pdl(span_bulk_kernel<false>, dim3((unsigned)bc), dim3(128), 0, s, static_cast<const uint8_t*>(src),
                 static_cast<uint8_t*>(dst), d_cu, B, S, row_bytes, nb, (int64_t)0, (int32_t)bc);
    UB_CHECK_LAUNCH();
    prof_record(pk, 1, s);
    return UB_OK;
  }
  prof_record(pk, 0, s);
  if (pad)
    launch_pdl(span_copy_kernel<true>, dim3((unsigned)(cc + zc)), dim3(kSpanThreads), 0, s, static_cast<const int4*>(src),
               static_cast<int4*>(dst), d_cu, static_cast<const int4*>(pad_row), B, S, V, n_copy, n_zero, (int32_t)cc);
  else
    launch_pdl(span_copy_kernel<false>, dim3((unsigned)cc), dim3(kSpanThreads), 0, s, static_cast<const int4*>(src),
               static_cast<int4*>(dst), d_cu, static_cast<const int4*>(nullptr), B, S, V, n_copy, (int64_t)0, (int32_t)cc);
  UB_CHECK_LAUNCH();
  prof_record(pk, 1, s);
  return UB_OK;
}

template <typename Vec>
static ub_status launch_unpad_pad(bool pad, const void* src, void* dst, const int32_t* d_cu, const void* pad_row,
                                  int32_t B, int32_t S, int64_t row_bytes, cudaStream_t s) {
  const uint64_t V = row_bytes / sizeof(Vec);
  const uint64_t n64 = (uint64_t)B * S * V;
  UB_REQUIRE(n64 < (1ull << 32) - 1, UB_ERR_UNSUPPORTED, "padded tensor too large for one launch (%llu elems)",
             (unsigned long long)n64);
  const uint32_t n = (uint32_t)n64;
  if (n == 0) return UB_OK;
  const int threads = 256;
  const uint64_t want = (n64 + threads * 4 - 1) / (threads * 4);
  const int blocks = (int)(want < 148ull * 16 ? (want ? want : 1) : 148ull * 16);
  FastDiv dv((uint32_t)V), ds((uint32_t)S);
  const int pk = pad ? kProfPad : kProfUnpad;
  prof_record(pk, 0, s);
  if (pad)
    unpad_pad_kernel<Vec, true><<<blocks, threads, 0, s>>>(static_cast<const Vec*>(src), static_cast<Vec*>(dst), d_cu,
                                                          static_cast<const Vec*>(pad_row), n, dv, ds);
  else
    unpad_pad_kernel<Vec, false><<<blocks, threads, 0, s>>>(static_cast<const Vec*>(src), static_cast<Vec*>(dst), d_cu,
                                                           nullptr, n, dv, ds);
  UB_CHECK_LAUNCH();
  prof_record(pk, 1, s);
  return UB_OK;
}

static ub_status unpad_pad_dispatch(bool pad, const void* src, void* dst, const int32_t* d_cu, const void* pad_row,
                                    int32_t B, int32_t S, int64_t T, int64_t row_bytes, void* stream) {
  clear_error();
  UB_REQUIRE(src && dst && d_cu, UB_ERR_INVALID_ARG, "null pointer");
  UB_REQUIRE(B >= 1 && S >= 1, UB_ERR_INVALID_ARG, "empty batch");
  UB_REQUIRE(row_bytes > 0, UB_ERR_SHAPE, "row_bytes <= 0");
  UB_REQUIRE(T >= 0 && T <= (int64_t)B * S, UB_ERR_CAPACITY, "T=%lld exceeds B*S", (long long)T);
  const uintptr_t al = (uintptr_t)src | (uintptr_t)dst | (uintptr_t)(pad_row ? pad_row : dst);
  cudaStream_t s = as_stream(stream);
  if (ub_status st = checked_cu(d_cu, B, S, T, s); st != UB_OK) return st;
  if (row_bytes % 16 == 0 && (al & 15) == 0) return launch_span(pad, src, dst, d_cu, pad_row, B, S, T, row_bytes, s);
  if (row_bytes % 4 == 0 && (al & 3) == 0)
    return launch_unpad_pad<uint32_t>(pad, src, dst, d_cu, pad_row, B, S, row_bytes, s);
  return launch_unpad_pad<uint8_t>(pad, src, dst, d_cu, pad_row, B, S, row_bytes, s);
}

// ------------------------------------------------------------------ exchange copy
// One CTA (or gridDim.y CTAs) per table entry: copies len*rec bytes of token records and srec bytes of the
// sample record.  tab = {src_tok[B], len[B], dst_tok[B], src_smp[B], dst_smp[B]} (row stride B, gridDim.x
// entries).  Gather form (the exchange's final reorder): a sixth row sel[B] picks the source per entry
// (0: st / ss, 1: st_b / ss_b -- this rank's own packed samples vs the receive buffer), and CTA (0, 0)
// also copies ncu int32 from cu_src to cu_dst (the new cu_seqlens staged with the tables).
template <typename Vec>
__global__ void __launch_bounds__(256) exchange_copy_kernel(const uint8_t* __restrict__ st, const uint8_t* __restrict__ st_b,
                                                            uint8_t* __restrict__ dt, const uint8_t* __restrict__ ss,
                                                            const uint8_t* __restrict__ ss_b, uint8_t* __restrict__ ds,
                                                            const int64_t* __restrict__ tab, const int64_t* __restrict__ sel,
                                                            int32_t B, int64_t rec, int64_t srec,
                                                            const int32_t* __restrict__ cu_src, int32_t* __restrict__ cu_dst,
                                                            int32_t ncu) {
  const int e = blockIdx.x;
  if (cu_dst != nullptr && e == 0 && blockIdx.y == 0)
    for (int32_t i = threadIdx.x; i < ncu; i += blockDim.x) cu_dst[i] = cu_src[i];
  const int64_t src_tok = tab[e], len = tab[B + e], dst_tok = tab[2 * B + e];
  const bool alt = sel != nullptr && sel[e] != 0;
  const Vec* s = reinterpret_cast<const Vec*>((alt ? st_b : st) + src_tok * rec);
  Vec* d = reinterpret_cast<Vec*>(dt + dst_tok * rec);
  const int64_t nv = len * rec / (int64_t)sizeof(Vec);
  // gridDim.y CTAs share an entry (large records): interleaved 256-vector blocks
  for (int64_t i = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.y * blockDim.x)
    d[i] = s[i];
  if (srec > 0 && blockIdx.y == 0) {
    const uint8_t* sp = alt ? ss_b : ss;
    const int64_t so = tab[3 * B + e] * srec, dso = tab[4 * B + e] * srec;
    for (int64_t i = threadIdx.x; i < srec; i += blockDim.x) ds[dso + i] = sp[so + i];
  }
}

ub_status exchange_gather(const void* src_a, const void* src_b, void* dst, const void* ssrc_a, const void* ssrc_b,
                          void* sdst, const int64_t* d_tab, const int64_t* d_sel, int32_t n, int32_t B, int64_t rec,
                          int64_t srec, const int32_t* cu_src, int32_t* cu_dst, int32_t ncu, cudaStream_t s) {
  if (n <= 0 && cu_dst == nullptr) return UB_OK;
  const uintptr_t al = (uintptr_t)src_a | (uintptr_t)(src_b ? src_b : src_a) | (uintptr_t)dst;
  auto* sa = static_cast<const uint8_t*>(src_a);
  auto* sb = static_cast<const uint8_t*>(src_b);
  auto* dt = static_cast<uint8_t*>(dst);
  auto* ssa = static_cast<const uint8_t*>(ssrc_a);
  auto* ssb = static_cast<const uint8_t*>(ssrc_b);
  auto* ds = static_cast<uint8_t*>(sdst);
  const dim3 grid(n > 0 ? n : 1, rec >= 256 ? 16 : 1);     // large records: 16 CTAs per entry
  if (n <= 0) {                                           // nothing to move: only the cu copy
    exchange_copy_kernel<uint8_t><<<1, 256, 0, s>>>(sa, sb, dt, ssa, ssb, ds, d_tab, nullptr, B, 0, 0, cu_src, cu_dst, ncu);
  } else if (rec % 16 == 0 && (al & 15) == 0) {
    exchange_copy_kernel<int4><<<grid, 256, 0, s>>>(sa, sb, dt, ssa, ssb, ds, d_tab, d_sel, B, rec, srec, cu_src, cu_dst, ncu);
  } else if (rec % 4 == 0 && (al & 3) == 0) {
    exchange_copy_kernel<uint32_t><<<grid, 256, 0, s>>>(sa, sb, dt, ssa, ssb, ds, d_tab, d_sel, B, rec, srec, cu_src, cu_dst,
                                                        ncu);
  } else {
    exchange_copy_kernel<uint8_t><<<grid, 256, 0, s>>>(sa, sb, dt, ssa, ssb, ds, d_tab, d_sel, B, rec, srec, cu_src, cu_dst,
                                                       ncu);
  }
  UB_CHECK_LAUNCH();
  return UB_OK;
}

}  // namespace ub

using namespace ub;

extern "C" ub_status ub_unpad(const void* padded, void* packed, const int32_t* d_cu, int32_t B, int32_t S,
                              int64_t T, int64_t row_bytes, void* stream) {
  return unpad_pad_dispatch(false, padded, packed, d_cu, nullptr, B, S, T, row_bytes, stream);
}

extern "C" ub_status ub_pad(const void* packed, void* padded, const int32_t* d_cu, int32_t B, int32_t S, int64_t T,
                            int64_t row_bytes, const void* d_pad_row, void* stream) {
  return unpad_pad_dispatch(true, packed, padded, d_cu, d_pad_row, B, S, T, row_bytes, stream);
}

extern "C" ub_status ub_exchange_copy(const void* src_tokens, void* dst_tokens, const void* src_samples,
                                      void* dst_samples, const int64_t* d_tab, int32_t B, int64_t rec_bytes,
                                      int64_t srec_bytes, void* stream) {
  clear_error();
  UB_REQUIRE(src_tokens && dst_tokens && d_tab, UB_ERR_INVALID_ARG, "null pointer");
  UB_REQUIRE(B >= 1 && rec_bytes > 0 && srec_bytes >= 0, UB_ERR_SHAPE, "bad sizes");
  UB_REQUIRE(srec_bytes == 0 || (src_samples && dst_samples), UB_ERR_INVALID_ARG, "null sample pointer");
  if (ub_status st = exchange_gather(src_tokens, nullptr, dst_tokens, src_samples, nullptr, dst_samples, d_tab, nullptr, B, B,
                                     rec_bytes, srec_bytes, nullptr, nullptr, 0, as_stream(stream));
      st != UB_OK)
    return st;
  UB_CHECK_LAUNCH();
  return UB_OK;
}
