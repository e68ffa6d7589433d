// Cross-rank token rebalancing over NCCL (NVLink 5 / NVSwitch): all-gather of the valid
// lengths + all-to-all-v of packed samples, replacing the paper's all-gather of five
// padded tensors and its CPU/MPI variant.
//
// Only lengths cross the fabric before the plan is known (W*B int32); each sample's
// token records then move exactly once (P:359's slice is realised as a grouped
// ncclSend/ncclRecv phase).  Everything is enqueued on the caller's side stream so that
// step n+1's exchange overlaps step n's compute.
#include <nccl.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ub_internal.h"

namespace ub {

constexpr int32_t kExSlots = UB_EXCHANGE_SLOTS + 1;  // the last one serves ub_balance_exchange

struct Comm {
  ncclComm_t nccl = nullptr;
  int32_t W = 0, rank = 0;
  // pinned host staging.  h_all: kExSlots rings of W*cap_B lengths, each filled by a begin
  // and guarded by ev_len[slot].  The plan tables / cu are rewritten by every finish only
  // after ev_staging (behind the previous finish's H2D copies) has fired.
  int32_t* h_all = nullptr;
  int64_t* h_stage = nullptr;         // tables + new cu_seqlens, one H2D per finish (stage_words(B) int64)
  int32_t cap_B = 0;
  int32_t slot_B[kExSlots] = {};      // B of the pending begin, 0 = free
  cudaEvent_t ev_len[kExSlots] = {};
  cudaEvent_t ev_staging = nullptr;
  // UB_EXCHANGE_TRACE=1: host time per finish phase, printed at ub_comm_destroy (dev aid)
  bool trace = false;
  // UB_COMM_FORCE_NCCL (ub_comm_set_options / UB_EXCHANGE_FORCE_NCCL=1): the self chunk and
  // the one-rank all-gather go through NCCL too (ncclAllGather, ncclSend/ncclRecv to self)
  // instead of device copies, so the collective data plane runs on a one-GPU box
  bool force_nccl = false;
  int64_t nccl_ops = 0;               // NCCL collectives / point-to-point calls issued (ub_comm_nccl_ops)
  double t_phase[8] = {};
  int64_t n_finish = 0;
};

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

#define UB_CHECK_NCCL(expr)                                                                  \
  do {                                                                                       \
    ncclResult_t r_ = (expr);                                                                \
    if (r_ != ncclSuccess)                                                                   \
      return ::ub::set_error(UB_ERR_NCCL, "%s: %s", #expr, ncclGetErrorString(r_));          \
  } while (0)

// staged per finish: pack table [5B] | gather table [6B] | new cu_seqlens [B+1] int32 (padded to int64)
static size_t stage_words(int32_t B) { return (size_t)11 * B + ((size_t)B + 2) / 2; }

static void free_staging(Comm* c) {
  cudaFreeHost(c->h_all);
  cudaFreeHost(c->h_stage);
  c->h_all = nullptr; c->h_stage = nullptr; c->cap_B = 0;
}

static ub_status ensure_staging(Comm* c, int32_t B) {
  if (!c->ev_staging) {
    for (auto& e : c->ev_len) UB_CHECK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    UB_CHECK_CUDA(cudaEventCreateWithFlags(&c->ev_staging, cudaEventDisableTiming));
  }
  if (c->cap_B >= B) return UB_OK;
  // growing: wait for every pending copy into / out of the old buffers, keep pending slots
  for (auto& e : c->ev_len) UB_CHECK_CUDA(cudaEventSynchronize(e));
  UB_CHECK_CUDA(cudaEventSynchronize(c->ev_staging));
  int32_t* old_all = c->h_all;
  const int32_t old_cap = c->cap_B;
  c->h_all = nullptr;
  free_staging(c);
  UB_CHECK_CUDA(cudaMallocHost(&c->h_all, sizeof(int32_t) * (size_t)kExSlots * c->W * B));
  UB_CHECK_CUDA(cudaMallocHost(&c->h_stage, sizeof(int64_t) * stage_words(B)));
  if (old_all) {
    for (int32_t k = 0; k < kExSlots; ++k)
      if (c->slot_B[k])
        std::memcpy(c->h_all + (size_t)k * c->W * B, old_all + (size_t)k * c->W * old_cap,
                    sizeof(int32_t) * (size_t)c->W * c->slot_B[k]);
    cudaFreeHost(old_all);
  }
  c->cap_B = B;
  return UB_OK;
}

struct ExWs {  // carve-up of the exchange workspace
  int32_t* all_lengths; int64_t* stage;
  uint8_t* send_tok; uint8_t* recv_tok; uint8_t* send_smp; uint8_t* recv_smp;
};
static size_t ex_layout(int32_t W, int32_t B, int64_t cap, int64_t rec, int64_t srec, void* base, ExWs* out) {
  size_t off = 0;
  auto take = [&](size_t n) { size_t o = off; off = align_up(off + n, 256); return o; };
  const size_t o_all = take(sizeof(int32_t) * (size_t)kExSlots * W * B);  // one gather target per slot
  const size_t o_tp = take(sizeof(int64_t) * stage_words(B));
  const size_t o_st = take((size_t)cap * rec);
  const size_t o_rt = take((size_t)cap * rec);
  const size_t o_ss = take((size_t)B * srec);
  const size_t o_rs = take((size_t)B * srec);
  if (out && base) {
    char* b = static_cast<char*>(base);
    out->all_lengths = reinterpret_cast<int32_t*>(b + o_all);
    out->stage = reinterpret_cast<int64_t*>(b + o_tp);
    out->send_tok = reinterpret_cast<uint8_t*>(b + o_st);
    out->recv_tok = reinterpret_cast<uint8_t*>(b + o_rt);
    out->send_smp = reinterpret_cast<uint8_t*>(b + o_ss);
    out->recv_smp = reinterpret_cast<uint8_t*>(b + o_rs);
  }
  return off;
}

}  // namespace ub

using namespace ub;

extern "C" ub_status ub_comm_unique_id(void* out_id_128) {
  clear_error();
  UB_REQUIRE(out_id_128, UB_ERR_INVALID_ARG, "null pointer");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  UB_CHECK_NCCL(ncclGetUniqueId(&id));
  std::memcpy(out_id_128, &id, sizeof(id));
  return UB_OK;
}

extern "C" ub_status ub_comm_init(void** out_comm, const void* id_128, int32_t W, int32_t rank) {
  clear_error();
  UB_REQUIRE(out_comm && id_128, UB_ERR_INVALID_ARG, "null pointer");
  UB_REQUIRE(W >= 1 && rank >= 0 && rank < W, UB_ERR_INVALID_ARG, "bad W/rank");
  ncclUniqueId id;
  std::memcpy(&id, id_128, sizeof(id));
  Comm* c = new Comm();
  const char* tr = std::getenv("UB_EXCHANGE_TRACE");
  c->trace = tr && tr[0] == '1';
  const char* fn = std::getenv("UB_EXCHANGE_FORCE_NCCL");
  c->force_nccl = fn && fn[0] == '1';
  c->W = W;
  c->rank = rank;
  ncclResult_t r = ncclCommInitRank(&c->nccl, W, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return set_error(UB_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  *out_comm = c;
  return UB_OK;
}

extern "C" ub_status ub_comm_destroy(void* comm) {
  clear_error();
  if (!comm) return UB_OK;
  Comm* c = static_cast<Comm*>(comm);
  if (c->trace && c->n_finish) {
    static const char* names[] = {"wait_lengths", "plan", "wait_staging", "tables", "pack", "nccl_p2p", "unpack_cu"};
    std::fprintf(stderr, "[ub exchange trace] rank %d, %lld finishes, host us per finish:", c->rank,
                 (long long)c->n_finish);
    for (int k = 0; k < 7; ++k) std::fprintf(stderr, " %s=%.1f", names[k], c->t_phase[k] / c->n_finish);
    std::fprintf(stderr, "\n");
  }
  for (auto e : c->ev_len)
    if (e) cudaEventSynchronize(e);
  if (c->ev_staging) cudaEventSynchronize(c->ev_staging);
  if (c->nccl) ncclCommDestroy(c->nccl);
  free_staging(c);
  for (auto e : c->ev_len)
    if (e) cudaEventDestroy(e);
  if (c->ev_staging) cudaEventDestroy(c->ev_staging);
  delete c;
  return UB_OK;
}

extern "C" ub_status ub_comm_set_options(void* comm, int32_t flags) {
  clear_error();
  UB_REQUIRE(comm, UB_ERR_INVALID_ARG, "null comm");
  UB_REQUIRE((flags & ~(UB_COMM_FORCE_NCCL | UB_COMM_HOST_PROFILE)) == 0, UB_ERR_INVALID_ARG,
             "unknown option bits 0x%x", flags);
  Comm* c = static_cast<Comm*>(comm);
  c->force_nccl = (flags & UB_COMM_FORCE_NCCL) != 0;
  if ((flags & UB_COMM_HOST_PROFILE) != 0 && !c->trace) {
    c->trace = true;                                   // restart the accumulation
    for (double& t : c->t_phase) t = 0.0;
    c->n_finish = 0;
  } else if ((flags & UB_COMM_HOST_PROFILE) == 0) {
    c->trace = false;
  }
  return UB_OK;
}

extern "C" ub_status ub_comm_host_profile(void* comm, double* out_us, int32_t n_out, int64_t* out_finishes) {
  clear_error();
  UB_REQUIRE(comm && out_us && out_finishes && n_out >= 1, UB_ERR_INVALID_ARG, "null pointer");
  const Comm* c = static_cast<const Comm*>(comm);
  for (int32_t k = 0; k < n_out; ++k) out_us[k] = k < 7 ? c->t_phase[k] : 0.0;
  *out_finishes = c->n_finish;
  return UB_OK;
}

extern "C" ub_status ub_comm_nccl_ops(void* comm, int64_t* out) {
  clear_error();
  UB_REQUIRE(comm && out, UB_ERR_INVALID_ARG, "null pointer");
  *out = static_cast<Comm*>(comm)->nccl_ops;
  return UB_OK;
}

extern "C" ub_status ub_allgather_lengths(void* comm, const int32_t* d_my, int32_t* d_all, int32_t B, void* stream) {
  clear_error();
  UB_REQUIRE(comm && d_my && d_all && B >= 1, UB_ERR_INVALID_ARG, "bad args");
  Comm* c = static_cast<Comm*>(comm);
  UB_CHECK_NCCL(ncclAllGather(d_my, d_all, (size_t)B, ncclInt32, c->nccl, as_stream(stream)));
  ++c->nccl_ops;
  return UB_OK;
}

extern "C" size_t ub_exchange_workspace_bytes(int32_t W, int32_t B, int64_t cap, int64_t rec, int64_t srec) {
  if (W < 1 || B < 1 || cap < 0 || rec < 0 || srec < 0) return 0;
  return ex_layout(W, B, cap, rec, srec, nullptr, nullptr);
}

static ub_status exchange_begin(Comm* c, int32_t slot, int32_t B, const int32_t* d_my_lengths, void* ws,
                                cudaStream_t s) {
  UB_REQUIRE(c->slot_B[slot] == 0, UB_ERR_INVALID_ARG, "exchange slot %d already holds an unfinished begin", slot);
  ub_status st = ensure_staging(c, B);
  if (st != UB_OK) return st;
  const size_t n = (size_t)c->W * B;
  int32_t* d_all = static_cast<int32_t*>(ws) + (size_t)slot * n;   // ex_layout: lengths at the front
  // 1. all-gather of lengths (P:355 step 1, lengths only), 2. D2H into the pinned ring
  // (one rank: the gather is the identity, no collective unless forced)
  const bool gather = c->W > 1 || c->force_nccl;
  if (gather) {
    UB_CHECK_NCCL(ncclAllGather(d_my_lengths, d_all, (size_t)B, ncclInt32, c->nccl, s));
    ++c->nccl_ops;
  }
  UB_CHECK_CUDA(cudaMemcpyAsync(c->h_all + (size_t)slot * c->W * c->cap_B, gather ? d_all : d_my_lengths,
                                sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
  UB_CHECK_CUDA(cudaEventRecord(c->ev_len[slot], s));
  c->slot_B[slot] = B;
  return UB_OK;
}

static ub_status exchange_finish(Comm* c, int32_t slot, int32_t mode, int32_t B, int32_t max_seqlen,
                                 const void* d_my_tokens, const void* d_my_samples, int64_t rec, int64_t srec,
                                 int64_t cap, void* d_out_tokens, void* d_out_samples, int32_t* d_out_cu,
                                 int32_t* h_perm, int64_t* h_out_T, void* ws, cudaStream_t s) {
  UB_REQUIRE(c->slot_B[slot] == B, UB_ERR_INVALID_ARG, "exchange slot %d: no begin with B=%d pending", slot, B);
  const int32_t W = c->W, me = c->rank;
  ExWs w;
  ex_layout(W, B, cap, rec, srec, ws, &w);
  double tp[9];
  int ip = 0;
  if (c->trace) tp[ip++] = now_us();
#define UB_PHASE() do { if (c->trace) tp[ip++] = now_us(); } while (0)
  // the single host wait: this slot's lengths (enqueued by the begin, normally long done)
  UB_CHECK_CUDA(cudaEventSynchronize(c->ev_len[slot]));
  UB_PHASE();
  c->slot_B[slot] = 0;
  const int32_t* h_all = c->h_all + (size_t)slot * W * c->cap_B;
  // 3. the deterministic plan, identical on every rank
  std::vector<int32_t> perm((size_t)W * B);
  ub_status st;
  if ((st = ub_balance_plan(h_all, W, B, max_seqlen, mode, perm.data(), nullptr, nullptr, nullptr)) != UB_OK)
    return st;
  UB_PHASE();
  // the previous finish's H2D copies out of the staging buffers must have completed
  UB_CHECK_CUDA(cudaEventSynchronize(c->ev_staging));
  UB_PHASE();
  std::vector<int64_t> send_cnt(W, 0), send_scnt(W, 0), recv_cnt(W, 0), recv_scnt(W, 0);
  const bool self_nccl = c->force_nccl;
  int64_t* hp = c->h_stage;                               // pack table, stride B
  int64_t* hu = c->h_stage + (size_t)5 * B;               // gather table, stride B, 6 rows
  int32_t* hcu = reinterpret_cast<int32_t*>(c->h_stage + (size_t)11 * B);
  int32_t n_pack = 0;
  int64_t T_out = 0;
  {
    // this rank's local cu_seqlens
    std::vector<int64_t> cu((size_t)B + 1, 0);
    for (int32_t k = 0; k < B; ++k) cu[k + 1] = cu[k] + h_all[(size_t)me * B + k];
    // pack: the samples of this rank that other ranks take, by destination, each in its perm
    // order (the part a rank keeps is read straight from its own buffer by the gather below,
    // unless force_nccl sends it to itself)
    int64_t off = 0;
    for (int32_t dst = 0; dst < W; ++dst) {
      if (dst == me && !self_nccl) continue;
      for (int32_t k = 0; k < B; ++k) {
        const int32_t g = perm[(size_t)dst * B + k];
        if (g / B != me) continue;
        hp[n_pack] = cu[g % B]; hp[B + n_pack] = h_all[g]; hp[2 * B + n_pack] = off;
        hp[3 * B + n_pack] = g % B; hp[4 * B + n_pack] = n_pack;
        off += h_all[g]; send_cnt[dst] += h_all[g]; send_scnt[dst] += 1; ++n_pack;
      }
    }
    UB_REQUIRE(off <= cap, UB_ERR_CAPACITY, "tokens sent (%lld) exceed capacity %lld", (long long)off, (long long)cap);
    // gather: output sample k (perm order) from this rank's buffer (sel 0) or from its source
    // rank's chunk of the receive buffer (sel 1, chunks by source rank ascending)
    for (int32_t k = 0; k < B; ++k) {
      const int32_t g = perm[(size_t)me * B + k], src = g / B;
      if (src == me && !self_nccl) continue;
      recv_cnt[src] += h_all[g];
      recv_scnt[src] += 1;
    }
    std::vector<int64_t> base(W, 0), sbase(W, 0);
    for (int32_t q = 1; q < W; ++q) { base[q] = base[q - 1] + recv_cnt[q - 1]; sbase[q] = sbase[q - 1] + recv_scnt[q - 1]; }
    hcu[0] = 0;
    for (int32_t k = 0; k < B; ++k) {
      const int32_t g = perm[(size_t)me * B + k], src = g / B;
      if (src == me && !self_nccl) {
        hu[k] = cu[g % B]; hu[3 * B + k] = g % B; hu[5 * B + k] = 0;
      } else {
        hu[k] = base[src]; hu[3 * B + k] = sbase[src]; hu[5 * B + k] = 1;
        base[src] += h_all[g]; sbase[src] += 1;
      }
      hu[B + k] = h_all[g]; hu[2 * B + k] = T_out; hu[4 * B + k] = k;
      T_out += h_all[g];
      UB_REQUIRE(T_out <= INT32_MAX, UB_ERR_SHAPE, "received tokens overflow int32");
      hcu[k + 1] = (int32_t)T_out;
    }
    UB_REQUIRE(T_out <= cap, UB_ERR_CAPACITY, "tokens received (%lld) exceed capacity %lld", (long long)T_out,
               (long long)cap);
  }
  UB_PHASE();
  // 4. one H2D of both tables and the new cu_seqlens; pack what leaves this rank
  UB_CHECK_CUDA(cudaMemcpyAsync(w.stage, c->h_stage, sizeof(int64_t) * stage_words(B), cudaMemcpyHostToDevice, s));
  if (n_pack > 0 &&
      (st = exchange_gather(d_my_tokens, nullptr, w.send_tok, d_my_samples, nullptr, w.send_smp, w.stage, nullptr, n_pack,
                            B, rec, srec, nullptr, nullptr, 0, s)) != UB_OK)
    return st;
  UB_PHASE();
  // 5. all-to-all-v over NVLink (grouped point-to-point; the self chunk only with force_nccl)
  bool any_peer = false;
  for (int32_t peer = 0; peer < W; ++peer)
    any_peer = any_peer || send_cnt[peer] > 0 || recv_cnt[peer] > 0 || send_scnt[peer] > 0 || recv_scnt[peer] > 0;
  if (any_peer) {
    UB_CHECK_NCCL(ncclGroupStart());
    int64_t so = 0, ro = 0, sso = 0, rso = 0;
    for (int32_t peer = 0; peer < W; ++peer) {
      if (send_cnt[peer] > 0)
        UB_CHECK_NCCL(ncclSend(w.send_tok + so * rec, (size_t)(send_cnt[peer] * rec), ncclUint8, peer, c->nccl, s));
      if (recv_cnt[peer] > 0)
        UB_CHECK_NCCL(ncclRecv(w.recv_tok + ro * rec, (size_t)(recv_cnt[peer] * rec), ncclUint8, peer, c->nccl, s));
      if (srec > 0 && send_scnt[peer] > 0)
        UB_CHECK_NCCL(ncclSend(w.send_smp + sso * srec, (size_t)(send_scnt[peer] * srec), ncclUint8, peer, c->nccl, s));
      if (srec > 0 && recv_scnt[peer] > 0)
        UB_CHECK_NCCL(ncclRecv(w.recv_smp + rso * srec, (size_t)(recv_scnt[peer] * srec), ncclUint8, peer, c->nccl, s));
      c->nccl_ops += (send_cnt[peer] > 0) + (recv_cnt[peer] > 0) + (srec > 0 && send_scnt[peer] > 0) +
                     (srec > 0 && recv_scnt[peer] > 0);
      so += send_cnt[peer]; ro += recv_cnt[peer]; sso += send_scnt[peer]; rso += recv_scnt[peer];
    }
    UB_CHECK_NCCL(ncclGroupEnd());
  }
  UB_PHASE();
  // 6. reorder into perm order (a5): kept samples from this rank's own buffer, the others from
  // the receive buffer; the same launch writes the new cu_seqlens (the input-only
  // operators run during the exchange)
  if ((st = exchange_gather(d_my_tokens, w.recv_tok, d_out_tokens, d_my_samples, w.recv_smp, d_out_samples,
                            w.stage + (size_t)5 * B, w.stage + (size_t)10 * B, B, B, rec, srec,
                            reinterpret_cast<const int32_t*>(w.stage + (size_t)11 * B), d_out_cu, B + 1, s)) != UB_OK)
    return st;
  UB_CHECK_CUDA(cudaEventRecord(c->ev_staging, s));
  UB_PHASE();
#undef UB_PHASE
  if (c->trace) {
    for (int k = 1; k < ip && k < 9; ++k) c->t_phase[k - 1] += tp[k] - tp[k - 1];
    ++c->n_finish;
  }
  if (h_perm) std::memcpy(h_perm, perm.data(), sizeof(int32_t) * perm.size());
  *h_out_T = T_out;
  return UB_OK;
}

#define UB_EXCHANGE_ARGS_CHECK()                                                                            \
  UB_REQUIRE(comm && d_my_tokens && d_out_tokens && d_out_cu && h_out_T && ws, UB_ERR_INVALID_ARG, "null pointer"); \
  UB_REQUIRE(B >= 1 && rec > 0 && srec >= 0 && cap >= 1, UB_ERR_SHAPE, "bad sizes");                        \
  UB_REQUIRE(srec == 0 || (d_my_samples && d_out_samples), UB_ERR_INVALID_ARG, "null sample pointer")

extern "C" ub_status ub_exchange_begin(void* comm, int32_t slot, int32_t B, const int32_t* d_my_lengths, void* ws,
                                       void* stream) {
  clear_error();
  UB_REQUIRE(comm && d_my_lengths && ws, UB_ERR_INVALID_ARG, "null pointer");
  UB_REQUIRE(B >= 1, UB_ERR_SHAPE, "B must be >= 1");
  UB_REQUIRE(slot >= 0 && slot < UB_EXCHANGE_SLOTS, UB_ERR_INVALID_ARG, "slot %d out of [0, %d)", slot,
             UB_EXCHANGE_SLOTS);
  return exchange_begin(static_cast<Comm*>(comm), slot, B, d_my_lengths, ws, as_stream(stream));
}

extern "C" ub_status ub_exchange_finish(void* comm, int32_t slot, int32_t mode, int32_t B, int32_t max_seqlen,
                                        const void* d_my_tokens, const void* d_my_samples, int64_t rec, int64_t srec,
                                        int64_t cap, void* d_out_tokens, void* d_out_samples, int32_t* d_out_cu,
                                        int32_t* h_perm, int64_t* h_out_T, void* ws, void* stream) {
  clear_error();
  UB_EXCHANGE_ARGS_CHECK();
  UB_REQUIRE(slot >= 0 && slot < UB_EXCHANGE_SLOTS, UB_ERR_INVALID_ARG, "slot %d out of [0, %d)", slot,
             UB_EXCHANGE_SLOTS);
  return exchange_finish(static_cast<Comm*>(comm), slot, mode, B, max_seqlen, d_my_tokens, d_my_samples, rec, srec,
                         cap, d_out_tokens, d_out_samples, d_out_cu, h_perm, h_out_T, ws, as_stream(stream));
}

extern "C" ub_status ub_exchange_slot_lengths(void* comm, int32_t slot, int32_t B, int32_t* h_out) {
  clear_error();
  UB_REQUIRE(comm && h_out, UB_ERR_INVALID_ARG, "null pointer");
  UB_REQUIRE(slot >= 0 && slot < UB_EXCHANGE_SLOTS, UB_ERR_INVALID_ARG, "slot %d out of [0, %d)", slot,
             UB_EXCHANGE_SLOTS);
  const Comm* c = static_cast<const Comm*>(comm);
  UB_REQUIRE(B >= 1 && B <= c->cap_B, UB_ERR_SHAPE, "B = %d: the slot holds at most %d per rank", B, c->cap_B);
  UB_REQUIRE(c->slot_B[slot] == 0, UB_ERR_INVALID_ARG, "slot %d has an unfinished begin", slot);
  std::memcpy(h_out, c->h_all + (size_t)slot * c->W * c->cap_B, sizeof(int32_t) * (size_t)c->W * B);
  return UB_OK;
}

extern "C" ub_status ub_exchange_fmha_schedule(void* comm, int32_t slot, const int32_t* h_perm, int32_t B,
                                               int32_t heads, int32_t max_seqlen, int32_t grid, int32_t is_bwd,
                                               int32_t* h_sched, size_t cap_ints, int32_t* d_sched, void* stream) {
  clear_error();
  UB_REQUIRE(comm && h_perm && h_sched, UB_ERR_INVALID_ARG, "null pointer");
  UB_REQUIRE(slot >= 0 && slot < UB_EXCHANGE_SLOTS, UB_ERR_INVALID_ARG, "slot %d out of [0, %d)", slot,
             UB_EXCHANGE_SLOTS);
  const Comm* c = static_cast<const Comm*>(comm);
  UB_REQUIRE(B >= 1 && B <= c->cap_B && B <= 4096, UB_ERR_SHAPE, "B = %d: the slot holds at most %d per rank", B,
             c->cap_B);
  UB_REQUIRE(c->slot_B[slot] == 0, UB_ERR_INVALID_ARG, "slot %d has an unfinished begin", slot);
  const int32_t* all = c->h_all + (size_t)slot * c->W * c->cap_B;
  int32_t lens[4096];
  for (int32_t k = 0; k < B; ++k) {
    const int32_t g = h_perm[(size_t)c->rank * B + k];
    UB_REQUIRE(g >= 0 && g < c->W * B, UB_ERR_INVALID_ARG, "perm entry %d out of range", g);
    lens[k] = all[g];
  }
  ub_status st = ub_fmha_schedule(lens, B, heads, max_seqlen, grid, is_bwd, h_sched, cap_ints);
  if (st != UB_OK || d_sched == nullptr) return st;
  const size_t n = fmha_schedule_ints(B, heads, max_seqlen, grid, is_bwd);
  UB_CHECK_CUDA(cudaMemcpyAsync(d_sched, h_sched, n * sizeof(int32_t), cudaMemcpyHostToDevice, as_stream(stream)));
  return UB_OK;
}

extern "C" ub_status ub_balance_exchange(void* comm, int32_t mode, int32_t B, int32_t max_seqlen,
                                         const int32_t* d_my_lengths, const void* d_my_tokens,
                                         const void* d_my_samples, int64_t rec, int64_t srec, int64_t cap,
                                         void* d_out_tokens, void* d_out_samples, int32_t* d_out_cu,
                                         int32_t* h_perm, int64_t* h_out_T, void* ws, void* side_stream) {
  clear_error();
  UB_EXCHANGE_ARGS_CHECK();
  UB_REQUIRE(d_my_lengths, UB_ERR_INVALID_ARG, "null pointer");
  Comm* c = static_cast<Comm*>(comm);
  cudaStream_t s = as_stream(side_stream);
  const int32_t slot = kExSlots - 1;
  ub_status st = exchange_begin(c, slot, B, d_my_lengths, ws, s);
  if (st != UB_OK) return st;
  return exchange_finish(c, slot, mode, B, max_seqlen, d_my_tokens, d_my_samples, rec, srec, cap, d_out_tokens,
                         d_out_samples, d_out_cu, h_perm, h_out_T, ws, s);
}
