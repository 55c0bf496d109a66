// rounds.h — the host-side round loop of a partitioned (multi-GPU) run
// (include/atos.h "multi-GPU").  Pure C++ (no CUDA): capi.cu
// instantiates it with the CUDA engine of dist_impl.cuh and an NCCL or
// host-callback exchange; tests/round_harness.cpp instantiates it with a
// serial CPU engine so the loop itself is tested without a GPU.
//
// One round (the worker loop "until the stop condition",
// with the remote activations of a 1-D vertex partition batched per round):
//   1. local_round: this rank's queue kernel runs (persistent: to local
//      quiescence; discrete: one superstep) and leaves its ROUND VECTOR —
//      messages per destination rank, local tasks still pending, abort code,
//      outbox overflow flag — in memory, with no host synchronisation;
//   2. gather: every rank's round vector reaches every rank (NCCL all-gather
//      on the device + ONE device->host copy: the round's only host sync);
//   3. every rank decides the same thing from the same matrix: an error on
//      any rank fails the run on all ranks (no rank is left waiting in a
//      collective); no message and no pending task anywhere ends the run —
//      PageRank first runs one closing round that flushes every remote
//      accumulation (flush_all), and ends when that round sends nothing;
//   4. alltoallv of the messages (device buffers with NCCL send/recv; host
//      staging with a callback exchange), then apply on the receiver.
#pragma once
#include <chrono>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/atos.h"

namespace atos_rounds {

// Round vector of one rank: K = world + 3 int64 entries.
enum { RV_PENDING = 0, RV_ABORT = 1, RV_OVERFLOW = 2 };  // offsets after the `world` send counts
inline int rv_len(int world) { return world + 3; }

// Exchange between the ranks of a communicator.
struct Exchange {
  int rank = 0, world = 1;
  atos_status (*errf)(atos_status, const char*, ...) = nullptr;  // records the detail string
  virtual ~Exchange() {}
  virtual bool on_device() const = 0;  // buffers passed in are device (true) or host (false) memory
  // Every rank's K-int64 vector `vec` -> M (host, world x K, rank order).
  virtual atos_status gather(const int64_t* vec, int K, int64_t* M) = 0;
  // uint64 messages: segment r of `send` at soff[r] (scnt[r] entries) goes to
  // rank r and arrives at recv + roff[r] (rcnt[r] entries).
  virtual atos_status alltoallv(const uint64_t* send, const int64_t* soff, const int64_t* scnt, uint64_t* recv,
                                const int64_t* roff, const int64_t* rcnt) = 0;
};

// One rank's local work.
struct Engine {
  virtual ~Engine() {}
  virtual bool on_device() const = 0;
  virtual atos_status local_round(int flush_all) = 0;
  virtual const int64_t* round_vector() = 0;  // K entries, device or host per on_device()
  virtual const uint64_t* outbox() = 0;        // per-destination segments ...
  virtual const int64_t* outbox_seg() = 0;     // ... starting at these (host) offsets
  virtual atos_status inbox(int64_t cap, uint64_t** p) = 0;
  virtual atos_status apply(int64_t count) = 0;  // apply inbox[0, count)
  // synchronous copies between the engine's memory and the host (staging)
  virtual atos_status to_host(void* dst, const void* src, size_t bytes) = 0;
  virtual atos_status to_engine(void* dst, const void* src, size_t bytes) = 0;
};

struct RoundStats {
  int64_t rounds = 0, bytes_sent = 0;
};

template <class ErrFn>
atos_status run_rounds(Exchange& comm, Engine& eng, bool closing_flush, double timeout_s, RoundStats& st,
                       ErrFn err) {
  const int W = comm.world, me = comm.rank, K = rv_len(W);
  const bool stage = eng.on_device() && !comm.on_device();
  std::vector<int64_t> M((size_t)W * K), hvec(K), soff(W), scnt(W), roff(W), rcnt(W), pk(W);
  std::vector<uint64_t> hsend, hrecv;
  const auto t0 = std::chrono::steady_clock::now();
  int flush_all = 0;
  for (;;) {
    atos_status s = eng.local_round(flush_all);
    if (s != ATOS_OK) return s;
    const int64_t* vec = eng.round_vector();
    if (stage) {
      if ((s = eng.to_host(hvec.data(), vec, sizeof(int64_t) * K)) != ATOS_OK) return s;
      vec = hvec.data();
    }
    if ((s = comm.gather(vec, K, M.data())) != ATOS_OK) return s;
    st.rounds++;
    for (int r = 0; r < W; ++r) {
      const int64_t ab = M[(size_t)r * K + W + RV_ABORT], ov = M[(size_t)r * K + W + RV_OVERFLOW];
      if (ab == 1) return err(ATOS_ERR_QUEUE_OVERFLOW, "task queue overflow on rank %d; retry with a larger queue_capacity", r);
      if (ab == 2) return err(ATOS_ERR_TIMEOUT, "device watchdog fired on rank %d", r);
      if (ab) return err(ATOS_ERR_CUDA, "rank %d aborted (code %lld)", r, (long long)ab);
      if (ov) return err(ATOS_ERR_QUEUE_OVERFLOW, "partition outbox overflow on rank %d", r);
    }
    int64_t total = 0;
    for (int r = 0; r < W; ++r)
      for (int j = 0; j <= W; ++j) total += M[(size_t)r * K + j];  // messages + pending tasks
    if (total == 0) {
      if (!closing_flush || flush_all) break;
      flush_all = 1;  // PageRank: one round that sends every remaining remote contribution
      continue;
    }
    flush_all = 0;
    int64_t nsend = 0, nrecv = 0;
    const int64_t* seg = eng.outbox_seg();
    for (int r = 0; r < W; ++r) {
      scnt[r] = r == me ? 0 : M[(size_t)me * K + r];
      rcnt[r] = r == me ? 0 : M[(size_t)r * K + me];
      soff[r] = seg[r];
      roff[r] = nrecv;
      nrecv += rcnt[r];
      nsend += scnt[r];
    }
    st.bytes_sent += nsend * (int64_t)sizeof(uint64_t);
    uint64_t* in = nullptr;
    if ((s = eng.inbox(nrecv, &in)) != ATOS_OK) return s;
    if (stage) {
      // host exchange of device buffers: pack this rank's segments on the host, unpack into the inbox
      hsend.resize((size_t)nsend + 1);
      hrecv.resize((size_t)nrecv + 1);
      int64_t o = 0;
      for (int r = 0; r < W; ++r) {
        pk[r] = o;
        if (scnt[r] && (s = eng.to_host(hsend.data() + o, eng.outbox() + soff[r], sizeof(uint64_t) * scnt[r])) != ATOS_OK)
          return s;
        o += scnt[r];
      }
      if ((s = comm.alltoallv(hsend.data(), pk.data(), scnt.data(), hrecv.data(), roff.data(), rcnt.data())) != ATOS_OK)
        return s;
      if (nrecv && (s = eng.to_engine(in, hrecv.data(), sizeof(uint64_t) * nrecv)) != ATOS_OK) return s;
    } else if ((s = comm.alltoallv(eng.outbox(), soff.data(), scnt.data(), in, roff.data(), rcnt.data())) != ATOS_OK) {
      return s;
    }
    if ((s = eng.apply(nrecv)) != ATOS_OK) return s;
    if (timeout_s > 0) {
      const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (el > timeout_s) return err(ATOS_ERR_TIMEOUT, "host watchdog: %.1f s in %lld rounds", el, (long long)st.rounds);
    }
  }
  return ATOS_OK;
}

// Exchange through caller callbacks on host memory (include/atos.h,
// atos_comm_init_host): e.g. a gloo process group driven from Python.
struct HostExchange : Exchange {
  atos_allgather_fn ag = nullptr;
  atos_alltoallv_fn a2a = nullptr;
  void* user = nullptr;
  std::vector<int64_t> sb, rb;
  bool on_device() const override { return false; }
  atos_status gather(const int64_t* vec, int K, int64_t* M) override {
    if (ag(user, vec, M, (int64_t)K * (int64_t)sizeof(int64_t)) != 0)
      return errf ? errf(ATOS_ERR_NCCL, "allgather callback failed") : ATOS_ERR_NCCL;
    return ATOS_OK;
  }
  atos_status alltoallv(const uint64_t* send, const int64_t* soff, const int64_t* scnt, uint64_t* recv,
                        const int64_t* roff, const int64_t* rcnt) override {
    // the callback takes packed segments in rank order with byte counts
    sb.assign(world, 0);
    rb.assign(world, 0);
    int64_t o = 0;
    for (int r = 0; r < world; ++r) {
      if (soff[r] != o)  // not packed (the loop packs staged sends)
        return errf ? errf(ATOS_ERR_INVALID_ARGUMENT, "host exchange needs packed segments") : ATOS_ERR_INVALID_ARGUMENT;
      o += scnt[r];
      sb[r] = scnt[r] * (int64_t)sizeof(uint64_t);
      rb[r] = rcnt[r] * (int64_t)sizeof(uint64_t);
    }
    (void)roff;
    if (a2a(user, send, sb.data(), recv, rb.data()) != 0)
      return errf ? errf(ATOS_ERR_NCCL, "alltoallv callback failed") : ATOS_ERR_NCCL;
    return ATOS_OK;
  }
};

}  // namespace atos_rounds
