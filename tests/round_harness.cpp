// round_harness.cpp — TEST INFRASTRUCTURE: drives the library's host-side
// round loop (paper_2112_00132_b200/csrc/rounds.h, the product code under
// test) with serial CPU engines, so the multi-rank protocol — round vectors,
// collective error handling, termination, PageRank's closing flush — runs
// over real gloo collectives without a GPU (tests/test_dist.py).  The engines
// are plain serial stand-ins for the CUDA kernels: a label-correcting BFS and
// a FIFO push PageRank on this rank's partition, with remote updates batched
// per destination exactly like dist_impl.cuh's.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <deque>
#include <vector>

#include "../paper_2112_00132_b200/csrc/rounds.h"

using namespace atos_rounds;

static atos_status herr(atos_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vfprintf(stderr, fmt, ap);
  va_end(ap);
  fputc('\n', stderr);
  return s;
}

struct FakeEngine : Engine {
  int app = 0, rank = 0, world = 1;
  int64_t N = 0, vb = 0, ve = 0;
  std::vector<int64_t> b, off;
  std::vector<int32_t> col;
  double alpha = 0.85, eps = 1e-6;
  int fail_round = -1;  // > 0: raise an abort code in that round (collective error test)
  int round = 0;
  // state
  std::vector<uint32_t> dist, sent;      // BFS
  std::vector<double> res, rank_, racc;  // PageRank
  std::deque<int64_t> q;
  std::vector<std::vector<uint64_t>> out;
  std::vector<uint64_t> outbuf, in;
  std::vector<int64_t> seg, rv;

  int owner(int64_t w) const {
    int r = 0;
    while (!(w >= b[r] && w < b[r + 1])) ++r;
    return r;
  }
  bool on_device() const override { return false; }
  void init(int64_t src) {
    const int64_t n = ve - vb;
    out.assign(world, {});
    if (app == 0) {
      dist.assign(n, 0xFFFFFFFFu);
      sent.assign(N, 0xFFFFFFFFu);
      if (src >= vb && src < ve) {
        dist[src - vb] = 0;
        q.push_back(src - vb);
      }
    } else {
      res.assign(n, 0.0);
      rank_.assign(n, 1.0 - alpha);
      racc.assign(N, 0.0);
      for (int64_t v = 0; v < n; ++v) {  // R4 seeding: one synchronous push from rank = 1 - alpha
        const int64_t d = off[v + 1] - off[v];
        for (int64_t e = off[v]; e < off[v + 1]; ++e) {
          const int64_t w = col[e];
          if (w >= vb && w < ve) res[w - vb] += (1.0 - alpha) * alpha / (double)d;
          else racc[w] += (1.0 - alpha) * alpha / (double)d;
        }
      }
      for (int64_t v = 0; v < n; ++v) q.push_back(v);  // every vertex queued
    }
  }
  void put(int64_t w, uint32_t payload) {
    const int r = owner(w);
    out[r].push_back(((uint64_t)(w - b[r]) << 32) | payload);
  }
  atos_status local_round(int flush_all) override {
    ++round;
    for (auto& o : out) o.clear();
    while (!q.empty()) {
      const int64_t v = q.front();
      q.pop_front();
      if (app == 0) {
        const uint32_t d = dist[v] + 1;
        for (int64_t e = off[v]; e < off[v + 1]; ++e) {
          const int64_t w = col[e];
          if (w >= vb && w < ve) {
            if (d < dist[w - vb]) {
              dist[w - vb] = d;
              q.push_back(w - vb);
            }
          } else if (d < sent[w]) {
            sent[w] = d;
            put(w, d);
          }
        }
      } else {
        const double r = res[v];
        res[v] = 0.0;
        if (r == 0.0) continue;
        rank_[v] += r;
        const int64_t deg = off[v + 1] - off[v];
        if (!deg) continue;
        const double c = alpha * r / (double)deg;
        for (int64_t e = off[v]; e < off[v + 1]; ++e) {
          const int64_t w = col[e];
          if (w >= vb && w < ve) {
            const double old = res[w - vb];
            res[w - vb] = old + c;
            if (old <= eps && old + c > eps) q.push_back(w - vb);
          } else {
            racc[w] += c;
          }
        }
      }
    }
    if (app == 1) {
      for (int64_t w = 0; w < N; ++w) {
        if (w >= vb && w < ve) continue;
        const double a = racc[w];
        if (flush_all ? a != 0.0 : a > eps) {
          const float f = (float)a;
          racc[w] = flush_all ? 0.0 : a - (double)f;
          uint32_t bits;
          std::memcpy(&bits, &f, 4);
          put(w, bits);
        }
      }
    }
    seg.assign(world + 1, 0);
    outbuf.clear();
    for (int r = 0; r < world; ++r) {
      seg[r] = (int64_t)outbuf.size();
      outbuf.insert(outbuf.end(), out[r].begin(), out[r].end());
    }
    seg[world] = (int64_t)outbuf.size();
    rv.assign(rv_len(world), 0);
    for (int r = 0; r < world; ++r) rv[r] = (int64_t)out[r].size();
    rv[world + RV_ABORT] = (fail_round > 0 && round == fail_round) ? 2 : 0;
    return ATOS_OK;
  }
  const int64_t* round_vector() override { return rv.data(); }
  const uint64_t* outbox() override { return outbuf.data(); }
  const int64_t* outbox_seg() override { return seg.data(); }
  atos_status inbox(int64_t cap, uint64_t** p) override {
    in.resize((size_t)cap + 1);
    *p = in.data();
    return ATOS_OK;
  }
  atos_status apply(int64_t count) override {
    for (int64_t i = 0; i < count; ++i) {
      const uint64_t m = in[i];
      const int64_t l = (int64_t)(m >> 32);
      const uint32_t pay = (uint32_t)m;
      if (app == 0) {
        if (pay < dist[l]) {
          dist[l] = pay;
          q.push_back(l);
        }
      } else {
        float c;
        std::memcpy(&c, &pay, 4);
        const double old = res[l];
        res[l] = old + (double)c;
        if (old <= eps && res[l] > eps) q.push_back(l);
      }
    }
    return ATOS_OK;
  }
  atos_status to_host(void* dst, const void* src, size_t bytes) override {
    std::memcpy(dst, src, bytes);
    return ATOS_OK;
  }
  atos_status to_engine(void* dst, const void* src, size_t bytes) override {
    std::memcpy(dst, src, bytes);
    return ATOS_OK;
  }
};

// app 0 = BFS from global src (out: depth as double), 1 = PageRank (out: rank).
// Returns the atos_status of the round loop.
extern "C" int harness_run(int app, int rank, int world, atos_allgather_fn ag, atos_alltoallv_fn a2a, int64_t N,
                           const int64_t* bounds, const int64_t* off, const int32_t* col, int64_t src, double alpha,
                           double eps, int fail_round, double* out, int64_t* rounds, int64_t* bytes) {
  FakeEngine e;
  e.app = app;
  e.rank = rank;
  e.world = world;
  e.N = N;
  e.b.assign(bounds, bounds + world + 1);
  e.vb = bounds[rank];
  e.ve = bounds[rank + 1];
  const int64_t n = e.ve - e.vb;
  e.off.assign(off, off + n + 1);
  e.col.assign(col, col + off[n]);
  e.alpha = alpha;
  e.eps = eps;
  e.fail_round = fail_round;
  e.init(src);
  HostExchange ex;
  ex.rank = rank;
  ex.world = world;
  ex.ag = ag;
  ex.a2a = a2a;
  ex.errf = herr;
  RoundStats st;
  const atos_status s = run_rounds(ex, e, app == 1, 0.0, st, herr);
  for (int64_t v = 0; v < n; ++v) out[v] = app == 0 ? (double)e.dist[v] : e.rank_[v];
  *rounds = st.rounds;
  *bytes = st.bytes_sent;
  return (int)s;
}
