// Host-side 1F1B program and communication plan of one pipeline stage.
//
// Program ("issues a forward task and a backward task in a round-robin
// manner", reading D8): stage k of N runs
//   w = min(N−k−1, M) warm-up forwards F(0..w−1),
//   then pairs F(w+j), B(j) for j = 0..M−w−1,
//   then cooldown backwards B(M−w..M−1).
// Version differences: Eq. 5 for F, Eq. 6 for B.
// Base versions: an F(i) runs after B(i−w−1), so c_F = max(0, i−w); a B(j) runs
// after B(j−1), so c_B = j.
//
// Communication plan. Per task: F(i) on k > 0 needs
// recv_fwd(i) before it; F(i) on k < N−1 is followed by send_fwd(i); B(j) on k < N−1
// needs recv_bwd(j); B(j) on k > 0 is followed by send_bwd(j). The plan lists these
// ops one per record, in issue order: at each task boundary n the trailing send of
// task n−1, then the leading receive of task n (before_op = n). The engine runs each
// direction on its own communicator and comm stream (activations: send_fwd /
// recv_fwd; gradients: send_bwd / recv_bwd), so the two directions never wait on
// each other and no send/recv pairing into groups is needed; within a direction the
// ops of every stage follow this order, which pairs them per peer in mini-batch order.
#include <vector>

#include <limits>

#include "engine.hpp"

namespace st {

int version_difference(int k, int N, int dir) {
  if (N < 1 || k < 0 || k >= N) return -1;
  return dir == ST_FWD ? (k / 2 + N - k - 1) : (k / 2);
}

int stage_s(int pred, int k, int N, int dir) {
  switch (pred) {
    case ST_PRED_SPECTRAIN: return version_difference(k, N, dir);
    // the staleness-free target: the forward predicts across the N−k−1
    // updates that land before its backward, the backward uses the current weights
    case ST_PRED_STALENESS_FREE: return dir == ST_FWD ? N - k - 1 : 0;
    default: return 0;  // ST_PRED_NONE, ST_PRED_STASH
  }
}

std::vector<Task> build_program(int N, int k, int64_t M) {
  std::vector<Task> p;
  if (M <= 0) return p;
  const int64_t w = std::min<int64_t>(N - k - 1, M);
  p.reserve((size_t)(2 * M));
  for (int64_t i = 0; i < w; ++i) p.push_back({ST_FWD, i});
  for (int64_t j = 0; j < M - w; ++j) {
    p.push_back({ST_FWD, w + j});
    p.push_back({ST_BWD, j});
  }
  for (int64_t j = M - w; j < M; ++j) p.push_back({ST_BWD, j});
  return p;
}

std::vector<st_event> program_events(int N, int k, int64_t M, int pred) {
  std::vector<Task> p = build_program(N, k, M);
  std::vector<st_event> ev;
  ev.reserve(p.size());
  int64_t version = 0;
  const int64_t sF = stage_s(pred, k, N, ST_FWD);
  const int64_t sB = stage_s(pred, k, N, ST_BWD);
  std::vector<int64_t> fwd_version((size_t)std::max<int64_t>(M, 0), 0);  // ST_PRED_STASH
  for (size_t n = 0; n < p.size(); ++n) {
    st_event e{};
    e.stage = k;
    e.op_idx = (int32_t)n;
    e.dir = p[n].dir;
    e.mb = p[n].mb;
    e.base_version = version;
    if (pred == ST_PRED_STASH) {  // a backward runs on the weights its forward stashed
      if (p[n].dir == ST_FWD) fwd_version[(size_t)p[n].mb] = version;
      else e.base_version = fwd_version[(size_t)p[n].mb];
    }
    e.s = p[n].dir == ST_FWD ? sF : sB;
    e.target = e.base_version + e.s;
    ev.push_back(e);
    if (p[n].dir == ST_BWD) ++version;
  }
  return ev;
}

namespace {
struct Op {
  int kind;  // CK_*
  int64_t mb;
};
}  // namespace

std::vector<CommGroup> build_comm_plan(int N, int k, int64_t M) {
  std::vector<Task> p = build_program(N, k, M);
  std::vector<CommGroup> plan;
  auto pre = [&](const Task& t, Op* o) -> bool {
    if (t.dir == ST_FWD && k > 0) { *o = {CK_RECV_FWD, t.mb}; return true; }
    if (t.dir == ST_BWD && k < N - 1) { *o = {CK_RECV_BWD, t.mb}; return true; }
    return false;
  };
  auto post = [&](const Task& t, Op* o) -> bool {
    if (t.dir == ST_FWD && k < N - 1) { *o = {CK_SEND_FWD, t.mb}; return true; }
    if (t.dir == ST_BWD && k > 0) { *o = {CK_SEND_BWD, t.mb}; return true; }
    return false;
  };
  for (size_t n = 0; n <= p.size(); ++n) {
    Op a{}, b{};
    if (n > 0 && post(p[n - 1], &a)) plan.push_back({(int32_t)n, 1, {a.kind, -1}, {a.mb, -1}});
    if (n < p.size() && pre(p[n], &b)) plan.push_back({(int32_t)n, 1, {b.kind, -1}, {b.mb, -1}});
  }
  return plan;
}

// Min-max contiguous partition (P:146, P:380, P:404 — stage
// imbalance bounds a pipeline): f[k][j] = the least possible maximum stage cost when
// layers j..L−1 form k non-empty contiguous stages (suffix DP over prefix sums); the
// cuts are then chosen front to back as the smallest index whose stage and best
// remaining suffix both stay within the global optimum, i.e. the lexicographically
// smallest optimal cut vector.
st_status partition_layers(const double* cost, int L, int N, int32_t* cuts, double* max_cost) {
  if (!cost || L < 1 || N < 1 || N > L || (N > 1 && !cuts))
    return set_error(ST_ERR_INPUT, "partition: need 1 <= N <= L and a cost per layer");
  std::vector<double> pre((size_t)L + 1, 0.0);
  for (int i = 0; i < L; ++i) {
    if (!(cost[i] >= 0.0)) return set_error(ST_ERR_INPUT, "partition: cost[%d] must be finite and >= 0", i);
    pre[(size_t)i + 1] = pre[(size_t)i] + cost[i];
  }
  const double inf = std::numeric_limits<double>::infinity();
  std::vector<std::vector<double>> f((size_t)N + 1, std::vector<double>((size_t)L + 1, inf));
  for (int j = 0; j < L; ++j) f[1][(size_t)j] = pre[(size_t)L] - pre[(size_t)j];
  for (int k = 2; k <= N; ++k)
    for (int j = 0; j + k <= L; ++j)
      for (int i = j + 1; i + (k - 1) <= L; ++i)
        f[(size_t)k][(size_t)j] = std::min(f[(size_t)k][(size_t)j], std::max(pre[(size_t)i] - pre[(size_t)j], f[(size_t)k - 1][(size_t)i]));
  const double opt = f[(size_t)N][0];
  int start = 0;
  for (int k = N; k >= 2; --k) {
    int pick = -1;
    for (int i = start + 1; i + (k - 1) <= L; ++i)
      if (std::max(pre[(size_t)i] - pre[(size_t)start], f[(size_t)k - 1][(size_t)i]) <= opt) {
        pick = i;
        break;
      }
    if (pick < 0) return set_error(ST_ERR_STATE, "partition: no cut reproduces the optimum (internal)");
    cuts[N - k] = pick;
    start = pick;
  }
  if (max_cost) *max_cost = opt;
  return ST_OK;
}

}  // namespace st
