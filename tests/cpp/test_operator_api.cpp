// The reference's unit-test scenarios for the scheduling primitives
// (proj/tests/execution_engine_test.cpp, workload_balancer_test.cpp,
// policies_test.cpp), re-expressed against the B200 build's operator API
// (namespace moespac, paper_2603_09983_b200/csrc/host/scheduler.hpp). Same
// calls, same expected values; built and run by tests/test_cpp_api.py.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <optional>
#include <random>
#include <vector>

#include "scheduler.hpp"

using namespace moespac;

static int g_checks = 0, g_fail = 0;
#define EXPECT(cond)                                                        \
  do {                                                                      \
    ++g_checks;                                                             \
    if (!(cond)) {                                                          \
      ++g_fail;                                                             \
      std::fprintf(stderr, "%s:%d: EXPECT(%s) failed\n", __FILE__, __LINE__, #cond); \
    }                                                                       \
  } while (0)
#define EXPECT_THROW(stmt, Ex)       \
  do {                               \
    bool thrown = false;             \
    try {                            \
      stmt;                          \
    } catch (const Ex&) {            \
      thrown = true;                 \
    } catch (...) {                  \
    }                                \
    EXPECT(thrown && #Ex);           \
  } while (0)

static ExpertKey key(int e) { return {0, e}; }

static HardwareProfile io_profile(std::int64_t t_io) {
  HardwareProfile p;
  p.t_cpu_unit_ns = p.t_gpu_unit_ns = p.t_draft_unit_ns = 1;
  p.t_io_unit_ns = t_io;
  p.expert_bytes = 10;
  p.vram_capacity_bytes = 1000;
  return p;
}

static std::vector<ExpertKey> drain_all(PrefetchQueues& q, int tau) {
  std::vector<ExpertKey> out;
  q.drain(tau, [&](ExpertKey k, int) {
    out.push_back(k);
    return true;
  });
  return out;
}

static void queues() {
  {  // descending level, FIFO inside a level; sub-tau requests stay
    PrefetchQueues q(4);
    q.enqueue(key(0), 4);
    q.enqueue(key(1), 2);
    q.enqueue(key(2), 4);
    q.enqueue(key(3), 3);
    const auto got = drain_all(q, 3);
    EXPECT(got.size() == 3 && got[0] == key(0) && got[1] == key(2) && got[2] == key(3));
    EXPECT(q.pending() == 1 && q.level_of(key(1)) == 2);
  }
  {  // coalescing keeps the higher level
    PrefetchQueues q(4);
    q.enqueue(key(7), 2);
    q.enqueue(key(7), 4);
    EXPECT(q.pending() == 1 && q.level_of(key(7)) == 4);
    q.enqueue(key(7), 1);
    EXPECT(q.level_of(key(7)) == 4);
    EXPECT(drain_all(q, 1).size() == 1);
  }
  {
    PrefetchQueues q(4);
    EXPECT_THROW(q.enqueue(key(0), 0), std::out_of_range);
    EXPECT_THROW(q.enqueue(key(0), 5), std::out_of_range);
    EXPECT_THROW(PrefetchQueues(0), std::invalid_argument);
    EXPECT_THROW(q.level_of(key(3)), std::out_of_range);
  }
  {  // a refusing visitor keeps its request
    PrefetchQueues q(3);
    q.enqueue(key(0), 3);
    q.enqueue(key(1), 3);
    int seen = 0;
    q.drain(1, [&](ExpertKey, int) { return ++seen == 1; });
    EXPECT(q.pending() == 1 && q.contains(key(1)));
  }
  {  // scrub
    PrefetchQueues q(3);
    q.enqueue(key(0), 3);
    q.enqueue(key(1), 2);
    q.enqueue(key(2), 2);
    q.scrub([](ExpertKey k, int) { return k.expert != 1; });
    EXPECT(q.pending() == 2 && !q.contains(key(1)));
    const auto got = drain_all(q, 1);
    EXPECT(got.size() == 2 && got[0] == key(0) && got[1] == key(2));
  }
}

static void pool() {
  {
    ResidencyPool p(4, 10, 30);
    EXPECT(p.frozen_score() == 5);
    EXPECT(p.admit(key(0), 2) && p.admit(key(1), 4) && p.admit(key(2), 1));
    EXPECT(p.free_bytes() == 0 && !p.admit(key(3), 4) && p.size() == 3);
    EXPECT(p.score_of(key(0)) == 2);
    EXPECT(p.admit(key(0), 3) && p.score_of(key(0)) == 3 && p.total_bytes() == 30);
    EXPECT(p.retag(key(2), 4) && p.score_of(key(2)) == 4);
    EXPECT(!p.retag(key(9), 1));
    EXPECT_THROW(p.score_of(key(9)), std::out_of_range);
    EXPECT_THROW(p.admit(key(5), 5), std::out_of_range);
    EXPECT_THROW(p.retag(key(0), -1), std::out_of_range);
  }
  {
    ResidencyPool p(4, 10, 100);
    p.admit(key(0), 1);
    p.admit(key(1), 3);
    p.admit(key(2), 4);
    p.freeze(key(2));
    const auto ev = apply_eviction(p, 3);
    EXPECT(ev.size() == 1 && ev[0].key == key(0) && ev[0].kind == IoEvent::Kind::evict && ev[0].duration_ns == 0);
    EXPECT(p.size() == 2 && apply_eviction(p, 1).empty());
    EXPECT_THROW(apply_eviction(p, 0), std::out_of_range);
    EXPECT_THROW(apply_eviction(p, 5), std::out_of_range);
  }
  {  // frozen survives, thawed goes first
    ResidencyPool p(4, 10, 100);
    p.admit(key(0), 2);
    p.freeze(key(0));
    p.freeze(key(0));
    EXPECT(p.score_of(key(0)) == p.frozen_score() && p.evict_below(4).empty());
    EXPECT(p.retag(key(0), 1) && p.score_of(key(0)) == p.frozen_score());
    p.thaw_and_recycle(key(0));
    EXPECT(p.score_of(key(0)) == 0);
    const auto ev = p.evict_below(1);
    EXPECT(ev.size() == 1 && ev[0] == key(0));
    EXPECT_THROW(p.freeze(key(9)), std::logic_error);
    EXPECT_THROW(p.thaw_and_recycle(key(9)), std::logic_error);
  }
  {  // evict_for_room: lowest scores first, only what is needed, capped by tau
    ResidencyPool p(4, 10, 50);
    for (int e = 0; e < 5; ++e) p.admit(key(e), e);
    const auto ev = p.evict_for_room(20, 4);
    EXPECT(ev.size() == 2 && ev[0] == key(0) && ev[1] == key(1) && p.free_bytes() == 20);
    EXPECT(p.evict_for_room(20, 4).empty());
    EXPECT(p.evict_for_room(30, 2).empty());
    p.freeze(key(2));
    p.freeze(key(3));
    p.freeze(key(4));
    EXPECT(p.evict_for_room(50, 4).empty());
  }
  {  // ties inside a score level go in ascending key order
    ResidencyPool p(4, 10, 100);
    p.admit(key(5), 1);
    p.admit(key(2), 1);
    p.admit(key(9), 0);
    p.admit(key(1), 1);
    const auto ev = p.evict_below(2);
    EXPECT(ev.size() == 4 && ev[0] == key(9) && ev[1] == key(1) && ev[2] == key(2) && ev[3] == key(5));
  }
}

static void drain() {
  {
    PrefetchQueues q(4);
    ResidencyPool p(4, 10, 1000);
    const HardwareProfile prof = io_profile(100);
    q.enqueue(key(0), 4);
    q.enqueue(key(1), 4);
    q.enqueue(key(2), 3);
    const auto loads = drain_prefetch(q, 1, 200, prof, p);
    EXPECT(loads.size() == 2 && loads[0].key == key(0) && loads[0].start_ns == 0 && loads[0].duration_ns == 100);
    EXPECT(loads[1].key == key(1) && loads[1].start_ns == 100);
    EXPECT(p.resident(key(0)) && p.resident(key(1)) && !p.resident(key(2)) && q.contains(key(2)));
    EXPECT(p.score_of(key(0)) == 4);
    EXPECT_THROW(drain_prefetch(q, 1, -1, prof, p), std::invalid_argument);
  }
  {
    PrefetchQueues q(4);
    ResidencyPool p(4, 10, 20);
    const HardwareProfile prof = io_profile(1);
    p.admit(key(0), 2);
    q.enqueue(key(0), 4);
    q.enqueue(key(1), 4);
    q.enqueue(key(2), 3);
    const auto loads = drain_prefetch(q, 1, 1000, prof, p);
    EXPECT(loads.size() == 1 && loads[0].key == key(1));
    EXPECT(!q.contains(key(0)) && q.contains(key(2)) && p.free_bytes() == 0);
  }
  {
    PrefetchQueues q(4);
    ResidencyPool p(4, 10, 1000);
    q.enqueue(key(0), 2);
    q.enqueue(key(1), 4);
    const auto loads = drain_prefetch(q, 3, 1000, io_profile(1), p);
    EXPECT(loads.size() == 1 && loads[0].key == key(1) && q.contains(key(0)));
  }
  // randomized invariants (capacity, byte accounting, frozen supremacy,
  // non-increasing drain levels)
  std::mt19937_64 rng(321);
  for (int trial = 0; trial < 50; ++trial) {
    const int cap = 1 + static_cast<int>(rng() % 5);
    const std::int64_t capacity = 10 * (1 + static_cast<std::int64_t>(rng() % 8));
    PrefetchQueues q(cap);
    ResidencyPool p(cap, 10, capacity);
    const HardwareProfile prof = io_profile(1 + static_cast<std::int64_t>(rng() % 50));
    std::vector<ExpertKey> frozen;
    for (int op = 0; op < 300; ++op) {
      const int e = static_cast<int>(rng() % 16);
      switch (rng() % 7) {
        case 0: q.enqueue(key(e), 1 + static_cast<int>(rng() % cap)); break;
        case 1: p.admit(key(e), static_cast<int>(rng() % (cap + 1))); break;
        case 2: p.retag(key(e), static_cast<int>(rng() % (cap + 1))); break;
        case 3:
          if (p.resident(key(e)) && p.score_of(key(e)) != p.frozen_score()) {
            p.freeze(key(e));
            frozen.push_back(key(e));
          }
          break;
        case 4:
          if (!frozen.empty()) {
            p.thaw_and_recycle(frozen.back());
            frozen.pop_back();
          }
          break;
        case 5: {
          const int tau = 1 + static_cast<int>(rng() % cap);
          p.evict_below(tau);
          for (const auto& [k, s] : p.entries()) EXPECT(s == p.frozen_score() || s >= tau);
          break;
        }
        case 6: {
          const int tau = 1 + static_cast<int>(rng() % cap);
          std::int64_t budget = static_cast<std::int64_t>(rng() % 200);
          int last = cap + 1;
          const std::size_t before = q.pending();
          q.drain(tau, [&](ExpertKey k, int level) {
            EXPECT(level <= last);
            last = level;
            if (p.resident(k)) return true;
            if (prof.t_io_unit_ns > budget) return false;
            if (!p.admit(k, level)) return false;
            budget -= prof.t_io_unit_ns;
            return true;
          });
          EXPECT(q.pending() <= before);
          break;
        }
      }
      EXPECT(p.total_bytes() <= capacity);
      EXPECT(p.total_bytes() == static_cast<std::int64_t>(p.size()) * 10);
      for (ExpertKey k : frozen) EXPECT(p.resident(k));
    }
  }
}

static HardwareProfile basic() {
  HardwareProfile p;
  p.t_cpu_unit_ns = p.t_gpu_unit_ns = p.t_io_unit_ns = p.t_draft_unit_ns = 1000000;
  p.expert_bytes = 1000000;
  p.vram_capacity_bytes = 1000000000;
  return p;
}

static void balancer() {
  {
    HardwareProfile p = basic();
    RatioEstimates r;
    r.cpu_ratio = {0.0, 0.5, 1.0};
    r.gpu_ratio = {1.0, 1.0 / 3.0, 0.0};
    std::vector<int> scores(4, 0);
    std::unordered_set<int> res;
    BalancerInput in;
    in.scores = scores;
    in.resident = &res;
    in.gamma = 2;
    in.top_k = 2;
    in.b_est = 3;
    in.ratios = &r;
    in.profile = &p;
    in.utility_cap = 3;
    EXPECT(predicted_times(2, in).cpu_ns == 2000000 && predicted_times(2, in).gpu_ns == 1000000);
    EXPECT(predicted_times(1, in).cpu_ns == 0 && predicted_times(3, in).gpu_ns == 0);
    EXPECT_THROW(predicted_times(0, in), std::out_of_range);
    EXPECT_THROW(predicted_times(4, in), std::out_of_range);
  }
  {
    const std::vector<int> scores = {4, 2, 4, 3};
    const std::unordered_set<int> none, res = {0, 2}, all = {0, 1, 2, 3};
    EXPECT(count_prefetch(3, scores, none) == 3 && count_prefetch(1, scores, none) == 4);
    EXPECT(count_prefetch(5, scores, none) == 0 && count_prefetch(3, scores, res) == 1);
    EXPECT(count_prefetch(1, scores, all) == 0);
  }
  auto input = [](std::vector<int>& scores, std::unordered_set<int>& res, RatioEstimates& r, HardwareProfile& p,
                  int cap, int b) {
    BalancerInput in;
    in.scores = scores;
    in.resident = &res;
    in.gamma = 2;
    in.top_k = 2;
    in.b_est = b;
    in.ratios = &r;
    in.profile = &p;
    in.vram_left_bytes = p.vram_capacity_bytes;
    in.utility_cap = cap;
    return in;
  };
  {  // |diff| 3,1,1,3 ms: tie resolves to the smaller tau
    HardwareProfile p = basic();
    RatioEstimates r;
    r.cpu_ratio = {0.25, 0.5, 0.75, 1.0};
    r.gpu_ratio = {1.0, 0.75, 0.5, 0.25};
    std::vector<int> s(8, 0);
    std::unordered_set<int> res;
    const ThresholdDecision d = solve_threshold(input(s, res, r, p, 4, 4));
    EXPECT(d.tau == 2 && !d.fallback && d.predicted_t_cpu_ns == 2000000 && d.predicted_t_gpu_ns == 3000000);
  }
  {  // exact balance
    HardwareProfile p = basic();
    RatioEstimates r;
    r.cpu_ratio = {0.0, 0.75, 1.0};
    r.gpu_ratio = {1.0, 0.75, 0.5};
    std::vector<int> s(4, 0);
    std::unordered_set<int> res;
    const ThresholdDecision d = solve_threshold(input(s, res, r, p, 3, 4));
    EXPECT(d.tau == 2 && d.predicted_t_cpu_ns == d.predicted_t_gpu_ns);
  }
  {  // nothing feasible -> tau = K, fallback
    HardwareProfile p = basic();
    RatioEstimates r = RatioEstimates::uniform(4);
    std::vector<int> s(8, 4);
    std::unordered_set<int> res;
    BalancerInput in = input(s, res, r, p, 4, 4);
    in.vram_left_bytes = 0;
    const ThresholdDecision d = solve_threshold(in);
    EXPECT(d.fallback && d.tau == 4);
  }
  // brute force over random instances (workload_balancer_test.cpp:166-231)
  std::mt19937_64 rng(2024);
  std::uniform_real_distribution<double> u01(0.0, 1.0);
  int feasible = 0, fallback = 0;
  for (int trial = 0; trial < 1000; ++trial) {
    const int cap = 2 + static_cast<int>(rng() % 7), n = 4 + static_cast<int>(rng() % 29);
    RatioEstimates r;
    r.cpu_ratio.resize(static_cast<size_t>(cap));
    r.gpu_ratio.resize(static_cast<size_t>(cap));
    for (int i = 0; i < cap; ++i) {
      r.cpu_ratio[static_cast<size_t>(i)] = u01(rng);
      r.gpu_ratio[static_cast<size_t>(i)] = u01(rng);
    }
    std::sort(r.cpu_ratio.begin(), r.cpu_ratio.end());
    std::sort(r.gpu_ratio.begin(), r.gpu_ratio.end(), std::greater<>());
    HardwareProfile p = basic();
    p.t_cpu_unit_ns = 1 + static_cast<std::int64_t>(rng() % 2000);
    p.t_gpu_unit_ns = 1 + static_cast<std::int64_t>(rng() % 2000);
    p.t_io_unit_ns = 1 + static_cast<std::int64_t>(rng() % 4000);
    p.expert_bytes = 1 + static_cast<std::int64_t>(rng() % 100);
    std::vector<int> scores(static_cast<size_t>(n));
    for (int& s : scores) s = static_cast<int>(rng() % (cap + 1));
    std::unordered_set<int> res;
    for (int e = 0; e < n; ++e)
      if (rng() % 3 == 0) res.insert(e);
    BalancerInput in;
    in.scores = scores;
    in.resident = &res;
    in.gamma = 1 + static_cast<int>(rng() % 8);
    in.top_k = 1 + static_cast<int>(rng() % 8);
    in.b_est = 1 + static_cast<int>(rng() % 16);
    in.ratios = &r;
    in.profile = &p;
    in.vram_left_bytes = static_cast<std::int64_t>(rng() % (n + 1)) * p.expert_bytes;
    in.draft_credit_ns = static_cast<std::int64_t>(rng() % 5000);
    in.utility_cap = cap;
    int evals = 0;
    const ThresholdDecision got = solve_threshold(in, &evals);
    std::optional<std::int64_t> best;
    for (int tau = 1; tau <= cap; ++tau) {
      const PredictedTimes t = predicted_times(tau, in);
      const int np = count_prefetch(tau, scores, res);
      if (p.t_io_unit_ns * np > std::max(t.cpu_ns, t.gpu_ns) + in.draft_credit_ns) continue;
      if (p.expert_bytes * np > in.vram_left_bytes) continue;
      const std::int64_t obj = std::llabs(t.cpu_ns - t.gpu_ns);
      if (!best || obj < *best) best = obj;
    }
    if (!best) {
      EXPECT(got.fallback && got.tau == cap);
      ++fallback;
    } else {
      const PredictedTimes t = predicted_times(got.tau, in);
      EXPECT(!got.fallback && std::llabs(t.cpu_ns - t.gpu_ns) == *best);
      ++feasible;
    }
    EXPECT(evals <= 2 * static_cast<int>(std::ceil(std::log2(cap))) + 8);
  }
  EXPECT(feasible > 100 && fallback > 10);
  {  // ratio EMA + anchored clip
    RatioEstimates r;
    r.cpu_ratio = {0.1, 0.2, 0.3};
    r.gpu_ratio = {0.9, 0.8, 0.7};
    update_ratio_estimates(r, 2, 0.9, 0.1, 1.0);
    EXPECT(std::abs(r.cpu_ratio[1] - 0.9) < 1e-12 && std::abs(r.cpu_ratio[2] - 0.9) < 1e-12);
    EXPECT(std::abs(r.cpu_ratio[0] - 0.1) < 1e-12 && std::abs(r.gpu_ratio[2] - 0.1) < 1e-12);
    r.validate();
    EXPECT_THROW(update_ratio_estimates(r, 0, 0.5, 0.5, 0.5), std::out_of_range);
    EXPECT_THROW(update_ratio_estimates(r, 1, 1.5, 0.5, 0.5), std::invalid_argument);
    EXPECT_THROW(update_ratio_estimates(r, 1, 0.5, 0.5, 1.5), std::invalid_argument);
    std::mt19937_64 rr(77);
    RatioEstimates f = RatioEstimates::uniform(6);
    for (int i = 0; i < 2000; ++i) {
      update_ratio_estimates(f, 1 + static_cast<int>(rr() % 6), u01(rr), u01(rr), u01(rr));
      f.validate();
    }
  }
  {
    HardwareProfile z;
    EXPECT_THROW(z.validate(), std::invalid_argument);
    RatioEstimates bad;
    bad.cpu_ratio = {0.5, 0.4};
    bad.gpu_ratio = {0.5, 0.5};
    EXPECT_THROW(bad.validate(), std::invalid_argument);
  }
}

static void policies() {
  PolicySpec spec;
  spec.kind = PolicyKind::fixed_tau;
  spec.fixed_tau = 3;
  HardwareProfile p = basic();
  RatioEstimates r = RatioEstimates::uniform(4);
  std::vector<int> s = {4, 3, 1, 0};
  std::unordered_set<int> res = {0};
  BalancerInput in;
  in.scores = s;
  in.resident = &res;
  in.gamma = 8;
  in.top_k = 8;
  in.b_est = 8;
  in.ratios = &r;
  in.profile = &p;
  in.vram_left_bytes = p.vram_capacity_bytes;
  in.utility_cap = 4;
  const ThresholdDecision d = choose_threshold(spec, in);
  EXPECT(d.tau == 3 && !d.fallback && d.n_prefetch == 1);
  EXPECT(estimator_config_for({PolicyKind::binary_utility}, EstimatorConfig{}).utility_cap == 1);
  const EstimatorConfig fb = estimator_config_for({PolicyKind::fixed_boundaries, 2, 5, 2}, EstimatorConfig{});
  EXPECT(!fb.adaptive_boundaries && fb.init_up == 5 && fb.init_down == 2);
  EXPECT(is_utility_family(PolicyKind::ar_mode) && !is_utility_family(PolicyKind::lru_cache));
  EXPECT_THROW((PolicySpec{PolicyKind::fixed_tau, 9, 3, 1}).validate(4), std::invalid_argument);
}

int main() {
  queues();
  pool();
  drain();
  balancer();
  policies();
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
