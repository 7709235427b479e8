// The reference's utility_estimator_test.cpp and trace_model_test.cpp
// scenarios (proj/tests/), re-expressed against the B200 build's host
// operator API: LayerEstimator (csrc/host/estimator.hpp) and the routing
// workload (csrc/host/trace_model.hpp). Same calls and expected values as
// the reference cases they cite; built and run by tests/test_cpp_api.py.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "estimator.hpp"
#include "trace_model.hpp"

using namespace moespac;

static int g_checks = 0, g_fail = 0;
#define EXPECT(cond)                                                                 \
  do {                                                                               \
    ++g_checks;                                                                      \
    if (!(cond)) {                                                                   \
      ++g_fail;                                                                      \
      std::fprintf(stderr, "%s:%d: EXPECT(%s) failed\n", __FILE__, __LINE__, #cond); \
    }                                                                                \
  } while (0)
#define EXPECT_THROW(stmt)  \
  do {                      \
    bool thrown = false;    \
    try {                   \
      stmt;                 \
    } catch (...) {         \
      thrown = true;        \
    }                       \
    EXPECT(thrown);         \
  } while (0)

static EstimatorConfig ecfg(int cap = 4, double lambda = 0.1, int gamma = 8) {
  EstimatorConfig c;
  c.utility_cap = cap;
  c.forgetting = lambda;
  c.gamma = gamma;
  return c;
}

static LayerEstimator from_record(const char* rec, int n, EstimatorConfig c) {
  std::istringstream in(rec);
  return LayerEstimator::load(in, n, c);
}

static void estimator() {
  // utility_estimator_test.cpp:25-43 — boundaries start at floor(gamma / 2)
  {
    LayerEstimator a(128, ecfg(4, 0.1, 8));
    bool all = true;
    for (int e = 0; e < 128; ++e) {
      const ExpertUtilityState& s = a.state(e);
      all = all && s.score == 0 && s.up_boundary == 4 && s.down_boundary == 4 && s.last_freq == 0;
    }
    EXPECT(all);
    EXPECT(LayerEstimator(1, ecfg(2, 0.1, 2)).state(0).up_boundary == 1);
    EXPECT(LayerEstimator(64, ecfg(1, 0.1, 3)).state(0).up_boundary == 1);
  }
  // :45-52 — explicit initial boundaries
  {
    EstimatorConfig c = ecfg();
    c.init_up = 3;
    c.init_down = 1;
    LayerEstimator a(4, c);
    EXPECT(a.state(0).up_boundary == 3 && a.state(0).down_boundary == 1);
  }
  // :54-62 — validation
  EXPECT_THROW(LayerEstimator(4, ecfg(0)));
  EXPECT_THROW(LayerEstimator(4, ecfg(4, -0.1)));
  EXPECT_THROW(LayerEstimator(4, ecfg(4, 0.1, 0)));
  EXPECT_THROW(LayerEstimator(4, ecfg(5, 0.1, 4)));
  EXPECT_THROW(LayerEstimator(0, ecfg()));
  {
    LayerEstimator a(2, ecfg());
    EXPECT_THROW(a.observe_step(std::vector<int>{1, 2, 3}));
  }
  // :64-81 — worked transition: s = 2, theta-up = 4, f 1 -> 6 gives s = 3,
  // theta-up = floor(0.9 * 4 + 0.1 * 5) = 4
  {
    LayerEstimator a(1, ecfg(4, 0.1, 8));
    a.observe_step(std::vector<int>{1});
    EXPECT(a.state(0).score == 0);
    a.observe_step(std::vector<int>{7});
    a.observe_step(std::vector<int>{13});
    EXPECT(a.state(0).score == 2);
    LayerEstimator w = from_record("0 0 2 4 4 1\n", 1, ecfg(4, 0.1, 8));
    w.observe_step(std::vector<int>{6});
    EXPECT(w.state(0).score == 3 && w.state(0).up_boundary == 4 && w.state(0).last_freq == 6);
  }
  // :83-90 — a zero fluctuation changes nothing
  {
    LayerEstimator a = from_record("0 0 2 3 2 5\n", 1, ecfg(4, 0.1, 8));
    a.observe_step(std::vector<int>{5});
    EXPECT(a.state(0).score == 2 && a.state(0).up_boundary == 3 && a.state(0).down_boundary == 2);
  }
  // :92-109 — scores saturate at K and at 0
  {
    LayerEstimator a(1, ecfg(2, 0.0, 2));
    int f = 0;
    for (int i = 0; i < 5; ++i) a.observe_step(std::vector<int>{f += 3});
    EXPECT(a.state(0).score == 2);
    while (f > 0) a.observe_step(std::vector<int>{f = std::max(0, f - 3)});
    for (int i = 0; i < 5; ++i) a.observe_step(std::vector<int>{0});
    EXPECT(a.state(0).score == 0);
  }
  // :111-120 — only the boundary on the fluctuation's side moves (lambda 0.2):
  // +4 -> theta-up floor(5.6) = 5; -10 -> theta-down floor(6.8) = 6
  {
    LayerEstimator a = from_record("0 0 1 6 6 10\n", 1, ecfg(4, 0.2, 8));
    a.observe_step(std::vector<int>{14});
    EXPECT(a.state(0).up_boundary == 5 && a.state(0).down_boundary == 6);
    a.observe_step(std::vector<int>{4});
    EXPECT(a.state(0).up_boundary == 5 && a.state(0).down_boundary == 6);
  }
  // :122-131 — boundaries never drop below 1 (lambda 1)
  {
    LayerEstimator a = from_record("0 0 0 1 1 0\n", 1, ecfg(4, 1.0, 8));
    a.observe_step(std::vector<int>{1});
    EXPECT(a.state(0).up_boundary == 1);
    a.observe_step(std::vector<int>{0});
    EXPECT(a.state(0).down_boundary == 1);
  }
  // :133-143 — lambda 0 freezes the boundaries
  {
    LayerEstimator a(1, ecfg(4, 0.0, 8));
    std::mt19937_64 rng(11);
    bool frozen = true;
    for (int i = 0; i < 200; ++i) {
      a.observe_step(std::vector<int>{static_cast<int>(rng() % 10)});
      frozen = frozen && a.state(0).up_boundary == 4 && a.state(0).down_boundary == 4;
    }
    EXPECT(frozen);
  }
  // :145-157 — adaptive boundaries off pins them at their initial values
  {
    EstimatorConfig c = ecfg(4, 0.5, 8);
    c.adaptive_boundaries = false;
    c.init_up = 3;
    c.init_down = 1;
    LayerEstimator a(1, c);
    std::mt19937_64 rng(12);
    bool pinned = true;
    for (int i = 0; i < 100; ++i) {
      a.observe_step(std::vector<int>{static_cast<int>(rng() % 9)});
      pinned = pinned && a.state(0).up_boundary == 3 && a.state(0).down_boundary == 1;
    }
    EXPECT(pinned);
  }
  // :159-174 — fluctuations inside the hysteresis band never move the score
  {
    std::mt19937_64 rng(42);
    bool still = true;
    for (int trial = 0; trial < 300; ++trial) {
      LayerEstimator a(1, ecfg(4, 0.3, 8));
      for (int step = 0; step < 50; ++step) {
        const ExpertUtilityState& s = a.state(0);
        const int lo = std::max(0, s.last_freq - s.down_boundary + 1), hi = s.last_freq + s.up_boundary - 1;
        a.observe_step(std::vector<int>{lo + static_cast<int>(rng() % (hi - lo + 1))});
        still = still && a.state(0).score == 0;
      }
    }
    EXPECT(still);
  }
  // :176-204 — fuzz: bounds, unit steps, determinism
  {
    std::mt19937_64 rng(99);
    bool ok = true;
    for (int trial = 0; trial < 500; ++trial) {
      const int cap = 1 + static_cast<int>(rng() % 4);
      const int gamma = std::max(2, cap) + static_cast<int>(rng() % 8);
      const double lambda = static_cast<double>(rng() % 11) / 10.0;
      LayerEstimator a(3, ecfg(cap, lambda, gamma)), b(3, ecfg(cap, lambda, gamma));
      for (int step = 0; step < 40; ++step) {
        std::vector<int> before = a.snapshot_scores(), f(3);
        for (int& x : f) x = static_cast<int>(rng() % static_cast<unsigned>(gamma + 2));
        a.observe_step(f);
        b.observe_step(f);
        for (int e = 0; e < 3; ++e) {
          const ExpertUtilityState& s = a.state(e);
          ok = ok && s.score >= 0 && s.score <= cap && std::abs(s.score - before[static_cast<size_t>(e)]) <= 1 &&
               s.up_boundary >= 1 && s.down_boundary >= 1 && s.score == b.state(e).score &&
               s.up_boundary == b.state(e).up_boundary;
        }
      }
    }
    EXPECT(ok);
  }
  // :206-228 — checkpoint round trip, truncated / malformed checkpoints
  {
    LayerEstimator a(5, ecfg(4, 0.25, 8));
    std::mt19937_64 rng(5);
    for (int step = 0; step < 30; ++step) {
      std::vector<int> f(5);
      for (int& x : f) x = static_cast<int>(rng() % 10);
      a.observe_step(f);
    }
    std::ostringstream out;
    a.dump(out, 3);
    std::istringstream in(out.str());
    LayerEstimator b = LayerEstimator::load(in, 5, ecfg(4, 0.25, 8));
    bool same = true;
    for (int e = 0; e < 5; ++e)
      same = same && b.state(e).score == a.state(e).score && b.state(e).up_boundary == a.state(e).up_boundary &&
             b.state(e).down_boundary == a.state(e).down_boundary && b.state(e).last_freq == a.state(e).last_freq;
    EXPECT(same);
    EXPECT(out.str().rfind("3 4 ", 0) != std::string::npos || out.str().find("\n3 4 ") != std::string::npos);
    EXPECT_THROW(from_record("0 0 1 2 3 4\n", 2, ecfg()));
    EXPECT_THROW(from_record("0 zero 1 2 3 4\n", 1, ecfg()));
    EXPECT_THROW(from_record("0 7 1 2 3 4\n", 1, ecfg()));  // expert id out of range
    // device layout round trip (the engine's checkpoint path)
    std::vector<std::int32_t> dev(20);
    a.to_device_layout(dev.data());
    LayerEstimator c(5, ecfg(4, 0.25, 8));
    c.from_device_layout(dev.data());
    EXPECT(c.snapshot_scores() == a.snapshot_scores() && c.state(4).last_freq == a.state(4).last_freq);
  }
}

static TraceConfig small_trace() {  // trace_model_test.cpp:24-36
  TraceConfig c;
  c.n_layers = 3;
  c.n_experts = 16;
  c.top_k = 4;
  c.gamma = 4;
  c.alpha = 0.8;
  c.drift_scale = 0.05;
  c.route_noise = 0.3;
  c.seed = 42;
  return c;
}

static void trace_model() {
  // trace_model_test.cpp:45-58 — config validation
  {
    TraceConfig c = small_trace();
    c.top_k = 17;
    EXPECT_THROW(c.validate());
    c = small_trace();
    c.gamma = 0;
    EXPECT_THROW(c.validate());
    c = small_trace();
    c.alpha = 1.2;
    EXPECT_THROW(c.validate());
    c = small_trace();
    c.drift_scale = -0.1;
    EXPECT_THROW(c.validate());
  }
  // :60-94 — accept-length pmf: alpha^(i-1)(1 - alpha) below gamma + 1, alpha^gamma at the top
  {
    std::mt19937_64 rng(7);
    const int gamma = 4, trials = 200000;
    const double alpha = 0.8;
    std::vector<int> hist(gamma + 2, 0);
    long long total = 0;
    bool in_range = true;
    for (int i = 0; i < trials; ++i) {
      const int n = sample_accept_length(alpha, gamma, rng);
      in_range = in_range && n >= 1 && n <= gamma + 1;
      ++hist[static_cast<size_t>(std::clamp(n, 0, gamma + 1))];
      total += n;
    }
    EXPECT(in_range);
    // closed-form expected tokens (1 - alpha^(gamma+1)) / (1 - alpha)
    const double omega = (1.0 - std::pow(alpha, gamma + 1)) / (1.0 - alpha);
    EXPECT(std::abs(static_cast<double>(total) / trials - omega) / omega < 0.01);
    for (int i = 1; i <= gamma; ++i)
      EXPECT(std::abs(static_cast<double>(hist[static_cast<size_t>(i)]) / trials -
                      std::pow(alpha, i - 1) * (1 - alpha)) < 0.01);
    EXPECT(std::abs(static_cast<double>(hist[gamma + 1]) / trials - std::pow(alpha, gamma)) < 0.01);
    bool degenerate = true;
    for (int i = 0; i < 50; ++i)
      degenerate = degenerate && sample_accept_length(0.0, 8, rng) == 1 && sample_accept_length(1.0, 8, rng) == 9;
    EXPECT(degenerate);
    EXPECT(sample_accept_length(0.5, 0, rng) == 1);
    EXPECT_THROW(sample_accept_length(-0.1, 4, rng));
    EXPECT_THROW(sample_accept_length(0.5, -1, rng));
  }
  // :96-117 — generated steps are well formed
  {
    const Trace t = TraceGenerator(small_trace()).generate(20);
    bool ok = t.steps.size() == 20;
    for (const StepActivations& s : t.steps) {
      ok = ok && s.accepted_count >= 1 && s.accepted_count <= 5 && s.experts.size() == 3;
      for (const auto& layer : s.experts) {
        ok = ok && layer.size() == 5;
        for (const auto& tok : layer) {
          const std::set<int> distinct(tok.begin(), tok.end());
          ok = ok && tok.size() == 4 && distinct.size() == 4 && std::is_sorted(tok.begin(), tok.end()) &&
               *std::min_element(tok.begin(), tok.end()) >= 0 && *std::max_element(tok.begin(), tok.end()) < 16;
        }
      }
    }
    EXPECT(ok);
  }
  // :119-127 — same seed, same trace; another seed, another trace
  {
    const Trace a = TraceGenerator(small_trace()).generate(30), b = TraceGenerator(small_trace()).generate(30);
    EXPECT(a == b);
    TraceConfig o = small_trace();
    o.seed = 43;
    EXPECT(!(a == TraceGenerator(o).generate(30)));
  }
  // :129-139 — no drift, no noise: every token picks the same top-k
  {
    TraceConfig c = small_trace();
    c.drift_scale = 0.0;
    c.route_noise = 0.0;
    const Trace t = TraceGenerator(c).generate(10);
    bool pinned = true;
    for (const StepActivations& s : t.steps)
      for (size_t l = 0; l < s.experts.size(); ++l)
        for (const auto& tok : s.experts[l]) pinned = pinned && tok == t.steps[0].experts[l][0];
    EXPECT(pinned);
  }
  // :141-159 — lower drift, less churn of the hot set
  {
    auto churn = [](double drift) {
      TraceConfig c = small_trace();
      c.drift_scale = drift;
      c.route_noise = 0.0;
      const Trace t = TraceGenerator(c).generate(60);
      int changes = 0;
      for (size_t s = 1; s < t.steps.size(); ++s) {
        const std::set<int> prev(t.steps[s - 1].experts[0][0].begin(), t.steps[s - 1].experts[0][0].end());
        for (int e : t.steps[s].experts[0][0]) changes += prev.count(e) ? 0 : 1;
      }
      return changes;
    };
    EXPECT(churn(0.0) == 0);
    EXPECT(churn(0.02) <= churn(0.5));
  }
  // :161-168 — activation_frequencies
  {
    StepActivations s;
    s.experts = {{{0, 1}, {0, 2}, {1, 0}}};
    s.accepted_count = 2;
    EXPECT((activation_frequencies(s, 0, 4) == std::vector<int>{3, 2, 1, 0}));
    EXPECT_THROW(activation_frequencies(s, 1, 4));
  }
  // :170-176 — trace file round trip is exact
  {
    const Trace t = TraceGenerator(small_trace()).generate(25);
    const std::string path = "/tmp/moespac_test_roundtrip.trace";
    write_trace_steps(t, path);
    EXPECT(read_trace_steps(path) == t);
    std::remove(path.c_str());
  }
}

int main() {
  estimator();
  trace_model();
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
