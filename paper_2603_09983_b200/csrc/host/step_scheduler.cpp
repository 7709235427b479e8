#include "step_scheduler.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>

namespace moespac {

// sim_core.cpp:31-34
int layer_capacity_experts(double cache_ratio, int n_experts) {
  return static_cast<int>(std::floor(cache_ratio * n_experts + 1e-9));
}

// sim_core.cpp:36-64 — total = drafts + per (step, layer) max(cpu, gpu) + stall.
std::int64_t recompute_total_time(const std::vector<SimEvent>& log) {
  std::int64_t total = 0;
  std::map<std::pair<int, int>, std::int64_t[3]> seg;
  for (const SimEvent& e : log) {
    if (e.kind == SimEvent::Kind::draft) {
      total += e.duration_ns;
    } else if (e.kind == SimEvent::Kind::cpu || e.kind == SimEvent::Kind::gpu ||
               e.kind == SimEvent::Kind::stall) {
      auto& s = seg[{e.step, e.layer}];
      s[static_cast<int>(e.kind) - 1] += e.duration_ns;
    }
  }
  for (auto& [k, s] : seg) total += std::max(s[0], s[1]) + s[2];
  return total;
}

void SchedConfig::validate() const {
  if (n_layers < 1 || n_experts < 1 || top_k < 1 || top_k > n_experts || gamma < 1)
    throw std::invalid_argument("SchedConfig: invalid workload shape");
  if (n_experts > 4096) throw std::invalid_argument("SchedConfig: n_experts must be <= 4096");
  estimator.validate();
  if (!(cache_ratio > 0.0 && cache_ratio <= 1.0))
    throw std::invalid_argument("SimConfig: cache_ratio must be in (0,1]");
  if (!(ratio_smoothing >= 0.0 && ratio_smoothing <= 1.0))
    throw std::invalid_argument("SimConfig: ratio_smoothing in [0,1]");
  if (shard_world < 1 || shard_world > n_experts)
    throw std::invalid_argument("SchedConfig: shard_world must be in [1, N]");
  if (!is_utility_family(policy.kind))
    throw std::invalid_argument("SchedConfig: only utility-family policies drive the engine");
}

StepScheduler::StepScheduler(const SchedConfig& cfg) : cfg_(cfg) {
  // Simulation ctor, sim_core.cpp:78-120: derived profile fields first.
  cfg_.estimator.gamma = cfg_.gamma;
  cfg_.validate();
  const int L = cfg_.n_layers, N = cfg_.n_experts, G = cfg_.shard_world;
  c1_ = layer_capacity_experts(cfg_.cache_ratio, N);
  cfg_.profile.n_layers = L;
  cfg_.profile.vram_capacity_bytes = static_cast<std::int64_t>(L) * c1_ * cfg_.profile.expert_bytes;
  cfg_.profile.validate();
  cfg_.policy.validate(cfg_.estimator.utility_cap);
  const EstimatorConfig ec = estimator_config_for(cfg_.policy, cfg_.estimator);
  cap_ = ec.utility_cap;
  ar_ = cfg_.policy.kind == PolicyKind::ar_mode;
  words_ = (N + 31) / 32;

  shard_slots_.assign(static_cast<std::size_t>(G), 0);
  for (int s = 0; s < G; ++s) {
    const int shard_size = (N - s + G - 1) / G;
    shard_slots_[static_cast<std::size_t>(s)] = std::min(shard_size, c1_);
  }
  slot_of_.assign(static_cast<std::size_t>(L) * N, -1);
  layers_.reserve(static_cast<std::size_t>(L));
  for (int l = 0; l < L; ++l) {
    Layer ly;
    ly.ratios = RatioEstimates::uniform(cap_);
    ly.b_est = cfg_.top_k;
    for (int s = 0; s < G; ++s) {
      const int slots = shard_slots_[static_cast<std::size_t>(s)];
      ly.queues.emplace_back(cap_);
      ly.pools.emplace_back(cap_, cfg_.profile.expert_bytes,
                            static_cast<std::int64_t>(slots) * cfg_.profile.expert_bytes);
      std::vector<int> fs;
      for (int i = slots - 1; i >= 0; --i) fs.push_back(i);
      ly.free_slots.push_back(std::move(fs));
    }
    layers_.push_back(std::move(ly));
  }
  for (int l = 0; l < L; ++l) {
    for (int s = 0; s < G; ++s)
      layers_[static_cast<std::size_t>(l)].pools[static_cast<std::size_t>(s)].set_observer(
          [this, l](ExpertKey k, bool admitted) { admit_slot(l, k, admitted); });
    // Deterministic warm fill (sim_core.cpp:108-111): each shard fills its
    // slots with its lowest expert ids at score 0.
    std::vector<int> filled(static_cast<std::size_t>(G), 0);
    for (int e = 0; e < N; ++e) {
      const int s = e % G;
      if (filled[static_cast<std::size_t>(s)] < shard_slots_[static_cast<std::size_t>(s)]) {
        layers_[static_cast<std::size_t>(l)].pools[static_cast<std::size_t>(s)].admit({l, e}, 0);
        ++filled[static_cast<std::size_t>(s)];
      }
    }
  }
  resident_bits_.assign(static_cast<std::size_t>(L) * words_, 0u);
  loaded_bits_.assign(static_cast<std::size_t>(L) * words_, 0u);
  taus_.assign(static_cast<std::size_t>(L), 1);
  decisions_.resize(static_cast<std::size_t>(L));
  for (int l = 0; l < L; ++l) {
    std::uint32_t* bits = resident_bits_.data() + static_cast<std::size_t>(l) * words_;
    std::fill(bits, bits + words_, 0u);
    for (int e = 0; e < N; ++e)
      if (slot_of_[static_cast<std::size_t>(l) * N + e] >= 0) bits[e >> 5] |= 1u << (e & 31);
  }
}

void StepScheduler::admit_slot(int layer, ExpertKey key, bool admitted) {
  const int N = cfg_.n_experts, s = key.expert % cfg_.shard_world;
  auto& fs = layers_[static_cast<std::size_t>(layer)].free_slots[static_cast<std::size_t>(s)];
  std::int32_t& slot = slot_of_[static_cast<std::size_t>(layer) * N + key.expert];
  if (admitted) {
    if (fs.empty()) throw std::logic_error("slot allocator: pool admitted beyond its slots");
    slot = fs.back();
    fs.pop_back();
  } else {
    if (slot < 0) throw std::logic_error("slot allocator: evicting an unslotted expert");
    fs.push_back(slot);
    slot = -1;
  }
}

void StepScheduler::decide(const std::int32_t* scores) {
  const int L = cfg_.n_layers, N = cfg_.n_experts, G = cfg_.shard_world;
  const HardwareProfile& prof = cfg_.profile;
  loads_.clear();
  std::fill(loaded_bits_.begin(), loaded_bits_.end(), 0u);
  for (int l = 0; l < L; ++l) {
    Layer& ly = layers_[static_cast<std::size_t>(l)];
    ly.snapshot.assign(scores + static_cast<std::size_t>(l) * N, scores + static_cast<std::size_t>(l + 1) * N);
    const std::vector<int>& sc = ly.snapshot;
    std::uint32_t* rbits = resident_bits_.data() + static_cast<std::size_t>(l) * words_;
    std::fill(rbits, rbits + words_, 0u);
    std::int64_t vram = 0;
    for (int s = 0; s < G; ++s) vram += ly.pools[static_cast<std::size_t>(s)].capacity_bytes();
    for (int e = 0; e < N; ++e)
      if (slot_of_[static_cast<std::size_t>(l) * N + e] >= 0) rbits[e >> 5] |= 1u << (e & 31);

    BalancerInput in;
    in.scores = std::span<const int>(sc.data(), sc.size());
    in.resident_view = ResidentView(rbits, N);
    in.gamma = ar_ ? 1 : cfg_.gamma;
    in.top_k = cfg_.top_k;
    in.b_est = ly.b_est;
    in.ratios = &ly.ratios;
    in.profile = &prof;
    in.vram_left_bytes = vram;  // residents below tau are reclaimable (sim_core.cpp:193-195)
    in.utility_cap = cap_;
    in.draft_credit_ns = ar_ ? 0 : BalancerInput::default_draft_credit(cfg_.gamma, prof);
    const ThresholdDecision dec = choose_threshold(cfg_.policy, in);
    decisions_[static_cast<std::size_t>(l)] = dec;
    taus_[static_cast<std::size_t>(l)] = dec.tau;
    ly.draft_credit = in.draft_credit_ns;

    const std::int64_t io_budget = std::max(dec.predicted_t_cpu_ns, dec.predicted_t_gpu_ns) + in.draft_credit_ns;
    ly.evicted.clear();
    ly.loaded.clear();
    for (int s = 0; s < G; ++s) {
      ResidencyPool& pool = ly.pools[static_cast<std::size_t>(s)];
      PrefetchQueues& q = ly.queues[static_cast<std::size_t>(s)];
      // retag residents to the fresh snapshot (sim_core.cpp:204)
      for (const auto& [key, score] : pool.entries()) pool.retag(key, sc[static_cast<std::size_t>(key.expert)]);
      // shard-local prefetch count; for G == 1 equals dec.n_prefetch
      int n_pf = dec.n_prefetch;
      if (G > 1) {
        n_pf = 0;
        for (int e = s; e < N; e += G)
          n_pf += (sc[static_cast<std::size_t>(e)] >= dec.tau && !pool.resident({l, e})) ? 1 : 0;
      }
      const std::int64_t loadable = std::min<std::int64_t>(n_pf, io_budget / prof.t_io_unit_ns);
      for (ExpertKey k : pool.evict_for_room(loadable * prof.expert_bytes, dec.tau)) ly.evicted.push_back(k.expert);
      q.scrub([&](ExpertKey key, int level) {
        return sc[static_cast<std::size_t>(key.expert)] == level && !pool.resident(key);
      });
      for (int e = s; e < N; e += G)
        if (sc[static_cast<std::size_t>(e)] >= 1 && !pool.resident({l, e})) q.enqueue({l, e}, sc[static_cast<std::size_t>(e)]);
      for (const IoEvent& ev : drain_prefetch(q, dec.tau, io_budget, prof, pool, 0)) {
        const int e = ev.key.expert;
        ly.loaded.push_back(e);
        loads_.push_back({l, e, s, slot_of_[static_cast<std::size_t>(l) * N + e]});
      }
    }
    std::fill(rbits, rbits + words_, 0u);
    std::uint32_t* lbits = loaded_bits_.data() + static_cast<std::size_t>(l) * words_;
    for (int e = 0; e < N; ++e)
      if (slot_of_[static_cast<std::size_t>(l) * N + e] >= 0) rbits[e >> 5] |= 1u << (e & 31);
    for (int e : ly.loaded) lbits[e >> 5] |= 1u << (e & 31);
  }
  decided_ = true;
}

LayerOutcome StepScheduler::split_on_host(int l, const std::int32_t* freqs) const {
  const int N = cfg_.n_experts;
  const std::uint32_t* rbits = resident_bits_.data() + static_cast<std::size_t>(l) * words_;
  const std::uint32_t* lbits = loaded_bits_.data() + static_cast<std::size_t>(l) * words_;
  const std::vector<int>& sc = layers_[static_cast<std::size_t>(l)].snapshot;
  const int tau = taus_[static_cast<std::size_t>(l)];
  LayerOutcome o;
  for (int e = 0; e < N; ++e) {
    const int f = freqs[e];
    const bool res = (rbits[e >> 5] >> (e & 31)) & 1u;
    if (f > 0) {
      ++o.distinct;
      if (res) {
        ++o.distinct_hits;
        o.hit_tokens += f;
      } else {
        o.miss_tokens += f;
      }
    }
    o.agree += ((sc[static_cast<std::size_t>(e)] >= 1) == (f >= 1)) ? 1 : 0;
    o.faults_fn += (f >= 1 && sc[static_cast<std::size_t>(e)] < tau) ? 1 : 0;
    o.faults_fp += (((lbits[e >> 5] >> (e & 31)) & 1u) && f == 0) ? 1 : 0;
  }
  return o;
}

StepReport StepScheduler::observe_freqs(const std::int32_t* freqs, int accepted_count) {
  if (!decided_) throw std::logic_error("StepScheduler: observe() without decide()");
  std::vector<LayerOutcome> out(static_cast<std::size_t>(cfg_.n_layers));
  for (int l = 0; l < cfg_.n_layers; ++l)
    out[static_cast<std::size_t>(l)] = split_on_host(l, freqs + static_cast<std::size_t>(l) * cfg_.n_experts);
  return observe(out.data(), accepted_count);
}

// Accounting half of sim_core.cpp:157-316 with the realized split supplied.
StepReport StepScheduler::observe(const LayerOutcome* outcomes, int accepted_count) {
  if (!decided_) throw std::logic_error("StepScheduler: observe() without decide()");
  decided_ = false;
  const int L = cfg_.n_layers, N = cfg_.n_experts;
  const HardwareProfile& prof = cfg_.profile;
  const int window = ar_ ? 1 : cfg_.gamma + 1;
  StepReport rep;
  rep.n_experts = N;
  rep.accepted_tokens = ar_ ? 1 : accepted_count;
  rep.draft_ns = ar_ ? 0 : static_cast<std::int64_t>(cfg_.gamma) * prof.t_draft_unit_ns;
  if (rep.draft_ns > 0) events_.push_back({SimEvent::Kind::draft, step_, -1, -1, clock_ns_, rep.draft_ns});
  std::int64_t t = clock_ns_ + rep.draft_ns;
  double acc_sum = 0.0;
  for (int l = 0; l < L; ++l) {
    Layer& ly = layers_[static_cast<std::size_t>(l)];
    const ThresholdDecision& dec = decisions_[static_cast<std::size_t>(l)];
    const LayerOutcome& o = outcomes[l];
    for (int e : ly.evicted) events_.push_back({SimEvent::Kind::evict, step_, l, e, t, 0});
    // Loads are back to back per shard's copy engine (drain_prefetch start
    // offsets); with G == 1 this is the reference's single engine.
    std::vector<std::int64_t> shard_clock(static_cast<std::size_t>(cfg_.shard_world), 0);
    std::int64_t io_used = 0;
    for (int e : ly.loaded) {
      std::int64_t& c = shard_clock[static_cast<std::size_t>(e % cfg_.shard_world)];
      events_.push_back({SimEvent::Kind::load, step_, l, e, t + c, prof.t_io_unit_ns});
      c += prof.t_io_unit_ns;
      io_used = std::max(io_used, c);
    }
    LayerTiming lt;
    lt.tau = dec.tau;
    lt.fallback = dec.fallback;
    lt.n_prefetch = dec.n_prefetch;
    lt.t_cpu_ns = static_cast<std::int64_t>(o.miss_tokens) * prof.t_cpu_unit_ns;
    lt.t_gpu_ns = static_cast<std::int64_t>(o.distinct_hits) * prof.t_gpu_unit_ns;
    lt.t_io_used_ns = io_used;
    const std::int64_t busy = std::max(lt.t_cpu_ns, lt.t_gpu_ns);
    lt.stall_ns = std::max<std::int64_t>(0, io_used - (busy + ly.draft_credit));
    lt.wall_ns = busy + lt.stall_ns;
    lt.bubble_ns = std::llabs(lt.t_cpu_ns - lt.t_gpu_ns) + lt.stall_ns;
    if (lt.t_cpu_ns > 0) events_.push_back({SimEvent::Kind::cpu, step_, l, -1, t, lt.t_cpu_ns});
    if (lt.t_gpu_ns > 0) events_.push_back({SimEvent::Kind::gpu, step_, l, -1, t, lt.t_gpu_ns});
    if (lt.stall_ns > 0) events_.push_back({SimEvent::Kind::stall, step_, l, -1, t + busy, lt.stall_ns});
    t += lt.wall_ns;
    rep.cache_hits += o.hit_tokens;
    rep.cache_misses += o.miss_tokens;
    rep.faults_fn += o.faults_fn;
    rep.faults_fp += o.faults_fp;
    acc_sum += static_cast<double>(o.agree) / N;
    // freeze/thaw_and_recycle (sim_core.cpp:247, :285) only move pool tags
    // that the next decide()'s retag overwrites before any read (SURVEY.md
    // §3.2), so the host skips them; on the device the same protection is
    // the per-slot completion event that gates every load into a slot.
    const double rc = std::clamp(static_cast<double>(o.miss_tokens) /
                                     (static_cast<double>(window) * cfg_.top_k),
                                 0.0, 1.0);
    const double rg = o.distinct > 0 ? static_cast<double>(o.distinct_hits) / o.distinct : 0.0;
    update_ratio_estimates(ly.ratios, dec.tau, rc, rg, cfg_.ratio_smoothing);
    ly.b_est = std::max(static_cast<int>(o.distinct), 1);
    rep.layers.push_back(lt);
  }
  rep.accuracy = acc_sum / L;
  rep.step_wall_ns = t - clock_ns_;
  clock_ns_ = t;
  tokens_ += rep.accepted_tokens;
  ++step_;
  return rep;
}

}  // namespace moespac
