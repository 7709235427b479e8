// Run metrics: summarize / emit / parse in the reference's `#moesim-metrics v1`
// schema (/root/reference/proj/core/src/metrics_report.cpp:12-183,
// core/include/moesim/metrics_report.hpp:15-46), over the StepReports the
// B200 step scheduler produces.
//
// summarize() follows metrics_report.cpp:12-55 (same accumulation order, so
// the doubles are bit-identical). emit() writes the same CSV bytes (shortest
// round-trip numbers via std::to_chars, as the reference does). JSONL rows
// have the reference's key order and number layout, with shortest
// round-trip digits; the reference's JSON library (nlohmann/json 3.11.3,
// Grisu2) prints a longer-than-shortest digit string for ~0.07% of doubles,
// so JSONL files are value-identical (parse -> the same doubles), not always
// byte-identical. parse_metrics() reads either format from either writer.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "step_scheduler.hpp"

namespace moespac {

struct RunSummary {
  std::string axis_name;
  double axis_value = 0.0;
  double tps = 0.0, latency_s = 0.0, hit_rate = 0.0, bubble_ratio = 0.0;
  double fault_rate = 0.0, fn_rate = 0.0, fp_rate = 0.0, mean_accuracy = 0.0;
  std::vector<double> accuracy_series;
  std::int64_t total_tokens = 0, total_time_ns = 0;
};

// std::invalid_argument on an empty run or one without time (as the reference).
RunSummary summarize(const std::vector<StepReport>& reports);

enum class MetricsFormat { csv, jsonl };
void emit(const std::vector<RunSummary>& summaries, MetricsFormat format, const std::string& path);
std::vector<RunSummary> parse_metrics(const std::string& path);

// shortest round-trip decimal (std::to_chars), the reference's CSV number form
std::string shortest(double v);

}  // namespace moespac
