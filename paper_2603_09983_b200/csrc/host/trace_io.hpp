// Routing-trace wire format `#moetrace v1` — the reference's trace file
// (/root/reference/proj/core/src/trace_model.cpp:132-254,
// core/include/moesim/trace_model.hpp:76-81), restated for the B200 path so
// recorded routing can be replayed through K2-K4 (moespac_step_ids) and
// synthetic routing can be exported in the reference's format.
//
//   #moetrace v1 layers=L experts=N k=K gamma=G
//   <step> <layer> <accepted> <id,id,..> x (gamma+1)      one line per (step, layer)
//
// Same validation and the same error text as the reference reader: every
// failure is std::runtime_error("read_trace: <path>:<line>: <what>") except a
// non-numeric header value (std::invalid_argument / std::out_of_range from
// the integer conversion, as std::stoi does).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace moespac {

struct TraceData {
  int n_layers = 0, n_experts = 0, top_k = 0, gamma = 0;
  std::vector<std::int32_t> accepted;  // [S]
  std::vector<std::int32_t> ids;       // [S][L][gamma+1][k], ids in file order
  std::int64_t steps() const { return static_cast<std::int64_t>(accepted.size()); }
};

// trace_model.cpp:132-155
void write_trace(const TraceData& trace, const std::string& path);
// trace_model.cpp:166-254 (an empty file is an empty trace)
TraceData read_trace(const std::string& path);

}  // namespace moespac
