#include "trace_io.hpp"

#include <cerrno>
#include <climits>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <stdexcept>

namespace moespac {

namespace {

// std::stoi semantics (strtol base 10: leading blanks, optional sign, the
// longest digit prefix; no digits -> invalid_argument, overflow ->
// out_of_range), so header values and expert ids parse exactly as the
// reference's reader parses them.
int stoi_like(const std::string& s) {
  const char* b = s.c_str();
  char* end = nullptr;
  errno = 0;
  const long v = std::strtol(b, &end, 10);
  if (end == b) throw std::invalid_argument("stoi");
  if (errno == ERANGE || v < INT_MIN || v > INT_MAX) throw std::out_of_range("stoi");
  return static_cast<int>(v);
}

[[noreturn]] void fail(const std::string& path, int line_no, const std::string& what) {
  throw std::runtime_error("read_trace: " + path + ":" + std::to_string(line_no) + ": " + what);
}

}  // namespace

void write_trace(const TraceData& tr, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("write_trace: cannot open " + path);
  out << "#moetrace v1 layers=" << tr.n_layers << " experts=" << tr.n_experts << " k=" << tr.top_k
      << " gamma=" << tr.gamma << '\n';
  const int T = tr.gamma + 1, k = tr.top_k;
  const std::size_t per_layer = static_cast<std::size_t>(T) * k;
  for (std::int64_t s = 0; s < tr.steps(); ++s) {
    for (int l = 0; l < tr.n_layers; ++l) {
      out << s << ' ' << l << ' ' << tr.accepted[static_cast<std::size_t>(s)];
      const std::int32_t* row = tr.ids.data() + (static_cast<std::size_t>(s) * tr.n_layers + l) * per_layer;
      for (int t = 0; t < T; ++t) {
        out << ' ';
        for (int j = 0; j < k; ++j) {
          if (j) out << ',';
          out << row[t * k + j];
        }
      }
      out << '\n';
    }
  }
  if (!out) throw std::runtime_error("write_trace: write failed on " + path);
}

TraceData read_trace(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("read_trace: cannot open " + path);
  TraceData tr;
  std::string line;
  int line_no = 1;
  if (!std::getline(in, line)) return tr;
  {
    std::istringstream hs(line);
    std::string magic, version, field;
    hs >> magic >> version;
    if (magic != "#moetrace" || version != "v1") fail(path, line_no, "bad header magic");
    while (hs >> field) {
      const auto eq = field.find('=');
      if (eq == std::string::npos) fail(path, line_no, "bad header field");
      const std::string key = field.substr(0, eq);
      const int value = stoi_like(field.substr(eq + 1));
      if (key == "layers") tr.n_layers = value;
      else if (key == "experts") tr.n_experts = value;
      else if (key == "k") tr.top_k = value;
      else if (key == "gamma") tr.gamma = value;
      else fail(path, line_no, "unknown header key " + key);
    }
    if (tr.n_layers < 1 || tr.n_experts < 1 || tr.top_k < 1 || tr.gamma < 1) fail(path, line_no, "incomplete header");
  }
  const int T = tr.gamma + 1, k = tr.top_k, L = tr.n_layers;
  const std::size_t per_layer = static_cast<std::size_t>(T) * k;
  std::vector<char> seen;  // [S][L]: record present
  while (std::getline(in, line)) {
    ++line_no;
    if (line.empty()) continue;
    std::istringstream ls(line);
    int step, layer, accepted;
    if (!(ls >> step >> layer >> accepted)) fail(path, line_no, "malformed record prefix");
    const int S = static_cast<int>(tr.accepted.size());
    if (step != S - 1 && step != S) fail(path, line_no, "step index out of order");
    if (step == S) {
      tr.accepted.push_back(accepted);
      tr.ids.resize(tr.ids.size() + static_cast<std::size_t>(L) * per_layer, 0);
      seen.resize(seen.size() + static_cast<std::size_t>(L), 0);
    }
    if (layer < 0 || layer >= L) fail(path, line_no, "layer out of range");
    if (accepted != tr.accepted.back()) fail(path, line_no, "inconsistent accepted count");
    if (accepted < 1 || accepted > T) fail(path, line_no, "accepted count out of range");
    const std::size_t rec = (tr.accepted.size() - 1) * static_cast<std::size_t>(L) + static_cast<std::size_t>(layer);
    if (seen[rec]) fail(path, line_no, "duplicate (step, layer) record");
    // the reference marks the record present once a token group was parsed;
    // a record without groups fails below either way
    std::int32_t* row = tr.ids.data() + rec * per_layer;
    int n_groups = 0;
    std::string group;
    while (ls >> group) {
      std::vector<int> ids;
      std::istringstream gs(group);
      std::string id;
      while (std::getline(gs, id, ',')) {
        try {
          ids.push_back(stoi_like(id));
        } catch (const std::exception&) {
          fail(path, line_no, "bad expert id '" + id + "'");
        }
      }
      if (static_cast<int>(ids.size()) != k) fail(path, line_no, "token group is not top-k sized");
      for (int e : ids)
        if (e < 0 || e >= tr.n_experts) fail(path, line_no, "expert id out of range");
      if (n_groups < T)
        for (int j = 0; j < k; ++j) row[static_cast<std::size_t>(n_groups) * k + j] = ids[static_cast<std::size_t>(j)];
      ++n_groups;
      seen[rec] = 1;
    }
    if (n_groups != T) fail(path, line_no, "expected gamma+1 token groups");
  }
  for (std::size_t s = 0; s < tr.accepted.size(); ++s)
    for (int l = 0; l < L; ++l)
      if (!seen[s * static_cast<std::size_t>(L) + static_cast<std::size_t>(l)])
        fail(path, line_no, "missing layer " + std::to_string(l) + " in step " + std::to_string(s));
  return tr;
}

}  // namespace moespac
