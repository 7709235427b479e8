#include "metrics.hpp"

#include <charconv>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <map>
#include <sstream>
#include <stdexcept>

namespace moespac {

RunSummary summarize(const std::vector<StepReport>& reports) {
  if (reports.empty()) throw std::invalid_argument("summarize: no step reports");
  RunSummary s;
  std::int64_t wall_sum = 0, bubble_sum = 0, hits = 0, misses = 0, fn = 0, fp = 0, expert_steps = 0;
  double accuracy_sum = 0.0;
  for (const StepReport& r : reports) {
    s.total_tokens += r.accepted_tokens;
    s.total_time_ns += r.step_wall_ns;
    hits += r.cache_hits;
    misses += r.cache_misses;
    fn += r.faults_fn;
    fp += r.faults_fp;
    expert_steps += static_cast<std::int64_t>(r.layers.size()) * r.n_experts;
    for (const LayerTiming& lt : r.layers) {
      wall_sum += lt.wall_ns;
      bubble_sum += lt.bubble_ns;
    }
    s.accuracy_series.push_back(r.accuracy);
    accuracy_sum += r.accuracy;
  }
  if (s.total_time_ns <= 0) throw std::invalid_argument("summarize: run has no simulated time");
  const double seconds = static_cast<double>(s.total_time_ns) * 1e-9;
  s.tps = static_cast<double>(s.total_tokens) / seconds;
  s.latency_s = seconds;
  s.hit_rate = hits + misses > 0 ? static_cast<double>(hits) / static_cast<double>(hits + misses) : 0.0;
  s.bubble_ratio = wall_sum > 0 ? static_cast<double>(bubble_sum) / static_cast<double>(wall_sum) : 0.0;
  s.fn_rate = static_cast<double>(fn) / static_cast<double>(expert_steps);
  s.fp_rate = static_cast<double>(fp) / static_cast<double>(expert_steps);
  s.fault_rate = s.fn_rate + s.fp_rate;
  s.mean_accuracy = accuracy_sum / static_cast<double>(reports.size());
  return s;
}

namespace {

constexpr const char* kMagic = "#moesim-metrics v1";
constexpr const char* kCsvColumns =
    "axis,axis_value,tps,latency_s,hit_rate,bubble_ratio,fault_rate,fn_rate,fp_rate,mean_accuracy,total_tokens,"
    "total_time_ns";

// JSON number layout of the reference's JSON library: integral-looking values
// get ".0", decimal exponents in (-4, 15] print positionally, others as
// d.ddde[+-]XX; non-finite values print as null.
std::string json_number(double v) {
  if (!std::isfinite(v)) return "null";
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::scientific);
  std::string sci(buf, r.ptr);
  std::string sign;
  if (sci[0] == '-') {
    sign = "-";
    sci.erase(0, 1);
  }
  const auto epos = sci.find('e');
  std::string digits;
  for (char c : sci.substr(0, epos))
    if (c != '.') digits += c;
  const int k = static_cast<int>(digits.size());
  const int n = std::stoi(sci.substr(epos + 1)) + 1;  // decimal point position
  std::string out;
  if (k <= n && n <= 15) {
    out = digits + std::string(static_cast<std::size_t>(n - k), '0') + ".0";
  } else if (0 < n && n <= 15) {
    out = digits.substr(0, static_cast<std::size_t>(n)) + "." + digits.substr(static_cast<std::size_t>(n));
  } else if (-4 < n && n <= 0) {
    out = "0." + std::string(static_cast<std::size_t>(-n), '0') + digits;
  } else {
    out = digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    const int x = n - 1;
    char eb[16];
    std::snprintf(eb, sizeof(eb), "e%c%02d", x < 0 ? '-' : '+', x < 0 ? -x : x);
    out += eb;
  }
  return sign + out;
}

std::string json_string(const std::string& s) {
  std::string o = "\"";
  for (unsigned char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (c < 0x20) {
          char u[8];
          std::snprintf(u, sizeof(u), "\\u%04x", c);
          o += u;
        } else {
          o += static_cast<char>(c);
        }
    }
  }
  return o + "\"";
}

double parse_double(const std::string& s) {
  double v = 0.0;
  const auto [ptr, ec] = std::from_chars(s.data(), s.data() + s.size(), v);
  if (ec != std::errc{} || ptr != s.data() + s.size()) throw std::runtime_error("parse_metrics: bad number '" + s + "'");
  return v;
}

// Minimal JSON reader for one metrics row: an object of strings, numbers
// (kept as text so integers stay exact) and arrays of numbers.
struct JVal {
  enum Kind { num, str, arr, null } kind = null;
  std::string text;             // num: literal, str: decoded
  std::vector<std::string> items;  // arr: number literals
};

struct JParser {
  const std::string& s;
  std::size_t i = 0;
  [[noreturn]] void bad() { throw std::runtime_error("parse_metrics: malformed JSON row"); }
  void ws() {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\t' || s[i] == '\r' || s[i] == '\n')) ++i;
  }
  char peek() {
    ws();
    if (i >= s.size()) bad();
    return s[i];
  }
  void expect(char c) {
    if (peek() != c) bad();
    ++i;
  }
  std::string str() {
    expect('"');
    std::string o;
    while (i < s.size() && s[i] != '"') {
      if (s[i] == '\\') {
        if (++i >= s.size()) bad();
        const char e = s[i++];
        switch (e) {
          case '"': o += '"'; break;
          case '\\': o += '\\'; break;
          case '/': o += '/'; break;
          case 'b': o += '\b'; break;
          case 'f': o += '\f'; break;
          case 'n': o += '\n'; break;
          case 'r': o += '\r'; break;
          case 't': o += '\t'; break;
          case 'u': {
            if (i + 4 > s.size()) bad();
            const unsigned cp = static_cast<unsigned>(std::stoul(s.substr(i, 4), nullptr, 16));
            i += 4;
            if (cp < 0x80) {
              o += static_cast<char>(cp);
            } else if (cp < 0x800) {
              o += static_cast<char>(0xC0 | (cp >> 6));
              o += static_cast<char>(0x80 | (cp & 0x3F));
            } else {
              o += static_cast<char>(0xE0 | (cp >> 12));
              o += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
              o += static_cast<char>(0x80 | (cp & 0x3F));
            }
            break;
          }
          default: bad();
        }
      } else {
        o += s[i++];
      }
    }
    expect('"');
    return o;
  }
  std::string number() {
    ws();
    const std::size_t b = i;
    while (i < s.size() && (std::isdigit(static_cast<unsigned char>(s[i])) || s[i] == '-' || s[i] == '+' ||
                            s[i] == '.' || s[i] == 'e' || s[i] == 'E'))
      ++i;
    if (i == b) bad();
    return s.substr(b, i - b);
  }
  JVal value() {
    JVal v;
    const char c = peek();
    if (c == '"') {
      v.kind = JVal::str;
      v.text = str();
    } else if (c == '[') {
      v.kind = JVal::arr;
      ++i;
      if (peek() == ']') {
        ++i;
        return v;
      }
      for (;;) {
        if (peek() == 'n' && s.compare(i, 4, "null") == 0) {
          i += 4;
          v.items.push_back("nan");
        } else {
          v.items.push_back(number());
        }
        if (peek() == ',') {
          ++i;
          continue;
        }
        expect(']');
        break;
      }
    } else if (c == 'n' && s.compare(i, 4, "null") == 0) {
      i += 4;
      v.kind = JVal::null;
    } else {
      v.kind = JVal::num;
      v.text = number();
    }
    return v;
  }
  std::map<std::string, JVal> object() {
    std::map<std::string, JVal> m;
    expect('{');
    if (peek() == '}') {
      ++i;
      return m;
    }
    for (;;) {
      const std::string k = str();
      expect(':');
      m[k] = value();
      if (peek() == ',') {
        ++i;
        continue;
      }
      expect('}');
      break;
    }
    return m;
  }
};

double jnum(const std::map<std::string, JVal>& m, const char* key) {
  const auto it = m.find(key);
  if (it == m.end()) throw std::runtime_error(std::string("parse_metrics: missing key ") + key);
  if (it->second.kind == JVal::null) return std::nan("");
  if (it->second.kind != JVal::num) throw std::runtime_error(std::string("parse_metrics: bad value for ") + key);
  return std::strtod(it->second.text.c_str(), nullptr);
}

std::int64_t jint(const std::map<std::string, JVal>& m, const char* key) {
  const auto it = m.find(key);
  if (it == m.end() || it->second.kind != JVal::num)
    throw std::runtime_error(std::string("parse_metrics: bad value for ") + key);
  const std::string& t = it->second.text;
  if (t.find_first_of(".eE") != std::string::npos) return static_cast<std::int64_t>(std::strtod(t.c_str(), nullptr));
  return std::stoll(t);
}

}  // namespace

std::string shortest(double v) {
  char buf[64];
  const auto [ptr, ec] = std::to_chars(buf, buf + sizeof(buf), v);
  if (ec != std::errc{}) throw std::runtime_error("fmt: to_chars failed");
  return {buf, ptr};
}

void emit(const std::vector<RunSummary>& summaries, MetricsFormat format, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("emit: cannot open " + path);
  if (format == MetricsFormat::csv) {
    out << kMagic << " csv\n" << kCsvColumns << '\n';
    for (const RunSummary& s : summaries)
      out << s.axis_name << ',' << shortest(s.axis_value) << ',' << shortest(s.tps) << ',' << shortest(s.latency_s)
          << ',' << shortest(s.hit_rate) << ',' << shortest(s.bubble_ratio) << ',' << shortest(s.fault_rate) << ','
          << shortest(s.fn_rate) << ',' << shortest(s.fp_rate) << ',' << shortest(s.mean_accuracy) << ','
          << s.total_tokens << ',' << s.total_time_ns << '\n';
  } else {
    out << kMagic << " jsonl\n";
    for (const RunSummary& s : summaries) {
      // keys in lexicographic order, as the reference's JSON object prints them
      std::string series = "[";
      for (std::size_t i = 0; i < s.accuracy_series.size(); ++i) {
        if (i) series += ',';
        series += json_number(s.accuracy_series[i]);
      }
      series += ']';
      out << "{\"accuracy_series\":" << series << ",\"axis\":" << json_string(s.axis_name)
          << ",\"axis_value\":" << json_number(s.axis_value) << ",\"bubble_ratio\":" << json_number(s.bubble_ratio)
          << ",\"fault_rate\":" << json_number(s.fault_rate) << ",\"fn_rate\":" << json_number(s.fn_rate)
          << ",\"fp_rate\":" << json_number(s.fp_rate) << ",\"hit_rate\":" << json_number(s.hit_rate)
          << ",\"latency_s\":" << json_number(s.latency_s) << ",\"mean_accuracy\":" << json_number(s.mean_accuracy)
          << ",\"total_time_ns\":" << s.total_time_ns << ",\"total_tokens\":" << s.total_tokens
          << ",\"tps\":" << json_number(s.tps) << "}\n";
    }
  }
  if (!out) throw std::runtime_error("emit: write failed on " + path);
}

std::vector<RunSummary> parse_metrics(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("parse_metrics: cannot open " + path);
  std::string line;
  if (!std::getline(in, line) || line.rfind(kMagic, 0) != 0)
    throw std::runtime_error("parse_metrics: missing schema header");
  const bool csv = line.find(" csv") != std::string::npos;
  std::vector<RunSummary> out;
  if (csv) {
    if (!std::getline(in, line) || line != kCsvColumns) throw std::runtime_error("parse_metrics: unexpected CSV columns");
    while (std::getline(in, line)) {
      if (line.empty()) continue;
      std::vector<std::string> cells;
      std::istringstream ls(line);
      std::string cell;
      while (std::getline(ls, cell, ',')) cells.push_back(cell);
      if (cells.size() != 12) throw std::runtime_error("parse_metrics: bad CSV row: " + line);
      RunSummary s;
      s.axis_name = cells[0];
      s.axis_value = parse_double(cells[1]);
      s.tps = parse_double(cells[2]);
      s.latency_s = parse_double(cells[3]);
      s.hit_rate = parse_double(cells[4]);
      s.bubble_ratio = parse_double(cells[5]);
      s.fault_rate = parse_double(cells[6]);
      s.fn_rate = parse_double(cells[7]);
      s.fp_rate = parse_double(cells[8]);
      s.mean_accuracy = parse_double(cells[9]);
      s.total_tokens = std::stoll(cells[10]);
      s.total_time_ns = std::stoll(cells[11]);
      out.push_back(std::move(s));
    }
  } else {
    while (std::getline(in, line)) {
      if (line.empty()) continue;
      JParser p{line};
      const auto m = p.object();
      RunSummary s;
      const auto ax = m.find("axis");
      if (ax == m.end() || ax->second.kind != JVal::str) throw std::runtime_error("parse_metrics: bad value for axis");
      s.axis_name = ax->second.text;
      s.axis_value = jnum(m, "axis_value");
      s.tps = jnum(m, "tps");
      s.latency_s = jnum(m, "latency_s");
      s.hit_rate = jnum(m, "hit_rate");
      s.bubble_ratio = jnum(m, "bubble_ratio");
      s.fault_rate = jnum(m, "fault_rate");
      s.fn_rate = jnum(m, "fn_rate");
      s.fp_rate = jnum(m, "fp_rate");
      s.mean_accuracy = jnum(m, "mean_accuracy");
      const auto se = m.find("accuracy_series");
      if (se == m.end() || se->second.kind != JVal::arr)
        throw std::runtime_error("parse_metrics: bad value for accuracy_series");
      for (const std::string& t : se->second.items) s.accuracy_series.push_back(std::strtod(t.c_str(), nullptr));
      s.total_tokens = jint(m, "total_tokens");
      s.total_time_ns = jint(m, "total_time_ns");
      out.push_back(std::move(s));
    }
  }
  return out;
}

}  // namespace moespac
