// result_io.cpp -- JSON summary and solution files of a SolveResult
// (reference /root/reference/proj/src/result_io.cpp:53-98,
// which serializes through nlohmann::ordered_json dump(2)).  Written directly:
// the same keys in the same order, two-space indentation, integers as
// integers, doubles as the reference writer's Grisu2 digits (grisu.hpp,
// round-trip but not always shortest) laid out like it (fixed notation for exponents in [-4, 15), otherwise
// d.ddde+XX with at least two exponent digits, ".0" on integral values,
// non-finite values as null).
#include "folp/result_io.hpp"

#include "grisu.hpp"

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>

namespace folp {

namespace {

void json_double(std::string& out, double v) {
  if (!std::isfinite(v)) {
    out += "null";
    return;
  }
  if (std::signbit(v)) {
    out += '-';
    v = -v;
  }
  if (v == 0.0) {
    out += "0.0";
    return;
  }
  char digits[32];
  int K = 0;
  const int k = grisu::digits(v, digits, K);  // the reference writer's digits (grisu.hpp)
  const int exp10 = K + k - 1;
  const int n = exp10 + 1;  // decimal point position relative to the digits
  constexpr int kMinExp = -4, kMaxExp = 15;
  if (k <= n && n <= kMaxExp) {
    out.append(digits, static_cast<std::size_t>(k));
    out.append(static_cast<std::size_t>(n - k), '0');
    out += ".0";
  } else if (0 < n && n <= kMaxExp) {
    out.append(digits, static_cast<std::size_t>(n));
    out += '.';
    out.append(digits + n, static_cast<std::size_t>(k - n));
  } else if (kMinExp < n && n <= 0) {
    out += "0.";
    out.append(static_cast<std::size_t>(-n), '0');
    out.append(digits, static_cast<std::size_t>(k));
  } else {
    out += digits[0];
    if (k > 1) {
      out += '.';
      out.append(digits + 1, static_cast<std::size_t>(k - 1));
    }
    char ex[16];
    const int x = n - 1;
    std::snprintf(ex, sizeof(ex), "e%c%02d", x < 0 ? '-' : '+', x < 0 ? -x : x);
    out += ex;
  }
}

struct Writer {
  std::string out;
  int depth = 0;
  bool first = true;
  void indent() { out.append(static_cast<std::size_t>(2 * depth), ' '); }
  void key(const char* k) {
    if (!first) out += ",\n";
    first = false;
    indent();
    out += '"';
    out += k;
    out += "\": ";
  }
  void open(char c) {
    out += c;
    ++depth;
    first = true;
  }
  void close(char c, bool empty) {
    --depth;
    if (!empty) {
      out += '\n';
      indent();
    }
    out += c;
    first = false;
  }
  void begin_member_object() {  // after key(): "{\n"
    open('{');
    out += '\n';
  }
  void field(const char* k, double v) {
    key(k);
    json_double(out, v);
  }
  void field_int(const char* k, long long v) {
    key(k);
    out += std::to_string(v);
  }
  void field_str(const char* k, const std::string& v) {
    key(k);
    out += '"';
    out += v;
    out += '"';
  }
};

void info_fields(Writer& w, const ConvergenceInfo& info) {
  w.field("primal_objective", info.primal_objective);
  w.field("dual_objective", info.dual_objective);
  w.field("gap_abs", info.gap_abs);
  w.field("primal_residual_norm", info.primal_residual_norm);
  w.field("dual_residual_norm", info.dual_residual_norm);
  w.field("norm_q", info.norm_q);
  w.field("norm_c", info.norm_c);
}

void write_vector(const std::string& path, const std::vector<double>& v) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw IoError("cannot open '" + path + "' for writing");
  std::string buf;
  buf.reserve(v.size() * 24);
  char one[40];
  for (double x : v) {
    const int len = std::snprintf(one, sizeof(one), "%.17g\n", x);
    buf.append(one, static_cast<std::size_t>(len));
  }
  out << buf;
  if (!out) throw IoError("failed writing '" + path + "'");
}

}  // namespace

std::string result_to_json(const SolveResult& r) {
  Writer w;
  w.begin_member_object();
  w.field_str("solver", "folp");
  w.field_str("version", "0.1.0");
  w.field_str("termination_reason", to_string(r.termination_reason));
  w.field_int("iterations", r.iterations);
  w.field("kkt_passes", r.kkt_passes);
  w.field("wall_seconds", r.wall_seconds);
  w.field_int("restarts", r.restarts);
  w.field_int("step_trials", r.step_trials);
  w.field("primal_objective", r.final_info.primal_objective);
  w.field("dual_objective", r.final_info.dual_objective);
  w.field("gap_abs", r.final_info.gap_abs);
  w.field("primal_residual_norm", r.final_info.primal_residual_norm);
  w.field("dual_residual_norm", r.final_info.dual_residual_norm);
  w.key("trace");
  w.open('[');
  for (const TraceEntry& t : r.trace) {
    if (!w.first) w.out += ',';
    w.out += '\n';
    w.first = false;
    w.indent();
    w.begin_member_object();
    w.field_int("iteration", t.iteration);
    w.field("kkt_passes", t.kkt_passes);
    w.key("current");
    w.begin_member_object();
    info_fields(w, t.current);
    w.close('}', false);
    w.key("average");
    w.begin_member_object();
    info_fields(w, t.average);
    w.close('}', false);
    w.close('}', false);
  }
  w.close(']', r.trace.empty());
  w.close('}', false);
  w.out += '\n';
  return w.out;
}

void write_result(const SolveResult& result, const std::string& output_dir) {
  std::error_code ec;
  std::filesystem::create_directories(output_dir, ec);
  if (ec) throw IoError("cannot create '" + output_dir + "': " + ec.message());
  const std::filesystem::path dir(output_dir);
  {
    const std::string path = (dir / "summary.json").string();
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot open '" + path + "' for writing");
    out << result_to_json(result);
    if (!out) throw IoError("failed writing '" + path + "'");
  }
  write_vector((dir / "primal_solution.txt").string(), result.primal_solution);
  write_vector((dir / "dual_solution.txt").string(), result.dual_solution);
  write_vector((dir / "reduced_costs.txt").string(), result.reduced_costs);
}

}  // namespace folp
