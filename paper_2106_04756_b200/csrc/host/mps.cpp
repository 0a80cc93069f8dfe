// mps.cpp -- multi-threaded MPS reader and writer.
//
// Semantics follow /root/reference/proj/src/mps.cpp (parse_mps :403-491,
// section handlers :115-325, assemble :327-401, write_mps :511-566): the
// same sections, row / bound types, quirks, error messages and line numbers,
// and the same LinearProgram bit for bit.  The work is split differently:
//
//   1. one parallel scan over the bytes finds the header lines (a line that
//      starts with neither whitespace nor '*') and counts newlines, so every
//      header knows its line number;
//   2. headers are walked in file order; the bulk sections (COLUMNS, RHS,
//      RANGES, BOUNDS) are cut into line-aligned pieces that are tokenized
//      and parsed in parallel into records against the tables the earlier
//      sections built (read-only during the section), then applied in file
//      order -- the first error in file order wins, as in the sequential
//      reader;
//   3. COLUMNS records carry runs of equal column names, so the column table
//      sees one lookup per run instead of one per entry;
//   4. the triplets of a file whose rows come out with increasing columns
//      (the usual column-major MPS) are compressed by a counting pass; other
//      files go through SparseMatrix::from_triplets exactly as the reference.
#include "folp/mps.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <thread>
#include <unordered_map>

#include "parallel.hpp"
#include "sparse_access.hpp"

namespace folp {

namespace {

inline bool is_space(unsigned char c) { return c == ' ' || (c >= '\t' && c <= '\r'); }

// Parallel pieces for `bytes` of text; FOLP_IO_PIECES forces a count (tests
// use it to split small files).
int io_pieces(std::size_t bytes) {
  if (const char* env = std::getenv("FOLP_IO_PIECES")) return std::max(1, std::atoi(env));
  return std::max(1, std::min<int>(host::host_threads(static_cast<int64_t>(bytes) / 8),
                                   static_cast<int>(bytes / 4096 + 1)));
}

void tokenize(std::string_view line, std::vector<std::string_view>& out) {
  out.clear();
  std::size_t i = 0;
  const std::size_t n = line.size();
  while (i < n) {
    while (i < n && is_space(static_cast<unsigned char>(line[i]))) ++i;
    const std::size_t s = i;
    while (i < n && !is_space(static_cast<unsigned char>(line[i]))) ++i;
    if (i > s) out.push_back(line.substr(s, i - s));
  }
}

std::string upper(std::string_view s) {
  std::string u(s);
  for (char& c : u) {
    if (c >= 'a' && c <= 'z') c = static_cast<char>(c - 'a' + 'A');
  }
  return u;
}

bool upper_equals(std::string_view s, std::string_view lit) {
  if (s.size() != lit.size()) return false;
  for (std::size_t i = 0; i < s.size(); ++i) {
    char c = s[i];
    if (c >= 'a' && c <= 'z') c = static_cast<char>(c - 'a' + 'A');
    if (c != lit[i]) return false;
  }
  return true;
}

// strtod on a NUL-terminated copy; the whole token must be consumed up to
// its first NUL (mps.cpp:73-80).
bool to_number(std::string_view tok, double* v) {
  char small[64];
  std::string big;
  const char* s;
  if (tok.size() < sizeof(small)) {
    std::memcpy(small, tok.data(), tok.size());
    small[tok.size()] = '\0';
    s = small;
  } else {
    big.assign(tok);
    s = big.c_str();
  }
  char* end = nullptr;
  *v = std::strtod(s, &end);
  return !(end == s || *end != '\0');
}

std::string number_error(std::string_view tok) {
  return "cannot parse number '" + std::string(tok) + "'";
}

enum class RowType : int8_t { kObjective, kFree, kLess, kGreater, kEqual };

struct RowInfo {
  RowType type;
  Index index;  // among constraint rows; -1 for objective / free rows
};

enum class Section { kNone, kName, kObjsense, kRows, kColumns, kRhs, kRanges, kBounds, kEnd };

// A failure inside a parallel piece: the first one in the piece.
struct PieceError {
  Index line = -1;
  std::string message;
};

struct ColumnsPiece {
  struct Run {
    std::string_view name;
    int64_t first;  // first item of the run
  };
  struct Item {
    Index row;  // constraint row, or -1 for the objective row
    double value;
  };
  std::vector<Run> runs;
  std::vector<Item> items;
  int64_t constraint_items = 0;
  PieceError err;
};

struct ValuePiece {  // RHS / RANGES / BOUNDS records
  struct Rec {
    int32_t kind;  // RHS: 0 row, 1 objective; BOUNDS: the bound type
    Index index;
    double value;
  };
  std::vector<Rec> recs;
  PieceError err;
};

enum BoundKind : int32_t { kLo, kUp, kFx, kFr, kMi, kPl, kBv };

struct Parser {
  std::string_view text;
  std::unordered_map<std::string_view, RowInfo> rows;
  std::vector<RowType> row_types;  // per constraint row
  std::vector<double> row_rhs;
  std::vector<char> row_has_range;
  std::vector<double> row_range;

  std::unordered_map<std::string_view, Index> columns;
  Index num_columns = 0;
  std::vector<double> objective, lower, upper_b;
  std::vector<char> lower_touched;
  std::vector<Triplet> entries;

  bool has_objective_row = false;
  double objective_rhs = 0.0;
  bool maximize = false;
  std::string problem_name = "UNNAMED";

  Index column_of(std::string_view name) {
    auto it = columns.find(name);
    if (it != columns.end()) return it->second;
    const Index idx = num_columns++;
    columns.emplace(name, idx);
    objective.push_back(0.0);
    lower.push_back(0.0);
    upper_b.push_back(kInf);
    lower_touched.push_back(0);
    return idx;
  }
};

// Line-aligned pieces of [b, e) with the line number of each piece's first
// line (newlines counted in parallel).
struct Pieces {
  std::vector<std::size_t> cut;  // [k + 1]
  std::vector<Index> line0;      // [k]
};

Pieces split_lines(std::string_view text, std::size_t b, std::size_t e, Index first_line) {
  Pieces p;
  const std::size_t bytes = e - b;
  const int k = io_pieces(bytes);
  p.cut.push_back(b);
  for (int i = 1; i < k; ++i) {
    std::size_t c = b + bytes * static_cast<std::size_t>(i) / static_cast<std::size_t>(k);
    c = std::max(c, p.cut.back());
    const std::size_t nl = text.find('\n', c);
    c = (nl == std::string_view::npos || nl >= e) ? e : nl + 1;
    p.cut.push_back(c);
  }
  p.cut.push_back(e);
  const int pieces = static_cast<int>(p.cut.size()) - 1;
  std::vector<Index> nl(static_cast<std::size_t>(pieces), 0);
  std::vector<std::thread> pool;
  for (int i = 0; i < pieces; ++i) {
    pool.emplace_back([&, i] {
      nl[i] = static_cast<Index>(std::count(text.data() + p.cut[i], text.data() + p.cut[i + 1], '\n'));
    });
  }
  for (auto& t : pool) t.join();
  p.line0.resize(static_cast<std::size_t>(pieces));
  Index line = first_line;
  for (int i = 0; i < pieces; ++i) {
    p.line0[i] = line;
    line += nl[i];
  }
  return p;
}

// f(line, line_number) for every line of [b, e) (lines end at '\n'; the
// piece ends on a line boundary).
template <class F>
void for_lines(std::string_view text, std::size_t b, std::size_t e, Index line0, F&& f) {
  std::size_t pos = b;
  Index line = line0;
  while (pos < e) {
    std::size_t eol = text.find('\n', pos);
    if (eol == std::string_view::npos || eol > e) eol = e;
    if (!f(text.substr(pos, eol - pos), line)) return;
    pos = eol + 1;
    ++line;
  }
}

template <class Piece, class Fn>
std::vector<Piece> run_pieces(const Pieces& p, Fn&& parse_piece) {
  const int k = static_cast<int>(p.line0.size());
  std::vector<Piece> out(static_cast<std::size_t>(k));
  std::vector<std::thread> pool;
  for (int i = 1; i < k; ++i) pool.emplace_back([&, i] { parse_piece(i, out[i]); });
  parse_piece(0, out[0]);
  for (auto& t : pool) t.join();
  for (const Piece& piece : out) {
    if (piece.err.line >= 0) throw MpsParseError(piece.err.message, piece.err.line);
  }
  return out;
}

// ---- sections ----------------------------------------------------------

void rows_line(Parser& p, const std::vector<std::string_view>& tok, Index line) {
  if (tok.size() != 2) throw MpsParseError("ROWS line needs a type and a name", line);
  const std::string_view name = tok[1];
  if (p.rows.count(name) != 0) throw MpsParseError("duplicate row '" + std::string(name) + "'", line);
  if (upper_equals(tok[0], "N")) {
    p.rows.emplace(name, RowInfo{p.has_objective_row ? RowType::kFree : RowType::kObjective, -1});
    p.has_objective_row = true;
    return;
  }
  RowType rt;
  if (upper_equals(tok[0], "L")) rt = RowType::kLess;
  else if (upper_equals(tok[0], "G")) rt = RowType::kGreater;
  else if (upper_equals(tok[0], "E")) rt = RowType::kEqual;
  else throw MpsParseError("unknown row type '" + std::string(tok[0]) + "'", line);
  p.rows.emplace(name, RowInfo{rt, static_cast<Index>(p.row_types.size())});
  p.row_types.push_back(rt);
  p.row_rhs.push_back(0.0);
  p.row_has_range.push_back(0);
  p.row_range.push_back(0.0);
}

void columns_section(Parser& p, std::size_t b, std::size_t e, Index line0) {
  const Pieces pc = split_lines(p.text, b, e, line0);
  auto pieces = run_pieces<ColumnsPiece>(pc, [&](int i, ColumnsPiece& out) {
    std::vector<std::string_view> tok;
    for_lines(p.text, pc.cut[i], pc.cut[i + 1], pc.line0[i], [&](std::string_view ln, Index line) {
      if (ln.empty() || ln[0] == '*') return true;
      tokenize(ln, tok);
      if (tok.empty()) return true;
      for (std::string_view t : tok) {
        if (upper_equals(t, "'MARKER'")) return true;  // integrality dropped: LP relaxation
      }
      if (tok.size() < 3 || tok.size() % 2 == 0) {
        out.err = {line, "COLUMNS line needs name and row/value pairs"};
        return false;
      }
      if (out.runs.empty() || out.runs.back().name != tok[0]) {
        out.runs.push_back({tok[0], static_cast<int64_t>(out.items.size())});
      }
      for (std::size_t k = 1; k + 1 < tok.size(); k += 2) {
        const auto it = p.rows.find(tok[k]);
        if (it == p.rows.end()) {
          out.err = {line, "reference to undeclared row '" + std::string(tok[k]) + "'"};
          return false;
        }
        double v;
        if (!to_number(tok[k + 1], &v)) {
          out.err = {line, number_error(tok[k + 1])};
          return false;
        }
        if (it->second.type == RowType::kObjective) {
          out.items.push_back({-1, v});
        } else if (it->second.type != RowType::kFree) {
          out.items.push_back({it->second.index, v});
          ++out.constraint_items;
        }
      }
      return true;
    });
  });
  // column ids in order of first appearance, one lookup per run
  std::vector<std::vector<Index>> run_col(pieces.size());
  std::vector<int64_t> offset(pieces.size() + 1, static_cast<int64_t>(p.entries.size()));
  for (std::size_t i = 0; i < pieces.size(); ++i) {
    run_col[i].reserve(pieces[i].runs.size());
    for (const auto& r : pieces[i].runs) run_col[i].push_back(p.column_of(r.name));
    offset[i + 1] = offset[i] + pieces[i].constraint_items;
  }
  // objective entries accumulate in file order (mps.cpp:171-173)
  for (std::size_t i = 0; i < pieces.size(); ++i) {
    const auto& pc_i = pieces[i];
    for (std::size_t r = 0; r < pc_i.runs.size(); ++r) {
      const int64_t e_ = r + 1 < pc_i.runs.size() ? pc_i.runs[r + 1].first
                                                  : static_cast<int64_t>(pc_i.items.size());
      for (int64_t k = pc_i.runs[r].first; k < e_; ++k) {
        if (pc_i.items[k].row < 0) p.objective[run_col[i][r]] += pc_i.items[k].value;
      }
    }
  }
  p.entries.resize(static_cast<std::size_t>(offset.back()));
  std::vector<std::thread> pool;
  for (std::size_t i = 0; i < pieces.size(); ++i) {
    pool.emplace_back([&, i] {
      const auto& pc_i = pieces[i];
      int64_t w = offset[i];
      for (std::size_t r = 0; r < pc_i.runs.size(); ++r) {
        const int64_t e_ = r + 1 < pc_i.runs.size() ? pc_i.runs[r + 1].first
                                                    : static_cast<int64_t>(pc_i.items.size());
        const Index col = run_col[i][r];
        for (int64_t k = pc_i.runs[r].first; k < e_; ++k) {
          if (pc_i.items[k].row >= 0) p.entries[w++] = {pc_i.items[k].row, col, pc_i.items[k].value};
        }
      }
    });
  }
  for (auto& t : pool) t.join();
}

// RHS and RANGES: [set name] (row value)+ (mps.cpp:182-230).
void pairs_section(Parser& p, std::size_t b, std::size_t e, Index line0, bool ranges) {
  const Pieces pc = split_lines(p.text, b, e, line0);
  auto pieces = run_pieces<ValuePiece>(pc, [&](int i, ValuePiece& out) {
    std::vector<std::string_view> tok;
    for_lines(p.text, pc.cut[i], pc.cut[i + 1], pc.line0[i], [&](std::string_view ln, Index line) {
      if (ln.empty() || ln[0] == '*') return true;
      tokenize(ln, tok);
      if (tok.empty()) return true;
      const std::size_t first = tok.size() % 2 == 1 ? 1 : 0;
      if (tok.size() < 2) {
        out.err = {line, ranges ? "RANGES line needs row/value pairs" : "RHS line needs row/value pairs"};
        return false;
      }
      for (std::size_t k = first; k + 1 < tok.size(); k += 2) {
        const auto it = p.rows.find(tok[k]);
        if (ranges) {
          if (it == p.rows.end() || it->second.index < 0) {
            out.err = {line, "RANGES references non-constraint row '" + std::string(tok[k]) + "'"};
            return false;
          }
        } else if (it == p.rows.end()) {
          out.err = {line, "reference to undeclared row '" + std::string(tok[k]) + "'"};
          return false;
        }
        double v;
        if (!to_number(tok[k + 1], &v)) {
          out.err = {line, number_error(tok[k + 1])};
          return false;
        }
        if (it->second.type == RowType::kObjective && !ranges) {
          out.recs.push_back({1, -1, v});
        } else if (it->second.type != RowType::kFree || ranges) {
          out.recs.push_back({0, it->second.index, v});
        }
      }
      return true;
    });
  });
  for (const auto& piece : pieces) {
    for (const auto& r : piece.recs) {
      if (ranges) {
        p.row_has_range[r.index] = 1;
        p.row_range[r.index] = r.value;
      } else if (r.kind == 1) {
        p.objective_rhs = r.value;  // minus the objective constant
      } else {
        p.row_rhs[r.index] = r.value;
      }
    }
  }
}

// BOUNDS: type [set name] column [value] (mps.cpp:232-289).
void bounds_section(Parser& p, std::size_t b, std::size_t e, Index line0) {
  const Pieces pc = split_lines(p.text, b, e, line0);
  auto pieces = run_pieces<ValuePiece>(pc, [&](int i, ValuePiece& out) {
    std::vector<std::string_view> tok;
    for_lines(p.text, pc.cut[i], pc.cut[i + 1], pc.line0[i], [&](std::string_view ln, Index line) {
      if (ln.empty() || ln[0] == '*') return true;
      tokenize(ln, tok);
      if (tok.empty()) return true;
      if (tok.size() < 2) {
        out.err = {line, "BOUNDS line needs a type and a column"};
        return false;
      }
      const std::string type = upper(tok[0]);
      const bool needs_value = type == "LO" || type == "UP" || type == "FX";
      const std::size_t col_field = tok.size() >= (needs_value ? 4u : 3u) ? 2 : 1;
      const auto it = p.columns.find(tok[col_field]);
      if (it == p.columns.end()) {
        out.err = {line, "bound on undeclared column '" + std::string(tok[col_field]) + "'"};
        return false;
      }
      if (needs_value && tok.size() < col_field + 2) {
        out.err = {line, "bound type " + type + " needs a value"};
        return false;
      }
      double v = 0.0;
      if (needs_value && !to_number(tok[col_field + 1], &v)) {
        out.err = {line, number_error(tok[col_field + 1])};
        return false;
      }
      int32_t kind;
      if (type == "LO") kind = kLo;
      else if (type == "UP") kind = kUp;
      else if (type == "FX") kind = kFx;
      else if (type == "FR") kind = kFr;
      else if (type == "MI") kind = kMi;
      else if (type == "PL") kind = kPl;
      else if (type == "BV") kind = kBv;
      else {
        out.err = {line, "unknown bound type '" + std::string(tok[0]) + "'"};
        return false;
      }
      out.recs.push_back({kind, it->second, v});
      return true;
    });
  });
  for (const auto& piece : pieces) {
    for (const auto& r : piece.recs) {
      const std::size_t c = static_cast<std::size_t>(r.index);
      switch (r.kind) {
        case kLo:
          p.lower[c] = r.value;
          p.lower_touched[c] = 1;
          break;
        case kUp:
          p.upper_b[c] = r.value;
          // a negative upper bound on a column whose lower bound was never
          // set releases the lower bound (classic MPS, mps.cpp:263-265)
          if (r.value < 0.0 && !p.lower_touched[c]) p.lower[c] = -kInf;
          break;
        case kFx:
          p.lower[c] = r.value;
          p.upper_b[c] = r.value;
          p.lower_touched[c] = 1;
          break;
        case kFr:
          p.lower[c] = -kInf;
          p.upper_b[c] = kInf;
          p.lower_touched[c] = 1;
          break;
        case kMi:
          p.lower[c] = -kInf;
          p.lower_touched[c] = 1;
          break;
        case kPl:
          p.upper_b[c] = kInf;
          break;
        default:  // kBv
          p.lower[c] = 0.0;
          p.upper_b[c] = 1.0;
          p.lower_touched[c] = 1;
      }
    }
  }
}

// Triplets -> K.  Rows of increasing columns after a stable counting pass
// by row (the column-major MPS layout): compressed directly, which equals
// from_triplets for duplicate-free input (single entries are kept as
// 0.0 + v, exact zeros dropped).  Anything else: from_triplets itself.
SparseMatrix build_matrix(Index m, Index n, const std::vector<Triplet>& t) {
  for (const Triplet& e : t) {
    if (!std::isfinite(e.value)) return SparseMatrix::from_triplets(m, n, t);  // throws its error
  }
  std::vector<Index> start(static_cast<std::size_t>(m) + 1, 0);
  for (const Triplet& e : t) ++start[static_cast<std::size_t>(e.row) + 1];
  for (Index r = 0; r < m; ++r) start[r + 1] += start[r];
  std::vector<Index> fill(start.begin(), start.end() - 1);
  std::vector<Index> cols(t.size());
  std::vector<double> vals(t.size());
  for (const Triplet& e : t) {
    const Index k = fill[e.row]++;
    cols[k] = e.col;
    vals[k] = e.value;
  }
  bool sorted = true;
  for (Index r = 0; r < m && sorted; ++r) {
    for (Index k = start[r] + 1; k < start[r + 1]; ++k) {
      if (cols[k] <= cols[k - 1]) {
        sorted = false;
        break;
      }
    }
  }
  if (!sorted) return SparseMatrix::from_triplets(m, n, t);
  // drop exact zeros
  std::vector<Index> s2(static_cast<std::size_t>(m) + 1, 0);
  Index w = 0;
  for (Index r = 0; r < m; ++r) {
    for (Index k = start[r]; k < start[r + 1]; ++k) {
      const double v = 0.0 + vals[k];
      if (v == 0.0) continue;
      cols[w] = cols[k];
      vals[w] = v;
      ++w;
    }
    s2[r + 1] = w;
  }
  cols.resize(static_cast<std::size_t>(w));
  vals.resize(static_cast<std::size_t>(w));
  return SparseMatrixAccess::build(m, n, std::move(s2), std::move(cols), std::move(vals));
}

// Rows -> activity intervals -> ">= rows, then the negated upper sides of
// two-sided rows, then equality rows" (mps.cpp:327-401).
MpsInstance assemble(Parser& p) {
  const Index nc = static_cast<Index>(p.row_types.size());
  const Index n = p.num_columns;
  std::vector<double> lo(static_cast<std::size_t>(nc)), hi(static_cast<std::size_t>(nc));
  for (Index r = 0; r < nc; ++r) {
    const double rhs = p.row_rhs[r];
    const double range = p.row_range[r];
    const bool has = p.row_has_range[r] != 0;
    double a = -kInf, b = kInf;
    switch (p.row_types[r]) {
      case RowType::kGreater:
        a = rhs;
        if (has) b = rhs + std::fabs(range);
        break;
      case RowType::kLess:
        b = rhs;
        if (has) a = rhs - std::fabs(range);
        break;
      case RowType::kEqual:
        if (has && range != 0.0) {
          if (range > 0.0) {
            a = rhs;
            b = rhs + range;
          } else {
            a = rhs + range;
            b = rhs;
          }
        } else {
          a = b = rhs;
        }
        break;
      default:
        break;
    }
    lo[r] = a;
    hi[r] = b;
  }
  std::vector<Index> primary(static_cast<std::size_t>(nc), -1), secondary(static_cast<std::size_t>(nc), -1);
  std::vector<char> negate(static_cast<std::size_t>(nc), 0);
  std::vector<double> rhs_out;
  rhs_out.reserve(static_cast<std::size_t>(nc));
  Index next = 0;
  for (Index r = 0; r < nc; ++r) {
    if (lo[r] == hi[r]) continue;
    if (lo[r] > -kInf) {
      primary[r] = next++;
      rhs_out.push_back(lo[r]);
    } else if (hi[r] < kInf) {
      primary[r] = next++;
      negate[r] = 1;
      rhs_out.push_back(-hi[r]);
    }
  }
  for (Index r = 0; r < nc; ++r) {
    if (lo[r] == hi[r] || lo[r] == -kInf || hi[r] == kInf) continue;
    secondary[r] = next++;
    rhs_out.push_back(-hi[r]);
  }
  const Index m1 = next;
  for (Index r = 0; r < nc; ++r) {
    if (lo[r] == hi[r]) {
      primary[r] = next++;
      rhs_out.push_back(lo[r]);
    }
  }
  std::vector<Triplet> trip;
  trip.reserve(p.entries.size());
  for (const Triplet& e : p.entries) {
    const Index pr = primary[e.row], sr = secondary[e.row];
    if (pr >= 0) trip.push_back({pr, e.col, negate[e.row] ? -e.value : e.value});
    if (sr >= 0) trip.push_back({sr, e.col, -e.value});
  }
  MpsInstance out;
  out.name = p.problem_name;
  out.was_maximization = p.maximize;
  LinearProgram& lp = out.lp;
  lp.objective = std::move(p.objective);
  lp.objective_constant = -p.objective_rhs;
  lp.constraint_matrix = build_matrix(next, n, trip);
  lp.right_hand_side = std::move(rhs_out);
  lp.num_inequality_rows = m1;
  lp.variable_lower = std::move(p.lower);
  lp.variable_upper = std::move(p.upper_b);
  if (out.was_maximization) {
    for (double& v : lp.objective) v = -v;
    lp.objective_constant = -lp.objective_constant;
  }
  return out;
}

// Header lines (first byte neither whitespace nor '*') with their line
// numbers, found by a parallel scan.
struct Header {
  std::size_t begin, end;  // the line, without its '\n'
  Index line;
};

std::vector<Header> find_headers(std::string_view text) {
  const std::size_t size = text.size();
  const int k = io_pieces(size);
  std::vector<std::vector<std::pair<std::size_t, Index>>> found(static_cast<std::size_t>(k));
  std::vector<Index> newlines(static_cast<std::size_t>(k), 0);
  std::vector<std::thread> pool;
  for (int i = 0; i < k; ++i) {
    pool.emplace_back([&, i] {
      const std::size_t b = size * i / k, e = size * (i + 1) / k;
      Index nl = 0;
      for (std::size_t pos = b; pos < e; ++pos) {
        const bool line_start = pos == 0 || text[pos - 1] == '\n';
        const unsigned char c = static_cast<unsigned char>(text[pos]);
        if (line_start && !is_space(c) && c != '*') found[i].push_back({pos, nl});
        if (c == '\n') ++nl;
      }
      newlines[i] = nl;
    });
  }
  for (auto& t : pool) t.join();
  std::vector<Header> out;
  Index base = 1;
  for (int i = 0; i < k; ++i) {
    for (const auto& [pos, nl] : found[i]) {
      std::size_t eol = text.find('\n', pos);
      if (eol == std::string_view::npos) eol = size;
      out.push_back({pos, eol, base + nl});
    }
    base += newlines[i];
  }
  return out;
}

}  // namespace

MpsInstance parse_mps(std::string_view text) {
  Parser p;
  p.text = text;
  const std::vector<Header> headers = find_headers(text);
  const Index total_lines = 1 + static_cast<Index>(std::count(text.begin(), text.end(), '\n'));
  Section section = Section::kNone;
  bool objsense_pending = false;
  Index last_line = total_lines;  // the reference's line counter at the end

  // data lines of [b, e) (first line number line0) in `section`
  auto data_range = [&](std::size_t b, std::size_t e, Index line0) {
    if (b >= e) return;
    switch (section) {
      case Section::kRows: {
        std::vector<std::string_view> tok;
        for_lines(text, b, e, line0, [&](std::string_view ln, Index line) {
          if (ln.empty() || ln[0] == '*') return true;
          tokenize(ln, tok);
          if (!tok.empty()) rows_line(p, tok, line);
          return true;
        });
        break;
      }
      case Section::kColumns:
        columns_section(p, b, e, line0);
        break;
      case Section::kRhs:
        pairs_section(p, b, e, line0, false);
        break;
      case Section::kRanges:
        pairs_section(p, b, e, line0, true);
        break;
      case Section::kBounds:
        bounds_section(p, b, e, line0);
        break;
      default: {  // OBJSENSE value line, or data outside any section
        std::vector<std::string_view> tok;
        for_lines(text, b, e, line0, [&](std::string_view ln, Index line) {
          if (ln.empty() || ln[0] == '*') return true;
          tokenize(ln, tok);
          if (tok.empty()) return true;
          if (section != Section::kObjsense) {
            throw MpsParseError("data line outside any section", line);
          }
          if (objsense_pending) {
            p.maximize = upper_equals(tok[0], "MAX") || upper_equals(tok[0], "MAXIMIZE");
            objsense_pending = false;
          }
          return true;
        });
      }
    }
  };

  std::size_t pos = 0;
  Index line0 = 1;
  bool ended = false;
  std::vector<std::string_view> tok;
  for (const Header& h : headers) {
    data_range(pos, h.begin, line0);
    tokenize(text.substr(h.begin, h.end - h.begin), tok);
    const std::string kw = upper(tok[0]);
    objsense_pending = false;
    if (kw == "NAME") {
      section = Section::kName;
      if (tok.size() > 1) p.problem_name = std::string(tok[1]);
    } else if (kw == "OBJSENSE") {
      section = Section::kObjsense;
      if (tok.size() > 1) {
        p.maximize = upper_equals(tok[1], "MAX") || upper_equals(tok[1], "MAXIMIZE");
      } else {
        objsense_pending = true;
      }
    } else if (kw == "ROWS") {
      section = Section::kRows;
    } else if (kw == "COLUMNS") {
      section = Section::kColumns;
    } else if (kw == "RHS") {
      section = Section::kRhs;
    } else if (kw == "RANGES") {
      section = Section::kRanges;
    } else if (kw == "BOUNDS") {
      section = Section::kBounds;
    } else if (kw == "ENDATA") {
      section = Section::kEnd;
      last_line = h.line;
      ended = true;
      break;
    } else {
      throw MpsParseError("unknown section '" + std::string(tok[0]) + "'", h.line);
    }
    pos = h.end < text.size() ? h.end + 1 : text.size();
    line0 = h.line + 1;
  }
  if (!ended) data_range(pos, text.size(), line0);
  if (!p.has_objective_row) throw MpsParseError("no objective (N) row declared", last_line);
  return assemble(p);
}

MpsInstance parse_mps_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open '" + path + "'");
  std::ostringstream buffer;
  buffer << in.rdbuf();
  return parse_mps(buffer.str());
}

namespace {

void append_value(std::string& out, double v) {
  char buf[40];
  const int len = std::snprintf(buf, sizeof(buf), "%.17g", v);
  out.append(buf, static_cast<std::size_t>(len));
}

void append_index(std::string& out, const char* prefix, Index i) {
  char buf[32];
  const int len = std::snprintf(buf, sizeof(buf), "%s%lld", prefix, static_cast<long long>(i));
  out.append(buf, static_cast<std::size_t>(len));
}

// f(begin, end, out) per piece of [0, count), concatenated in order.
template <class F>
void append_parallel(std::string& out, int64_t count, F&& f) {
  const int k = std::max(1, host::host_threads(count * 4));
  std::vector<std::string> part(static_cast<std::size_t>(k));
  std::vector<std::thread> pool;
  for (int i = 0; i < k; ++i) {
    pool.emplace_back([&, i] { f(count * i / k, count * (i + 1) / k, part[i]); });
  }
  for (auto& t : pool) t.join();
  for (const auto& s : part) out += s;
}

}  // namespace

// write_mps (mps.cpp:511-566): the same bytes, columns / rows / bounds
// formatted in parallel pieces.
std::string write_mps(const LinearProgram& lp, const std::string& name) {
  const Index m = lp.num_rows();
  const Index n = lp.num_variables();
  std::string out = "NAME " + (name.empty() ? std::string("FOLP") : name) + "\nROWS\n N OBJ\n";
  append_parallel(out, m, [&](int64_t b, int64_t e, std::string& s) {
    for (Index r = b; r < e; ++r) {
      append_index(s, r < lp.num_inequality_rows ? " G R" : " E R", r);
      s += '\n';
    }
  });
  out += "COLUMNS\n";
  const auto start = lp.constraint_matrix.col_start();
  const auto rows = lp.constraint_matrix.col_rows();
  const auto values = lp.constraint_matrix.col_values();
  append_parallel(out, n, [&](int64_t b, int64_t e, std::string& s) {
    for (Index c = b; c < e; ++c) {
      append_index(s, "    X", c);
      s += " OBJ ";
      append_value(s, lp.objective[static_cast<std::size_t>(c)]);
      s += '\n';
      for (Index k = start[c]; k < start[c + 1]; ++k) {
        append_index(s, "    X", c);
        append_index(s, " R", rows[k]);
        s += ' ';
        append_value(s, values[k]);
        s += '\n';
      }
    }
  });
  out += "RHS\n";
  if (lp.objective_constant != 0.0) {
    out += "    RHS OBJ ";
    append_value(out, -lp.objective_constant);
    out += '\n';
  }
  append_parallel(out, m, [&](int64_t b, int64_t e, std::string& s) {
    for (Index r = b; r < e; ++r) {
      const double q = lp.right_hand_side[static_cast<std::size_t>(r)];
      if (q == 0.0) continue;
      append_index(s, "    RHS R", r);
      s += ' ';
      append_value(s, q);
      s += '\n';
    }
  });
  out += "BOUNDS\n";
  append_parallel(out, n, [&](int64_t b, int64_t e, std::string& s) {
    for (Index c = b; c < e; ++c) {
      const double lo = lp.variable_lower[static_cast<std::size_t>(c)];
      const double hi = lp.variable_upper[static_cast<std::size_t>(c)];
      if (lo == 0.0 && hi == kInf) continue;
      if (lo == hi) {
        append_index(s, " FX BND X", c);
        s += ' ';
        append_value(s, lo);
        s += '\n';
        continue;
      }
      if (lo == -kInf && hi == kInf) {
        append_index(s, " FR BND X", c);
        s += '\n';
        continue;
      }
      if (lo == -kInf) {
        append_index(s, " MI BND X", c);
        s += '\n';
      } else if (lo != 0.0) {
        append_index(s, " LO BND X", c);
        s += ' ';
        append_value(s, lo);
        s += '\n';
      }
      if (hi < kInf) {
        append_index(s, " UP BND X", c);
        s += ' ';
        append_value(s, hi);
        s += '\n';
      }
    }
  });
  out += "ENDATA\n";
  return out;
}

void write_mps_file(const LinearProgram& lp, const std::string& name, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw IoError("cannot open '" + path + "' for writing");
  out << write_mps(lp, name);
  if (!out) throw IoError("failed writing '" + path + "'");
}

}  // namespace folp
