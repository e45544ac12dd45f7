// MPS reader and writer: the ingestion step in front of Solve (SURVEY §2 C6,
// §8f rank 3). Same normalisations, errors and messages as the reference
// (proj/core/src/mps_reader.cpp:33-475, mps_writer.cpp:37-116, mps.hpp:26-56):
//   E rows -> A/b; G rows -> G/h; L rows negated into G/h; a RANGES entry turns
//   its row into two G rows (lower side, then negated upper side); secondary N
//   rows dropped; MARKER integrality discarded; OBJSENSE MAX negates c and the
//   offset and sets negated_objective; the RHS of the objective row becomes
//   objective_offset = -value; fixed-format field columns 2-3, 5-12, 15-22,
//   25-36, 40-47, 50-61; .gz files through zlib.
//
// Built for throughput instead of by translation: the whole file is read into
// one buffer and split in place (string_views, no per-token allocation);
// names are looked up with heterogeneous (string_view) hashing; the column of
// the previous COLUMNS line is cached; numbers go through std::from_chars
// (correctly rounded, so identical to strtod on decimal input) with strtod
// as the fallback for the spellings only strtod accepts (leading '+', hex,
// out-of-range values); A and G are assembled straight into CSR by a stable
// counting sort on rows (FromTriplets semantics, sparse_matrix.cpp:25-69:
// sorted columns, duplicates summed -- here in file order -- zeros dropped).
#include <zlib.h>

#include <algorithm>
#include <chrono>
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/pdhg.h"
#include "host_logic.h"
#include "instance.h"

namespace {

using I = int64_t;
constexpr double kInf = std::numeric_limits<double>::infinity();

struct ParseError {
  int line;
  std::string msg;
};

struct IoError {
  std::string msg;
};

struct SvHash {
  using is_transparent = void;
  size_t operator()(std::string_view s) const { return std::hash<std::string_view>{}(s); }
};
// Keys are views into the text being parsed, which outlives the Reader (no
// per-name allocation).
using NameMap = std::unordered_map<std::string_view, I, SvHash, std::equal_to<>>;

enum class Section { kNone, kName, kObjsense, kRows, kColumns, kRhs, kRanges, kBounds, kEndata };

int Rank(Section s) {
  switch (s) {
    case Section::kRows: return 1;
    case Section::kColumns: return 2;
    case Section::kRhs:
    case Section::kRanges:
    case Section::kBounds: return 3;
    case Section::kEndata: return 4;
    default: return 0;
  }
}

bool IsSpace(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }

// Trim of " \t\r\n" (mps_reader.cpp Trim).
std::string_view Trim(std::string_view s) {
  auto t = [](char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n'; };
  size_t b = 0, e = s.size();
  while (b < e && t(s[b])) ++b;
  while (e > b && t(s[e - 1])) --e;
  return s.substr(b, e - b);
}

std::string Upper(std::string_view s) {
  std::string r(s);
  for (char& c : r) c = static_cast<char>(std::toupper(static_cast<unsigned char>(c)));
  return r;
}

// Whitespace tokens (operator>> semantics: isspace separators).
void SplitWs(std::string_view s, std::vector<std::string_view>& out) {
  out.clear();
  size_t i = 0;
  while (i < s.size()) {
    while (i < s.size() && IsSpace(s[i])) ++i;
    size_t j = i;
    while (j < s.size() && !IsSpace(s[j])) ++j;
    if (j > i) out.push_back(s.substr(i, j - i));
    i = j;
  }
}

// Fixed MPS fields, 1-based columns 2-3, 5-12, 15-22, 25-36, 40-47, 50-61.
void SplitFixed(std::string_view line, std::vector<std::string_view>& out) {
  static constexpr int kStarts[] = {1, 4, 14, 24, 39, 49};
  static constexpr int kEnds[] = {3, 12, 22, 36, 47, 61};
  out.clear();
  for (int f = 0; f < 6; ++f) {
    if (static_cast<size_t>(kStarts[f]) >= line.size()) break;
    const size_t e = std::min<size_t>(kEnds[f], line.size());
    std::string_view field = Trim(line.substr(kStarts[f], e - kStarts[f]));
    if (!field.empty()) out.push_back(field);
  }
}

struct Row {
  char type;
  double rhs = 0.0;
  bool has_range = false;
  double range = 0.0;
};

struct Entry {
  I row;
  I col;
  double v;
};

class Reader {
 public:
  explicit Reader(bool fixed) : fixed_(fixed) {
    row_index_.reserve(1 << 12);
    col_index_.reserve(1 << 12);
  }

  void Line(std::string_view raw) {
    ++line_;
    if (raw.empty() || raw[0] == '*') return;
    const std::string_view t = Trim(raw);
    if (t.empty()) return;
    if (!IsSpace(raw[0])) return Header(t);
    switch (sec_) {
      case Section::kObjsense: return Objsense(Upper(t));
      case Section::kRows: SplitWs(t, tok_); return RowLine();
      case Section::kColumns: Fields(raw); return ColumnLine();
      case Section::kRhs: Fields(raw); return RhsLine(false);
      case Section::kRanges: Fields(raw); return RhsLine(true);
      case Section::kBounds: Fields(raw); return BoundLine();
      case Section::kEndata: return;
      default: Fail("data line outside of any section");
    }
  }

  bool InColumns() const { return sec_ == Section::kColumns; }

  // The COLUMNS data lines up to the next section header, tokenised on
  // worker threads (row names are looked up in the finished ROWS map, which
  // is read-only from here on), merged in file order on this thread: column
  // indices are assigned in order of first appearance, objective terms
  // accumulate and entries append exactly as the serial ColumnLine does. The
  // first error in file order wins, with its line number.
  void ColumnsBlock(std::string_view block, int threads);

  pdhg_instance* Finish() {
    if (Rank(sec_) < Rank(Section::kColumns)) Fail("missing COLUMNS section");
    if (n_ == 0) Fail("no variables");
    const auto t0 = std::chrono::steady_clock::now();
    pdhg_instance* p = Assemble();
    if (std::getenv("PDHG_TRACE"))
      std::fprintf(stderr, "[mps] assemble %.3fs\n",
                   std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    return p;
  }

 private:
  [[noreturn]] void Fail(const std::string& m) const { throw ParseError{line_, m}; }

  void Fields(std::string_view raw) {
    if (fixed_) SplitFixed(raw, tok_);
    else SplitWs(Trim(raw), tok_);
  }

  void Header(std::string_view h) {
    SplitWs(h, tok_);
    const std::string key = Upper(tok_[0]);
    Section next;
    if (key == "NAME") {
      next = Section::kName;
      if (tok_.size() > 1) name_ = std::string(tok_[1]);
    } else if (key == "OBJSENSE") {
      next = Section::kObjsense;
      if (tok_.size() > 1) Objsense(Upper(tok_[1]));
    } else if (key == "ROWS") {
      next = Section::kRows;
    } else if (key == "COLUMNS") {
      next = Section::kColumns;
    } else if (key == "RHS") {
      next = Section::kRhs;
    } else if (key == "RANGES") {
      next = Section::kRanges;
    } else if (key == "BOUNDS") {
      next = Section::kBounds;
    } else if (key == "ENDATA") {
      next = Section::kEndata;
    } else {
      Fail("unknown section '" + std::string(tok_[0]) + "'");
    }
    if (Rank(next) < Rank(sec_)) Fail("section " + key + " out of order");
    if (next == Section::kRows && Rank(sec_) >= 1) Fail("duplicate ROWS section");
    sec_ = next;
  }

  void Objsense(const std::string& t) {
    if (t == "MAX" || t == "MAXIMIZE") max_ = true;
    else if (t == "MIN" || t == "MINIMIZE") max_ = false;
    else Fail("unknown OBJSENSE '" + t + "'");
  }

  void RowLine() {
    if (tok_.size() != 2) Fail("ROWS line needs a type and a name");
    const std::string type = Upper(tok_[0]);
    const std::string_view name = tok_[1];
    if (row_index_.find(name) != row_index_.end()) Fail("duplicate row '" + std::string(name) + "'");
    if (type == "N") {
      if (!have_obj_) {
        have_obj_ = true;
        row_index_.emplace(name, kObj);
      } else {
        row_index_.emplace(name, kFree);
      }
      return;
    }
    if (type != "E" && type != "G" && type != "L") Fail("unknown row type '" + std::string(tok_[0]) + "'");
    row_index_.emplace(name, static_cast<I>(rows_.size()));
    rows_.push_back({type[0]});
  }

  I Var(std::string_view name) {
    if (last_col_ >= 0 && name == last_name_) return last_col_;
    auto it = col_index_.find(name);
    I j;
    if (it == col_index_.end()) {
      j = n_++;
      col_index_.emplace(name, j);
      obj_.push_back(0.0);
      lo_.push_back(0.0);
      up_.push_back(kInf);
    } else {
      j = it->second;
    }
    last_col_ = j;
    last_name_ = name;
    return j;
  }

  I LookupRow(std::string_view name) const {
    auto it = row_index_.find(name);
    if (it == row_index_.end()) Fail("unknown row '" + std::string(name) + "'");
    return it->second;
  }

  // Numeric field -> double; false with the reference's message on error.
  static bool ParseValue(std::string_view t, double* out, std::string* err) {
    double v = 0.0;
    const char* b = t.data();
    const char* e = b + t.size();
    auto r = std::from_chars(b, e, v);
    if (r.ec != std::errc() || r.ptr != e) {
      const std::string s(t);  // strtod-only spellings: '+', hex, overflow / underflow
      char* end = nullptr;
      v = std::strtod(s.c_str(), &end);
      if (end != s.c_str() + s.size()) {
        *err = "bad numeric value '" + s + "'";
        return false;
      }
    }
    if (std::isnan(v)) {
      *err = "NaN value";
      return false;
    }
    *out = v;
    return true;
  }

  double Value(std::string_view t) const {
    double v = 0.0;
    std::string err;
    if (!ParseValue(t, &v, &err)) Fail(err);
    return v;
  }

  void ColumnLine() {
    if (tok_.size() >= 3 && tok_[1] == "'MARKER'") return;  // integrality markers: discarded
    if (tok_.size() < 3 || tok_.size() % 2 == 0) Fail("COLUMNS line needs a column name and (row, value) pairs");
    const I j = Var(tok_[0]);
    for (size_t i = 1; i + 1 < tok_.size(); i += 2) {
      // The reference evaluates AddCoefficient(LookupRow(..), var, ParseValue(..))'s
      // arguments right to left (GCC x86-64): the value is parsed first.
      const double v = Value(tok_[i + 1]);
      const I r = LookupRow(tok_[i]);
      if (r == kFree) continue;
      if (r == kObj) obj_[j] += v;
      else if (v != 0.0) entries_.push_back({r, j, v});
    }
  }

  void RhsLine(bool range) {
    if (tok_.empty()) Fail("empty data line");
    if (tok_.size() % 2 == 1 && row_index_.find(tok_[0]) == row_index_.end()) tok_.erase(tok_.begin());
    if (tok_.empty() || tok_.size() % 2 != 0) Fail(range ? "malformed RANGES line" : "malformed RHS line");
    for (size_t i = 0; i + 1 < tok_.size(); i += 2) {
      const I r = LookupRow(tok_[i]);
      const double v = Value(tok_[i + 1]);
      if (r == kFree) continue;
      if (r == kObj) {
        if (range) Fail("RANGES entry on objective row");
        obj_rhs_ = v;
        continue;
      }
      if (range) {
        rows_[r].has_range = true;
        rows_[r].range = v;
      } else {
        rows_[r].rhs = v;
      }
    }
  }

  void BoundLine() {
    if (tok_.size() < 2) Fail("malformed BOUNDS line");
    const std::string type = Upper(tok_[0]);
    const bool val = type == "LO" || type == "UP" || type == "FX" || type == "LI" || type == "UI";
    const bool flag = type == "FR" || type == "MI" || type == "PL" || type == "BV";
    if (!val && !flag) Fail("unknown bound type '" + std::string(tok_[0]) + "'");
    const size_t expected = val ? 3 : 2;
    if (tok_.size() == expected + 1 && col_index_.find(tok_[1]) == col_index_.end()) tok_.erase(tok_.begin() + 1);
    if (tok_.size() != expected) Fail("malformed BOUNDS line");
    auto it = col_index_.find(tok_[1]);
    if (it == col_index_.end()) Fail("unknown column '" + std::string(tok_[1]) + "'");
    const I j = it->second;
    const double v = val ? Value(tok_[2]) : 0.0;
    if (type == "LO" || type == "LI") {
      lo_[j] = v;
    } else if (type == "UP" || type == "UI") {
      up_[j] = v;
    } else if (type == "FX") {
      lo_[j] = v;
      up_[j] = v;
    } else if (type == "FR") {
      lo_[j] = -kInf;
      up_[j] = kInf;
    } else if (type == "MI") {
      lo_[j] = -kInf;
    } else if (type == "PL") {
      up_[j] = kInf;
    } else {  // BV
      lo_[j] = 0.0;
      up_[j] = 1.0;
    }
    if (lo_[j] > up_[j]) Fail("conflicting bounds for column '" + std::string(tok_[1]) + "'");
  }

  // Stable counting sort of (row, col, v) by row, then per row by column,
  // duplicates summed in order, zeros dropped.
  static void ToCsr(I rows, std::vector<Entry>& t, std::vector<I>& ptr, std::vector<I>& idx,
                    std::vector<double>& val) {
    std::vector<I> cnt(rows + 1, 0);
    for (const Entry& e : t) ++cnt[e.row + 1];
    for (I r = 0; r < rows; ++r) cnt[r + 1] += cnt[r];
    std::vector<Entry> s(t.size());
    {
      std::vector<I> fill(cnt.begin(), cnt.end() - 1);
      for (const Entry& e : t) s[fill[e.row]++] = e;
    }
    t = std::vector<Entry>();
    ptr.assign(rows + 1, 0);
    idx.clear();
    val.clear();
    idx.reserve(s.size());
    val.reserve(s.size());
    for (I r = 0; r < rows; ++r) {
      auto b = s.begin() + cnt[r], e = s.begin() + cnt[r + 1];
      if (!std::is_sorted(b, e, [](const Entry& x, const Entry& y) { return x.col < y.col; }))
        std::stable_sort(b, e, [](const Entry& x, const Entry& y) { return x.col < y.col; });
      for (auto k = b; k != e;) {
        const I c = k->col;
        double v = 0.0;
        while (k != e && k->col == c) v += (k++)->v;
        if (v != 0.0) {
          idx.push_back(c);
          val.push_back(v);
        }
      }
      ptr[r + 1] = static_cast<I>(idx.size());
    }
  }

  pdhg_instance* Assemble() {
    std::vector<Entry> eq, ineq;
    std::vector<double> b, h;
    // Per-row entry lists in file order (entries_ is in file order already).
    std::vector<I> start(rows_.size() + 1, 0);
    for (const Entry& e : entries_) ++start[e.row + 1];
    for (size_t r = 0; r < rows_.size(); ++r) start[r + 1] += start[r];
    std::vector<Entry> by_row(entries_.size());
    {
      std::vector<I> fill(start.begin(), start.end() - 1);
      for (const Entry& e : entries_) by_row[fill[e.row]++] = e;
    }
    entries_ = std::vector<Entry>();
    for (size_t ri = 0; ri < rows_.size(); ++ri) {
      const Row& row = rows_[ri];
      auto rb = by_row.begin() + start[ri], re = by_row.begin() + start[ri + 1];
      if (!row.has_range) {
        if (row.type == 'E') {
          const I r = static_cast<I>(b.size());
          for (auto k = rb; k != re; ++k) eq.push_back({r, k->col, k->v});
          b.push_back(row.rhs);
        } else {
          const double sign = row.type == 'G' ? 1.0 : -1.0;
          const I r = static_cast<I>(h.size());
          for (auto k = rb; k != re; ++k) ineq.push_back({r, k->col, sign * k->v});
          h.push_back(sign * row.rhs);
        }
        continue;
      }
      double lb, ub;  // lb <= a x <= ub as two G rows
      const double rr = row.range;
      if (row.type == 'G') {
        lb = row.rhs;
        ub = row.rhs + std::abs(rr);
      } else if (row.type == 'L') {
        ub = row.rhs;
        lb = row.rhs - std::abs(rr);
      } else {
        lb = rr >= 0 ? row.rhs : row.rhs + rr;
        ub = rr >= 0 ? row.rhs + rr : row.rhs;
      }
      const I lo = static_cast<I>(h.size());
      for (auto k = rb; k != re; ++k) {
        ineq.push_back({lo, k->col, k->v});
        ineq.push_back({lo + 1, k->col, -k->v});
      }
      h.push_back(lb);
      h.push_back(-ub);
    }
    auto* p = new pdhg_instance;
    try {
      p->name = name_;
      p->n = n_;
      p->a_rows = static_cast<I>(b.size());
      p->g_rows = static_cast<I>(h.size());
      ToCsr(p->a_rows, eq, p->a_ptr, p->a_idx, p->a_val);
      ToCsr(p->g_rows, ineq, p->g_ptr, p->g_idx, p->g_val);
      p->b = std::move(b);
      p->h = std::move(h);
      p->c = std::move(obj_);
      p->l = std::move(lo_);
      p->u = std::move(up_);
      p->offset = -obj_rhs_;
      if (max_) {
        for (double& v : p->c) v = -v;
        p->offset = -p->offset;
        p->negated = 1;
      }
      pdhg_lp view;
      pdhg_instance_view(p, &view);
      pdhg::ValidateLpHost(view);  // LpProblem::Validate (lp_problem.cpp:22-58)
    } catch (...) {
      delete p;
      throw;
    }
    return p;
  }

  static constexpr I kObj = -1;
  static constexpr I kFree = -2;

  bool fixed_;
  int line_ = 0;
  Section sec_ = Section::kNone;
  std::string name_;
  bool max_ = false;
  bool have_obj_ = false;
  double obj_rhs_ = 0.0;
  NameMap row_index_, col_index_;
  std::vector<Row> rows_;
  std::vector<Entry> entries_;
  I n_ = 0;
  std::vector<double> obj_, lo_, up_;
  std::vector<std::string_view> tok_;
  I last_col_ = -1;
  std::string_view last_name_;
};

// One COLUMNS line's worth of work, produced on a worker thread.
struct ColRun {
  std::string_view name;
  size_t e0, e1;  // entries [e0, e1) of the chunk
  size_t o0, o1;  // objective terms [o0, o1) of the chunk
};
struct ColChunk {
  std::string_view text;
  std::vector<ColRun> runs;
  std::vector<std::pair<I, double>> entries;  // (row, value), file order
  std::vector<double> obj;                    // objective terms, file order
  int lines = 0;                              // lines in the chunk
  int err_line = -1;                          // chunk-local line of the first error
  std::string err;
};

void Reader::ColumnsBlock(std::string_view block, int threads) {
  // Chunks of roughly equal bytes, cut at line starts.
  const size_t nb = block.size();
  int T = std::max(1, std::min<int>(threads, static_cast<int>(nb >> 20)));  // >= 1 MB per chunk
  std::vector<ColChunk> ch(static_cast<size_t>(T));
  size_t a = 0;
  for (int k = 0; k < T; ++k) {
    size_t b = (k == T - 1) ? nb : std::max(a, nb * static_cast<size_t>(k + 1) / T);
    if (b < nb) {
      const size_t nl = block.find('\n', b);
      b = nl == std::string_view::npos ? nb : nl + 1;
    }
    ch[k].text = block.substr(a, b - a);
    a = b;
  }
  auto work = [this](ColChunk& c) {
    std::vector<std::string_view> tok;
    std::string_view last;
    bool have = false;
    size_t i = 0;
    const std::string_view t = c.text;
    while (i < t.size()) {
      size_t j = t.find('\n', i);
      if (j == std::string_view::npos) j = t.size();
      const std::string_view raw = t.substr(i, j - i);
      i = j + 1;
      ++c.lines;
      if (raw.empty() || raw[0] == '*' || Trim(raw).empty()) continue;
      if (fixed_) SplitFixed(raw, tok);
      else SplitWs(Trim(raw), tok);
      if (tok.size() >= 3 && tok[1] == "'MARKER'") continue;
      auto fail = [&](std::string m) {
        c.err_line = c.lines;
        c.err = std::move(m);
      };
      if (tok.size() < 3 || tok.size() % 2 == 0) {
        fail("COLUMNS line needs a column name and (row, value) pairs");
        return;
      }
      if (!have || tok[0] != last) {
        c.runs.push_back({tok[0], c.entries.size(), c.entries.size(), c.obj.size(), c.obj.size()});
        last = tok[0];
        have = true;
      }
      for (size_t k = 1; k + 1 < tok.size(); k += 2) {
        double v;  // value first, then the row (the reference's argument order)
        if (!ParseValue(tok[k + 1], &v, &c.err)) {
          c.err_line = c.lines;
          return;
        }
        auto it = row_index_.find(tok[k]);
        if (it == row_index_.end()) {
          fail("unknown row '" + std::string(tok[k]) + "'");
          return;
        }
        const I r = it->second;
        if (r == kFree) continue;
        if (r == kObj) c.obj.push_back(v);
        else if (v != 0.0) c.entries.emplace_back(r, v);
      }
      c.runs.back().e1 = c.entries.size();
      c.runs.back().o1 = c.obj.size();
    }
  };
  const auto tw0 = std::chrono::steady_clock::now();
  if (T == 1) {
    work(ch[0]);
  } else {
    std::vector<std::thread> pool;
    for (int k = 1; k < T; ++k) pool.emplace_back(work, std::ref(ch[k]));
    work(ch[0]);
    for (std::thread& th : pool) th.join();
  }
  const auto tw1 = std::chrono::steady_clock::now();
  // Merge in file order; stop at the first error.
  size_t nruns = 0, nent = 0;
  for (const ColChunk& c : ch) {
    nruns += c.runs.size();
    nent += c.entries.size();
  }
  col_index_.reserve(col_index_.size() + nruns);
  obj_.reserve(obj_.size() + nruns);
  lo_.reserve(lo_.size() + nruns);
  up_.reserve(up_.size() + nruns);
  entries_.reserve(entries_.size() + nent);
  for (const ColChunk& c : ch) {
    for (const ColRun& r : c.runs) {
      const I j = Var(r.name);
      for (size_t k = r.o0; k < r.o1; ++k) obj_[j] += c.obj[k];
      for (size_t k = r.e0; k < r.e1; ++k) entries_.push_back({c.entries[k].first, j, c.entries[k].second});
    }
    if (c.err_line >= 0) throw ParseError{line_ + c.err_line, c.err};
    line_ += c.lines;
  }
  if (std::getenv("PDHG_TRACE"))
    std::fprintf(stderr, "[mps] COLUMNS %zu bytes: %d chunks, tokenise %.3fs, merge %.3fs\n", nb, T,
                 std::chrono::duration<double>(tw1 - tw0).count(),
                 std::chrono::duration<double>(std::chrono::steady_clock::now() - tw1).count());
}

pdhg_instance* ParseText(std::string_view text, bool fixed) {
  Reader rd(fixed);
  static const int kThreads = [] {
    const char* e = std::getenv("PDHG_MPS_THREADS");  // "1": serial COLUMNS (A/B)
    const int hw = static_cast<int>(std::thread::hardware_concurrency());
    return e ? std::max(1, std::atoi(e)) : std::max(1, std::min(hw, 32));
  }();
  size_t i = 0;
  while (i < text.size()) {  // std::getline semantics: no empty line after a final '\n'
    if (rd.InColumns() && kThreads > 1) {
      // The COLUMNS block: every line up to the next header line.
      size_t k = i;
      while (k < text.size()) {
        const char c0 = text[k];
        if (c0 != '*' && !IsSpace(c0)) break;  // a header starts in column 1
        const size_t nl = text.find('\n', k);
        k = nl == std::string_view::npos ? text.size() : nl + 1;
      }
      if (k > i) {
        rd.ColumnsBlock(text.substr(i, k - i), kThreads);
        i = k;
        continue;
      }
    }
    size_t j = text.find('\n', i);
    if (j == std::string_view::npos) j = text.size();
    rd.Line(text.substr(i, j - i));
    i = j + 1;
  }
  return rd.Finish();
}

std::string ReadFile(const std::string& path) {
  if (path.size() > 3 && path.compare(path.size() - 3, 3, ".gz") == 0) {
    gzFile f = gzopen(path.c_str(), "rb");
    if (!f) throw IoError{"cannot open " + path};
    gzbuffer(f, 1 << 20);
    std::string out;
    std::vector<char> buf(1 << 20);
    int n;
    while ((n = gzread(f, buf.data(), static_cast<unsigned>(buf.size()))) > 0) out.append(buf.data(), n);
    const bool bad = n < 0;
    gzclose(f);
    if (bad) throw IoError{"gzip read error in " + path};
    return out;
  }
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw IoError{"cannot open " + path};
  std::string out;
  std::fseek(f, 0, SEEK_END);
  const long len = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  if (len > 0) {
    out.resize(static_cast<size_t>(len));
    const size_t got = std::fread(out.data(), 1, out.size(), f);
    out.resize(got);
  }
  std::fclose(f);
  return out;
}

// %.17g, as the reference writer (mps_writer.cpp Num).
void Num(std::string& out, double v) {
  char buf[64];
  const int k = std::snprintf(buf, sizeof(buf), "%.17g", v);
  out.append(buf, k);
}

// WriteMps (mps_writer.cpp:37-107): free format, E rows, G rows, every
// column with its objective entry, RHS / BOUNDS only where not default.
std::string WriteText(const pdhg_lp& p, const char* name) {
  pdhg::ValidateLpHost(p);
  const I m1 = p.a.rows, m2 = p.g.rows, n = p.n;
  // Column-major view of A and G (CSC): counting sort by column.
  auto csc = [n](const pdhg_csr& m, std::vector<I>& cp, std::vector<I>& ri, std::vector<double>& cv) {
    const I nnz = m.rows ? m.row_ptr[m.rows] : 0;
    cp.assign(n + 1, 0);
    for (I k = 0; k < nnz; ++k) ++cp[m.col_idx[k] + 1];
    for (I j = 0; j < n; ++j) cp[j + 1] += cp[j];
    ri.resize(nnz);
    cv.resize(nnz);
    std::vector<I> fill(cp.begin(), cp.end() - 1);
    for (I r = 0; r < m.rows; ++r)
      for (I k = m.row_ptr[r]; k < m.row_ptr[r + 1]; ++k) {
        const I d = fill[m.col_idx[k]]++;
        ri[d] = r;
        cv[d] = m.values[k];
      }
  };
  std::vector<I> acp, ari, gcp, gri;
  std::vector<double> acv, gcv;
  csc(p.a, acp, ari, acv);
  csc(p.g, gcp, gri, gcv);
  std::string o;
  o.reserve(static_cast<size_t>(64) * (acv.size() + gcv.size() + n + m1 + m2) + 256);
  o += "NAME ";
  o += (name && name[0]) ? name : "LP";
  o += "\n";
  if (p.negated_objective) o += "OBJSENSE\n MAX\n";
  o += "ROWS\n N OBJ\n";
  for (I i = 0; i < m1; ++i) o += " E E" + std::to_string(i) + "\n";
  for (I i = 0; i < m2; ++i) o += " G G" + std::to_string(i) + "\n";
  const double sign = p.negated_objective ? -1.0 : 1.0;
  o += "COLUMNS\n";
  for (I j = 0; j < n; ++j) {
    const std::string cn = " X" + std::to_string(j) + " ";
    o += cn + "OBJ ";
    Num(o, sign * p.c[j]);
    o += "\n";
    for (I k = acp[j]; k < acp[j + 1]; ++k) {
      o += cn + "E" + std::to_string(ari[k]) + " ";
      Num(o, acv[k]);
      o += "\n";
    }
    for (I k = gcp[j]; k < gcp[j + 1]; ++k) {
      o += cn + "G" + std::to_string(gri[k]) + " ";
      Num(o, gcv[k]);
      o += "\n";
    }
  }
  o += "RHS\n";
  if (p.objective_offset != 0.0) {
    o += " RHS OBJ ";
    Num(o, sign * -p.objective_offset);
    o += "\n";
  }
  for (I i = 0; i < m1; ++i)
    if (p.b[i] != 0.0) {
      o += " RHS E" + std::to_string(i) + " ";
      Num(o, p.b[i]);
      o += "\n";
    }
  for (I i = 0; i < m2; ++i)
    if (p.h[i] != 0.0) {
      o += " RHS G" + std::to_string(i) + " ";
      Num(o, p.h[i]);
      o += "\n";
    }
  o += "BOUNDS\n";
  for (I j = 0; j < n; ++j) {
    const double l = p.l[j], u = p.u[j];
    if (l == 0.0 && u == kInf) continue;
    const std::string cn = " BND X" + std::to_string(j);
    if (std::isinf(l) && std::isinf(u)) {
      o += " FR" + cn + "\n";
      continue;
    }
    if (l == u) {
      o += " FX" + cn + " ";
      Num(o, l);
      o += "\n";
      continue;
    }
    if (std::isinf(l)) {
      o += " MI" + cn + "\n";
    } else if (l != 0.0) {
      o += " LO" + cn + " ";
      Num(o, l);
      o += "\n";
    }
    if (!std::isinf(u)) {
      o += " UP" + cn + " ";
      Num(o, u);
      o += "\n";
    }
  }
  o += "ENDATA\n";
  return o;
}

template <class F>
int Guard(char* err, size_t len, int* err_line, F&& f) {
  if (err_line) *err_line = 0;
  try {
    f();
    return PDHG_OK;
  } catch (const ParseError& e) {
    if (err && len) std::snprintf(err, len, "mps parse error at line %d: %s", e.line, e.msg.c_str());
    if (err_line) *err_line = e.line;
    return PDHG_PARSE_ERROR;
  } catch (const IoError& e) {
    if (err && len) std::snprintf(err, len, "%s", e.msg.c_str());
    return PDHG_IO_ERROR;
  } catch (const std::invalid_argument& e) {
    if (err && len) std::snprintf(err, len, "%s", e.what());
    return PDHG_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    if (err && len) std::snprintf(err, len, "%s", e.what());
    return PDHG_IO_ERROR;
  }
}

}  // namespace

extern "C" {

int pdhg_mps_read_string(const char* text, size_t len, int fixed_format, pdhg_instance** out, char* err,
                         size_t errlen, int* err_line) {
  return Guard(err, errlen, err_line, [&] {
    if (!out || (!text && len)) throw std::invalid_argument("null argument");
    *out = ParseText(std::string_view(text ? text : "", len), fixed_format != 0);
  });
}

int pdhg_mps_read_file(const char* path, int fixed_format, pdhg_instance** out, char* err, size_t errlen,
                       int* err_line) {
  return Guard(err, errlen, err_line, [&] {
    if (!out || !path) throw std::invalid_argument("null argument");
    const std::string text = ReadFile(path);
    *out = ParseText(text, fixed_format != 0);
  });
}

const char* pdhg_instance_name(const pdhg_instance* p) { return p ? p->name.c_str() : ""; }

int pdhg_mps_write_string(const pdhg_lp* lp, const char* name, char** out, size_t* out_len, char* err,
                          size_t errlen) {
  return Guard(err, errlen, nullptr, [&] {
    if (!lp || !out || !out_len) throw std::invalid_argument("null argument");
    const std::string s = WriteText(*lp, name);
    char* buf = static_cast<char*>(std::malloc(s.size() + 1));
    if (!buf) throw std::bad_alloc();
    std::memcpy(buf, s.data(), s.size());
    buf[s.size()] = '\0';
    *out = buf;
    *out_len = s.size();
  });
}

void pdhg_free_string(char* s) { std::free(s); }

int pdhg_mps_write_file(const pdhg_lp* lp, const char* name, const char* path, char* err, size_t errlen) {
  return Guard(err, errlen, nullptr, [&] {
    if (!lp || !path) throw std::invalid_argument("null argument");
    const std::string s = WriteText(*lp, name);
    std::FILE* f = std::fopen(path, "wb");
    if (!f) throw IoError{std::string("cannot open ") + path + " for writing"};
    const size_t w = std::fwrite(s.data(), 1, s.size(), f);
    const bool bad = std::fclose(f) != 0 || w != s.size();
    if (bad) throw IoError{std::string("write failed for ") + path};
  });
}

}  // extern "C"
