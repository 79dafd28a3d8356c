// hpr_mps.cpp -- MPS reader / writer: the step before
// the solve path for real instances.  Host C++ behind the C ABI
// (include/hprlp_b200.h, hpr_mps_*), same semantics as the reference
// /root/reference/pkg/src/hprlp/mps.py:
//
//   read_document   mps.py:60-154  fixed/free format, '*' comments, section order
//                                  checks, N/E/L/G rows, 'MARKER' lines skipped,
//                                  optional RHS/RANGES set names, bound kinds
//                                  LO UP FX FR MI PL BV; errors "line N: ..."
//   document_to_problem 157-278    columns numbered by first appearance,
//                                  objective entries summed, objective-row RHS
//                                  -> constant -rhs, RANGES split into a >= / <=
//                                  pair, L rows negated into >= form, OBJSENSE
//                                  MAX negates c and the constant; CSR blocks in
//                                  canonical form (columns sorted, duplicates
//                                  summed in file order, zeros dropped)
//   write_mps       mps.py:295-364 the same text, %.17g numbers
//
// Parsing is a single pass over the text with no per-token allocations
// beyond the name tables; the output arrays are owned by the result object
// and released with hpr_mps_free.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

#include "../../include/hprlp_b200.h"

namespace {

thread_local std::string g_mps_err;

struct ParseError {
  long long line;
  std::string msg;
};

enum Section { S_NONE = -1, S_NAME, S_OBJSENSE, S_ROWS, S_COLUMNS, S_RHS, S_RANGES, S_BOUNDS, S_ENDATA };

int section_order(Section s) {
  switch (s) {
    case S_NAME: return 0;
    case S_OBJSENSE: return 1;
    case S_ROWS: return 2;
    case S_COLUMNS: return 3;
    case S_RHS: case S_RANGES: case S_BOUNDS: return 4;
    case S_ENDATA: return 5;
    default: return -1;
  }
}

Section section_of(std::string_view h) {
  if (h == "NAME") return S_NAME;
  if (h == "OBJSENSE") return S_OBJSENSE;
  if (h == "ROWS") return S_ROWS;
  if (h == "COLUMNS") return S_COLUMNS;
  if (h == "RHS") return S_RHS;
  if (h == "RANGES") return S_RANGES;
  if (h == "BOUNDS") return S_BOUNDS;
  if (h == "ENDATA") return S_ENDATA;
  return S_NONE;
}

bool is_space(char ch) {
  return ch == ' ' || ch == '\t' || ch == '\n' || ch == '\r' || ch == '\v' || ch == '\f' ||
         ch == '\x1c' || ch == '\x1d' || ch == '\x1e' || ch == '\x1f';
}

// Python float(): decimal literals, optional sign, inf/infinity/nan in any
// case, single underscores between digits; no hex.
bool py_float(std::string_view tok, double *out) {
  std::string s;
  s.reserve(tok.size());
  for (size_t i = 0; i < tok.size(); ++i) {
    const char ch = tok[i];
    if (ch == '_') {
      if (i == 0 || i + 1 == tok.size() || !isdigit((unsigned char)tok[i - 1]) ||
          !isdigit((unsigned char)tok[i + 1]))
        return false;
      continue;
    }
    if (ch == 'x' || ch == 'X' || ch == 'p' || ch == 'P' || ch == '(' || ch == ')') return false;
    s.push_back(ch);
  }
  if (s.empty()) return false;
  std::string low;
  for (char ch : s) low.push_back((char)tolower((unsigned char)ch));
  std::string_view body = low;
  double sign = 1.0;
  if (!body.empty() && (body[0] == '+' || body[0] == '-')) {
    if (body[0] == '-') sign = -1.0;
    body.remove_prefix(1);
  }
  if (body == "inf" || body == "infinity") {
    *out = sign * INFINITY;
    return true;
  }
  if (body == "nan") {
    *out = sign * NAN;
    return true;
  }
  // remaining: digits, '.', 'e', sign after e
  bool digit = false;
  for (char ch : body) {
    if (isdigit((unsigned char)ch)) digit = true;
    else if (ch != '.' && ch != 'e' && ch != '+' && ch != '-') return false;
  }
  if (!digit) return false;
  errno = 0;
  char *end = nullptr;
  const double v = strtod(s.c_str(), &end);
  if (end != s.c_str() + s.size()) return false;
  *out = v;   // overflow gives +-inf like Python; underflow gives the rounded subnormal / 0
  return true;
}

struct ColRec {
  int col;
  int row;    // -1: objective row, -2: unknown (name stored)
  double val;
  long long line;
  std::string unknown;
};
struct RowRec {
  std::string row;
  double val;
  long long line;
};
struct BoundRec {
  std::string kind, col;
  double val;
  bool has_val;
  long long line;
};

struct Doc {
  std::string name = "UNNAMED";
  bool maximize = false;
  std::vector<char> kinds;            // row kinds (E/L/G), file order
  std::vector<std::string> rows;      // row names
  std::unordered_map<std::string, int> row_index;
  std::string objective_row;
  bool has_objective = false;
  int extra_objective_rows = 0;
  std::vector<std::string> cols;
  std::unordered_map<std::string, int> col_index;
  std::vector<ColRec> columns;
  std::vector<RowRec> rhs, ranges;
  std::vector<BoundRec> bounds;
};

void split(std::string_view line, std::vector<std::string_view> &tok) {
  tok.clear();
  size_t i = 0;
  while (i < line.size()) {
    while (i < line.size() && is_space(line[i])) ++i;
    size_t j = i;
    while (j < line.size() && !is_space(line[j])) ++j;
    if (j > i) tok.emplace_back(line.substr(i, j - i));
    i = j;
  }
}

[[noreturn]] void perr(long long line, const std::string &msg) { throw ParseError{line, msg}; }

void pairs_of(const std::vector<std::string_view> &t, long long ln, std::vector<RowRec> &out) {
  const size_t first = (t.size() % 2 == 1) ? 1 : 0;   // odd count: a set name leads
  const size_t np = t.size() - first;
  if (np == 0 || np % 2 != 0) perr(ln, "expected '[setname] (<row> <value>)+'");
  for (size_t i = first; i < t.size(); i += 2) {
    double v;
    if (!py_float(t[i + 1], &v)) perr(ln, "bad numeric '" + std::string(t[i + 1]) + "'");
    out.push_back({std::string(t[i]), v, ln});
  }
}

void read_document(const char *text, size_t len, Doc &doc) {
  std::vector<std::string_view> tok;
  std::vector<Section> seen;
  Section section = S_NONE;
  long long line_no = 0;
  size_t pos = 0;
  bool have_rows = false, have_cols = false;
  while (pos < len) {
    size_t e = pos;
    while (e < len && text[e] != '\n') ++e;
    std::string_view raw(text + pos, e - pos);
    pos = e + 1;
    ++line_no;
    if (!raw.empty() && raw[0] == '*') continue;
    split(raw, tok);
    if (tok.empty()) continue;
    const bool is_header = !is_space(raw[0]);
    const std::string_view head = tok[0];
    const Section hs = section_of(head);
    if (is_header && hs != S_NONE) {
      if (!seen.empty() && section_order(hs) < section_order(seen.back()))
        perr(line_no, "section " + std::string(head) + " out of order");
      if ((hs == S_RHS || hs == S_RANGES || hs == S_BOUNDS) && !have_cols)
        perr(line_no, "section " + std::string(head) + " before COLUMNS");
      if (hs == S_COLUMNS && !have_rows) perr(line_no, "COLUMNS before ROWS");
      seen.push_back(hs);
      if (hs == S_ROWS) have_rows = true;
      if (hs == S_COLUMNS) have_cols = true;
      section = hs;
      if (hs == S_NAME && tok.size() > 1) doc.name = std::string(tok[1]);
      if (hs == S_OBJSENSE && tok.size() > 1) {
        std::string u(tok[1]);
        for (auto &ch : u) ch = (char)toupper((unsigned char)ch);
        doc.maximize = u.rfind("MAX", 0) == 0;
      }
      if (hs == S_ENDATA) break;
      continue;
    }
    if (is_header) perr(line_no, "unknown section '" + std::string(head) + "'");
    switch (section) {
      case S_OBJSENSE: {
        std::string u(head);
        for (auto &ch : u) ch = (char)toupper((unsigned char)ch);
        doc.maximize = u.rfind("MAX", 0) == 0;
        break;
      }
      case S_ROWS: {
        if (tok.size() != 2 || tok[0].size() != 1 ||
            (tok[0][0] != 'N' && tok[0][0] != 'E' && tok[0][0] != 'L' && tok[0][0] != 'G'))
          perr(line_no, "expected '<N|E|L|G> <rowname>'");
        const char kind = tok[0][0];
        std::string nm(tok[1]);
        if (kind == 'N') {
          if (!doc.has_objective) {
            doc.objective_row = nm;
            doc.has_objective = true;
          } else {
            doc.extra_objective_rows += 1;
          }
          break;
        }
        if (doc.row_index.count(nm)) perr(line_no, "duplicate row '" + nm + "'");
        doc.row_index.emplace(nm, (int)doc.rows.size());
        doc.rows.push_back(nm);
        doc.kinds.push_back(kind);
        break;
      }
      case S_COLUMNS: {
        if (tok.size() >= 3 && tok[1] == "'MARKER'") break;   // integrality markers
        if (tok.size() < 3 || tok.size() % 2 == 0) perr(line_no, "expected '<col> (<row> <value>)+'");
        std::string col(tok[0]);
        for (size_t i = 1; i < tok.size(); i += 2) {
          double v;
          if (!py_float(tok[i + 1], &v)) perr(line_no, "bad numeric '" + std::string(tok[i + 1]) + "'");
          ColRec r;
          auto it = doc.col_index.find(col);
          int j;
          if (it == doc.col_index.end()) {
            j = (int)doc.cols.size();
            doc.col_index.emplace(col, j);
            doc.cols.push_back(col);
          } else {
            j = it->second;
          }
          r.col = j;
          r.val = v;
          r.line = line_no;
          const std::string rn(tok[i]);
          if (doc.has_objective && rn == doc.objective_row) {
            r.row = -1;
          } else {
            auto ri = doc.row_index.find(rn);
            if (ri == doc.row_index.end()) {
              r.row = -2;
              r.unknown = rn;
            } else {
              r.row = ri->second;
            }
          }
          doc.columns.push_back(std::move(r));
        }
        break;
      }
      case S_RHS:
        pairs_of(tok, line_no, doc.rhs);
        break;
      case S_RANGES:
        pairs_of(tok, line_no, doc.ranges);
        break;
      case S_BOUNDS: {
        std::string kind(tok[0]);
        for (auto &ch : kind) ch = (char)toupper((unsigned char)ch);
        if (kind == "FR" || kind == "MI" || kind == "PL" || kind == "BV") {
          if (tok.size() < 3) perr(line_no, "expected '<kind> <setname> <col>'");
          doc.bounds.push_back({kind, std::string(tok[2]), 0.0, false, line_no});
        } else if (kind == "LO" || kind == "UP" || kind == "FX") {
          if (tok.size() < 4) perr(line_no, "expected '<kind> <setname> <col> <value>'");
          double v;
          if (!py_float(tok[3], &v)) perr(line_no, "bad numeric '" + std::string(tok[3]) + "'");
          doc.bounds.push_back({kind, std::string(tok[2]), v, true, line_no});
        } else {
          perr(line_no, "unknown bound kind '" + std::string(tok[0]) + "'");
        }
        break;
      }
      default:
        perr(line_no, "data before any section header");
    }
  }
  if (!have_rows || !have_cols) perr(0, "missing ROWS or COLUMNS section");
}

// canonical CSR of rows given as (col, val) lists: stable column sort,
// duplicates summed in file order, zeros dropped (SparseMatrix.from_coo)
void build_csr(const std::vector<std::vector<std::pair<int, double>>> &rows,
               const std::vector<double> &sign, std::vector<int64_t> &rp, std::vector<int64_t> &ci,
               std::vector<double> &val) {
  rp.assign(rows.size() + 1, 0);
  std::vector<std::pair<int, double>> tmp;
  for (size_t i = 0; i < rows.size(); ++i) {
    tmp = rows[i];
    std::stable_sort(tmp.begin(), tmp.end(),
                     [](const std::pair<int, double> &a, const std::pair<int, double> &b) {
                       return a.first < b.first;
                     });
    size_t k = 0;
    while (k < tmp.size()) {
      const int c = tmp[k].first;
      double s = sign[i] * tmp[k].second;
      size_t q = k + 1;
      while (q < tmp.size() && tmp[q].first == c) {
        s += sign[i] * tmp[q].second;
        ++q;
      }
      if (s != 0.0) {
        ci.push_back(c);
        val.push_back(s);
      }
      k = q;
    }
    rp[i + 1] = (int64_t)ci.size();
  }
}

template <class T>
T *dup_vec(const std::vector<T> &v) {
  T *p = (T *)malloc(sizeof(T) * (v.size() ? v.size() : 1));
  if (!v.empty()) memcpy(p, v.data(), sizeof(T) * v.size());
  return p;
}

char *dup_names(const std::vector<std::string> &names, size_t *bytes) {
  size_t total = 0;
  for (auto &s : names) total += s.size() + 1;
  char *p = (char *)malloc(total ? total : 1);
  size_t o = 0;
  for (auto &s : names) {
    memcpy(p + o, s.c_str(), s.size() + 1);
    o += s.size() + 1;
  }
  *bytes = total;
  return p;
}

void to_problem(const Doc &doc, hpr_mps_result *R) {
  const int nrows = (int)doc.rows.size();
  const int n = (int)doc.cols.size();
  std::vector<std::vector<std::pair<int, double>>> entries(nrows);
  std::vector<double> obj(n, 0.0);
  for (const auto &r : doc.columns) {
    if (r.row == -1) {
      obj[r.col] = obj[r.col] + r.val;
      continue;
    }
    if (r.row == -2) perr(r.line, "unknown row '" + r.unknown + "'");
    entries[r.row].push_back({r.col, r.val});
  }
  std::vector<double> rhs(nrows, 0.0);
  double objective_constant = 0.0;
  for (const auto &r : doc.rhs) {
    if (doc.has_objective && r.row == doc.objective_row) {
      objective_constant = -r.val;
      continue;
    }
    auto it = doc.row_index.find(r.row);
    if (it == doc.row_index.end()) perr(r.line, "unknown row '" + r.row + "'");
    rhs[it->second] = r.val;
  }
  std::vector<char> has_range(nrows, 0);
  std::vector<double> range_val(nrows, 0.0);
  for (const auto &r : doc.ranges) {
    auto it = doc.row_index.find(r.row);
    if ((doc.has_objective && r.row == doc.objective_row) || it == doc.row_index.end())
      perr(r.line, "RANGES references unknown row '" + r.row + "'");
    has_range[it->second] = 1;
    range_val[it->second] = r.val;
  }
  std::vector<double> lower(n, 0.0), upper(n, INFINITY);
  for (const auto &b : doc.bounds) {
    auto it = doc.col_index.find(b.col);
    if (it == doc.col_index.end()) perr(b.line, "BOUNDS references unknown column '" + b.col + "'");
    const int j = it->second;
    if (b.kind == "LO") lower[j] = b.val;
    else if (b.kind == "UP") upper[j] = b.val;
    else if (b.kind == "FX") lower[j] = upper[j] = b.val;
    else if (b.kind == "FR") { lower[j] = -INFINITY; upper[j] = INFINITY; }
    else if (b.kind == "MI") lower[j] = -INFINITY;
    else if (b.kind == "PL") upper[j] = INFINITY;
    else if (b.kind == "BV") { lower[j] = 0.0; upper[j] = 1.0; }
    if (lower[j] > upper[j]) perr(b.line, "conflicting bounds for column '" + b.col + "'");
  }
  // equality rows first, then >= rows (L negated, ranged rows split)
  std::vector<std::vector<std::pair<int, double>>> eq_rows, ge_rows;
  std::vector<double> eq_b, ge_b, eq_sign, ge_sign;
  std::vector<std::string> eq_names, ge_names;
  for (int i = 0; i < nrows; ++i) {
    const char kind = doc.kinds[i];
    const double bi = rhs[i];
    if (has_range[i]) {
      const double r = range_val[i];
      double lo, hi;
      if (kind == 'G') {
        lo = bi;
        hi = bi + std::fabs(r);
      } else if (kind == 'L') {
        lo = bi - std::fabs(r);
        hi = bi;
      } else if (r >= 0) {
        lo = bi;
        hi = bi + r;
      } else {
        lo = bi + r;
        hi = bi;
      }
      ge_rows.push_back(entries[i]);
      ge_b.push_back(lo);
      ge_sign.push_back(1.0);
      ge_names.push_back(doc.rows[i]);
      ge_rows.push_back(entries[i]);
      ge_b.push_back(-hi);
      ge_sign.push_back(-1.0);
      ge_names.push_back(doc.rows[i] + ":rng");
    } else if (kind == 'E') {
      eq_rows.push_back(entries[i]);
      eq_b.push_back(bi);
      eq_sign.push_back(1.0);
      eq_names.push_back(doc.rows[i]);
    } else if (kind == 'G') {
      ge_rows.push_back(entries[i]);
      ge_b.push_back(bi);
      ge_sign.push_back(1.0);
      ge_names.push_back(doc.rows[i]);
    } else {
      ge_rows.push_back(entries[i]);
      ge_b.push_back(-bi);
      ge_sign.push_back(-1.0);
      ge_names.push_back(doc.rows[i]);
    }
  }
  std::vector<int64_t> erp, eci, irp, ici;
  std::vector<double> ev, iv;
  build_csr(eq_rows, eq_sign, erp, eci, ev);
  build_csr(ge_rows, ge_sign, irp, ici, iv);
  std::vector<double> c = obj;
  if (doc.maximize) {
    for (auto &v : c) v = -v;
    objective_constant = -objective_constant;
  }
  R->m1 = (int64_t)eq_rows.size();
  R->m2 = (int64_t)ge_rows.size();
  R->n = n;
  R->eq_rp = dup_vec(erp);
  R->eq_ci = dup_vec(eci);
  R->eq_val = dup_vec(ev);
  R->in_rp = dup_vec(irp);
  R->in_ci = dup_vec(ici);
  R->in_val = dup_vec(iv);
  R->b_eq = dup_vec(eq_b);
  R->b_ineq = dup_vec(ge_b);
  R->c = dup_vec(c);
  R->lower = dup_vec(lower);
  R->upper = dup_vec(upper);
  R->objective_constant = objective_constant;
  R->objective_negated = doc.maximize ? 1 : 0;
  R->extra_objective_rows = doc.extra_objective_rows;
  std::vector<std::string> rn = eq_names;
  rn.insert(rn.end(), ge_names.begin(), ge_names.end());
  size_t b1 = 0, b2 = 0;
  R->row_names = dup_names(rn, &b1);
  R->col_names = dup_names(doc.cols, &b2);
  R->name = strdup(doc.name.c_str());
}

void fmt17(std::string &out, double v) {
  char buf[64];
  if (std::isinf(v)) {
    out += v > 0 ? "inf" : "-inf";
    return;
  }
  snprintf(buf, sizeof(buf), "%.17g", v);
  out += buf;
}

}  // namespace

extern "C" {

int hpr_mps_parse(const char *text, size_t len, hpr_mps_result **out) {
  if (!out || (!text && len)) {
    g_mps_err = "null argument";
    return HPR_EINVAL;
  }
  *out = nullptr;
  hpr_mps_result *R = (hpr_mps_result *)calloc(1, sizeof(hpr_mps_result));
  try {
    Doc doc;
    read_document(text, len, doc);
    to_problem(doc, R);
  } catch (const ParseError &e) {
    hpr_mps_free(R);
    g_mps_err = "line " + std::to_string(e.line) + ": " + e.msg;
    return HPR_EINVAL;
  } catch (const std::exception &e) {
    hpr_mps_free(R);
    g_mps_err = std::string("mps: ") + e.what();
    return HPR_ENOMEM;
  }
  *out = R;
  return HPR_OK;
}

const char *hpr_mps_last_error(void) { return g_mps_err.c_str(); }

int hpr_mps_free(hpr_mps_result *R) {
  if (!R) return HPR_OK;
  free(R->eq_rp); free(R->eq_ci); free(R->eq_val);
  free(R->in_rp); free(R->in_ci); free(R->in_val);
  free(R->b_eq); free(R->b_ineq); free(R->c); free(R->lower); free(R->upper);
  free(R->row_names); free(R->col_names); free(R->name);
  free(R);
  return HPR_OK;
}

// write_mps (mps.py:295-364)
int hpr_mps_write(const hpr_mps_problem *p, const char *name, char **text, size_t *len) {
  if (!p || !text || !len) {
    g_mps_err = "null argument";
    return HPR_EINVAL;
  }
  const int64_t m1 = p->m1, m2 = p->m2, n = p->n;
  std::vector<std::string> rows, cols;
  if (p->row_names) {
    const char *s = p->row_names;
    for (int64_t i = 0; i < m1 + m2; ++i) {
      rows.emplace_back(s);
      s += rows.back().size() + 1;
    }
  } else {
    for (int64_t i = 0; i < m1; ++i) rows.push_back("EQ" + std::to_string(i));
    for (int64_t i = 0; i < m2; ++i) rows.push_back("GE" + std::to_string(i));
  }
  if (p->col_names) {
    const char *s = p->col_names;
    for (int64_t j = 0; j < n; ++j) {
      cols.emplace_back(s);
      s += cols.back().size() + 1;
    }
  } else {
    for (int64_t j = 0; j < n; ++j) cols.push_back("X" + std::to_string(j));
  }
  const double sign = p->objective_negated ? -1.0 : 1.0;
  std::string out;
  out.reserve(64 * (size_t)(n + m1 + m2) + 48 * (size_t)(p->eq_rp[m1] + p->in_rp[m2]));
  out += "NAME          ";
  out += name ? name : "LP";
  out += "\n";
  if (p->objective_negated) out += "OBJSENSE\n    MAX\n";
  out += "ROWS\n N  OBJ\n";
  for (int64_t i = 0; i < m1; ++i) out += " E  " + rows[i] + "\n";
  for (int64_t i = 0; i < m2; ++i) out += " G  " + rows[m1 + i] + "\n";
  // per-column entries in row order (equality block, then inequality block)
  std::vector<int64_t> cnt(n + 1, 0);
  for (int64_t e = 0; e < p->eq_rp[m1]; ++e) cnt[p->eq_ci[e] + 1]++;
  for (int64_t e = 0; e < p->in_rp[m2]; ++e) cnt[p->in_ci[e] + 1]++;
  for (int64_t j = 0; j < n; ++j) cnt[j + 1] += cnt[j];
  std::vector<int64_t> er(cnt[n]);
  std::vector<double> ev(cnt[n]);
  std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
  for (int64_t i = 0; i < m1; ++i)
    for (int64_t e = p->eq_rp[i]; e < p->eq_rp[i + 1]; ++e) {
      const int64_t j = p->eq_ci[e];
      er[fill[j]] = i;
      ev[fill[j]++] = p->eq_val[e];
    }
  for (int64_t i = 0; i < m2; ++i)
    for (int64_t e = p->in_rp[i]; e < p->in_rp[i + 1]; ++e) {
      const int64_t j = p->in_ci[e];
      er[fill[j]] = m1 + i;
      ev[fill[j]++] = p->in_val[e];
    }
  out += "COLUMNS\n";
  std::vector<std::pair<const std::string *, double>> items;
  static const std::string OBJ = "OBJ";
  for (int64_t j = 0; j < n; ++j) {
    items.clear();
    if (p->c[j] != 0.0) items.push_back({&OBJ, sign * p->c[j]});
    for (int64_t k = cnt[j]; k < cnt[j + 1]; ++k) items.push_back({&rows[er[k]], ev[k]});
    if (items.empty()) items.push_back({&OBJ, 0.0});
    for (size_t s = 0; s < items.size(); s += 2) {
      out += "    " + cols[j] + "  ";
      for (size_t t = s; t < s + 2 && t < items.size(); ++t) {
        if (t > s) out += "  ";
        out += *items[t].first + "  ";
        fmt17(out, items[t].second);
      }
      out += "\n";
    }
  }
  out += "RHS\n";
  if (p->objective_constant != 0.0) {
    out += "    RHS  OBJ  ";
    fmt17(out, -sign * p->objective_constant);
    out += "\n";
  }
  for (int64_t i = 0; i < m1; ++i)
    if (p->b_eq[i] != 0.0) {
      out += "    RHS  " + rows[i] + "  ";
      fmt17(out, p->b_eq[i]);
      out += "\n";
    }
  for (int64_t i = 0; i < m2; ++i)
    if (p->b_ineq[i] != 0.0) {
      out += "    RHS  " + rows[m1 + i] + "  ";
      fmt17(out, p->b_ineq[i]);
      out += "\n";
    }
  std::string bl;
  for (int64_t j = 0; j < n; ++j) {
    const double lo = p->lower[j], up = p->upper[j];
    if (lo == 0.0 && std::isinf(up) && up > 0) continue;
    if (lo == up) {
      bl += " FX BND " + cols[j] + "  ";
      fmt17(bl, lo);
      bl += "\n";
      continue;
    }
    const bool lo_ninf = std::isinf(lo) && lo < 0, up_pinf = std::isinf(up) && up > 0;
    if (lo_ninf && up_pinf) {
      bl += " FR BND " + cols[j] + "\n";
      continue;
    }
    if (lo_ninf) {
      bl += " MI BND " + cols[j] + "\n";
    } else if (lo != 0.0) {
      bl += " LO BND " + cols[j] + "  ";
      fmt17(bl, lo);
      bl += "\n";
    }
    if (!up_pinf) {
      bl += " UP BND " + cols[j] + "  ";
      fmt17(bl, up);
      bl += "\n";
    }
  }
  if (!bl.empty()) {
    out += "BOUNDS\n";
    out += bl;
  }
  out += "ENDATA\n";
  char *buf = (char *)malloc(out.size() + 1);
  memcpy(buf, out.c_str(), out.size() + 1);
  *text = buf;
  *len = out.size();
  return HPR_OK;
}

int hpr_mps_free_text(char *text) {
  free(text);
  return HPR_OK;
}

}  // extern "C"
