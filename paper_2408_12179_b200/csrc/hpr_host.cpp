// hpr_host.cpp -- host-side packing of a batch of LPs (solve_batch, C5) into the
// upload layout, in native code.
//
// PackedBatch's numpy path concatenates each batch array over the LPs' pieces
// with the GIL held: ~80 ms of a 4096-LP call on the GPU box, more than the
// 88 ms the device needs for the whole batch, so the pipelined solve_batch was
// host-bound.  Here the per-LP array pointers are read once (GIL held: the
// only per-LP Python work), then the GIL is released and the copies -- with
// the int64 -> int32 index casts and the row-pointer rebasing -- run on a few
// threads, each over a contiguous range of LPs.
//
// Layout (batch.py PackedBatch.ORDER): rp[R + count] (LP i's m_i + 1 local row
// pointers at row_off[i] + i: a_eq's rebased to 0, then a_ineq's shifted by
// a_eq's entry count), ci[Z], val[Z], b[R], c[C], lower[C], upper[C].
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

namespace py = pybind11;

namespace {

struct Idx {  // an index array of either width
  const void *p = nullptr;
  int64_t n = 0;
  bool i64 = true;
  int64_t at(int64_t k) const {
    return i64 ? ((const int64_t *)p)[k] : (int64_t)((const int32_t *)p)[k];
  }
};

struct Lp {
  Idx rpt, rpb, cit, cib;
  const double *vt = nullptr, *vb = nullptr, *be = nullptr, *bi = nullptr, *c = nullptr,
               *lo = nullptr, *up = nullptr;
  int64_t nt = 0, nb = 0, mt = 0, mb = 0, n = 0;
};

// every array whose buffer is read after the GIL is released stays referenced
// here (an attribute may be a property that builds a fresh array)
thread_local std::vector<py::object> *g_keep = nullptr;

py::array as_array(const py::handle &o) {   // an ndarray, or a conversion of a sequence
  py::array a = py::array::ensure(o);
  if (!a) throw std::invalid_argument("expected an array");
  if (g_keep) g_keep->push_back(a);
  return a;
}

Idx idx_of(const py::handle &o) {
  py::array a = as_array(o);
  if (!(a.flags() & py::array::c_style)) throw std::invalid_argument("index array not contiguous");
  Idx r;
  r.p = a.data();
  r.n = a.size();
  if (a.dtype().is(py::dtype::of<int64_t>())) r.i64 = true;
  else if (a.dtype().is(py::dtype::of<int32_t>())) r.i64 = false;
  else throw std::invalid_argument("index arrays must be int32 or int64");
  return r;
}

const double *f64_of(const py::handle &o, int64_t need) {
  py::array a = as_array(o);
  if (!a.dtype().is(py::dtype::of<double>()) || !(a.flags() & py::array::c_style))
    throw std::invalid_argument("value arrays must be contiguous float64");
  if (a.size() < need) throw std::invalid_argument("value array too short");
  return (const double *)a.data();
}

template <class T>
T *out_of(py::dict &out, const char *k, int64_t need) {
  py::array a = py::reinterpret_borrow<py::array>(out[k]);
  if (a.itemsize() != (py::ssize_t)sizeof(T) || !(a.flags() & py::array::c_style) ||
      a.size() < need)
    throw std::invalid_argument(std::string("bad output array ") + k);
  return (T *)a.mutable_data();
}

// pack_batch(problems, out, row_off, col_off, nz_off, threads): out maps
// rp / ci / val / b / c / lower / upper to preallocated contiguous arrays
// (int32 rp / ci, float64 others).  Raises ValueError on a mismatch.
void pack_batch(py::sequence problems, py::dict out, py::array_t<int64_t> row_off,
                py::array_t<int64_t> col_off, py::array_t<int64_t> nz_off, int threads) {
  const int64_t cnt = (int64_t)py::len(problems);
  const int64_t *ro = row_off.data(), *co = col_off.data(), *zo = nz_off.data();
  std::vector<Lp> lps(cnt);
  std::vector<py::object> keep;
  keep.reserve((size_t)cnt * 11);
  struct KeepScope {
    explicit KeepScope(std::vector<py::object> *k) { g_keep = k; }
    ~KeepScope() { g_keep = nullptr; }
  } keep_scope(&keep);
  for (int64_t i = 0; i < cnt; ++i) {     // GIL held: attribute reads only
    py::handle p = problems[i];
    py::object at = p.attr("a_eq"), ab = p.attr("a_ineq");
    Lp &L = lps[i];
    L.rpt = idx_of(at.attr("row_offsets"));
    L.rpb = idx_of(ab.attr("row_offsets"));
    L.cit = idx_of(at.attr("col_indices"));
    L.cib = idx_of(ab.attr("col_indices"));
    L.mt = L.rpt.n - 1;
    L.mb = L.rpb.n - 1;
    L.nt = L.rpt.at(L.mt) - L.rpt.at(0);
    L.nb = L.rpb.at(L.mb) - L.rpb.at(0);
    L.n = co[i + 1] - co[i];
    if (L.mt + L.mb != ro[i + 1] - ro[i] || L.nt + L.nb != zo[i + 1] - zo[i])
      throw std::invalid_argument("problem sizes changed while packing");
    L.vt = f64_of(at.attr("values"), L.rpt.at(L.mt));
    L.vb = f64_of(ab.attr("values"), L.rpb.at(L.mb));
    L.be = f64_of(p.attr("b_eq"), L.mt);
    L.bi = f64_of(p.attr("b_ineq"), L.mb);
    L.c = f64_of(p.attr("c"), L.n);
    L.lo = f64_of(p.attr("lower"), L.n);
    L.up = f64_of(p.attr("upper"), L.n);
  }
  const int64_t R = ro[cnt], C = co[cnt], Z = zo[cnt];
  int32_t *rp = out_of<int32_t>(out, "rp", R + cnt);
  int32_t *ci = out_of<int32_t>(out, "ci", Z);
  double *val = out_of<double>(out, "val", Z), *b = out_of<double>(out, "b", R);
  double *c = out_of<double>(out, "c", C), *lo = out_of<double>(out, "lower", C);
  double *up = out_of<double>(out, "upper", C);
  auto work = [&](int64_t a, int64_t z) {
    for (int64_t i = a; i < z; ++i) {
      const Lp &L = lps[i];
      int32_t *r = rp + ro[i] + i;
      const int64_t t0 = L.rpt.at(0), b0 = L.rpb.at(0);
      for (int64_t k = 0; k <= L.mt; ++k) r[k] = (int32_t)(L.rpt.at(k) - t0);
      for (int64_t k = 1; k <= L.mb; ++k) r[L.mt + k] = (int32_t)(L.rpb.at(k) - b0 + L.nt);
      int32_t *cc = ci + zo[i];
      for (int64_t k = 0; k < L.nt; ++k) cc[k] = (int32_t)L.cit.at(t0 + k);
      for (int64_t k = 0; k < L.nb; ++k) cc[L.nt + k] = (int32_t)L.cib.at(b0 + k);
      std::memcpy(val + zo[i], L.vt + t0, sizeof(double) * L.nt);
      std::memcpy(val + zo[i] + L.nt, L.vb + b0, sizeof(double) * L.nb);
      std::memcpy(b + ro[i], L.be, sizeof(double) * L.mt);
      std::memcpy(b + ro[i] + L.mt, L.bi, sizeof(double) * L.mb);
      std::memcpy(c + co[i], L.c, sizeof(double) * L.n);
      std::memcpy(lo + co[i], L.lo, sizeof(double) * L.n);
      std::memcpy(up + co[i], L.up, sizeof(double) * L.n);
    }
  };
  py::gil_scoped_release nogil;
  const int T = (int)std::max<int64_t>(1, std::min<int64_t>(threads, cnt));
  if (T == 1) {
    work(0, cnt);
    return;
  }
  std::vector<std::thread> pool;
  const int64_t step = (cnt + T - 1) / T;
  for (int64_t a = 0; a < cnt; a += step) pool.emplace_back(work, a, std::min(cnt, a + step));
  for (auto &t : pool) t.join();
}

}  // namespace

PYBIND11_MODULE(_hpr_host, m) {
  m.doc() = "native host-side helpers of paper_2408_12179_b200 (batch packing)";
  m.def("pack_batch", &pack_batch, py::arg("problems"), py::arg("out"), py::arg("row_off"),
        py::arg("col_off"), py::arg("nz_off"), py::arg("threads") = 8);
}
