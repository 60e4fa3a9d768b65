// The reference's own model problems and its two-level coarse space: host
// setup behind pdb_problem_assemble and pdb_precond_create_combo.
//
//   * configuration: the JSON keys of parse_config (experiments.cpp:45-95),
//     defaults of ExperimentConfig (experiments.hpp:18-55), coefficient
//     selection of resolve_coefficient (experiments.cpp:139-166) with the
//     "constant" fallback pdb_problem_assemble uses (capi.cpp:169-179);
//   * assembly: uniform Q_p mesh of [0,1]^dim, tensor Gauss-Legendre with p+1
//     points, -div(rho grad u) with the manufactured u = prod sin(pi x_d),
//     Dirichlet rows replaced by identity rows without column elimination
//     (fem.cpp:248-346, manufactured_rhs :195-238, exact_solution :240-246);
//   * l2_error (fem.cpp:481-526) with p+3 points;
//   * coarse space: bilinear P0 from the cell-corner vertices, R0 = P0^T and
//     R0 A P0 by row-wise sparse products (fem.cpp:385-479).
//
// Every floating-point expression is evaluated in the reference's operation
// order (host x86-64, no FMA contraction), so matrix, right-hand side, exact
// solution, P0 and R0 A P0 are bitwise the reference's
// (tests/test_model_problem.py compares them with the compiled reference).
// Duplicate triplets are summed in cell order, which is the order the
// reference's stable sort (sparse.cpp:12-48) leaves them in.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "fem1d.hpp"
#include "host.hpp"

namespace pdb {

namespace {

constexpr double kPi = 3.14159265358979323846;

// ---------------------------------------------------------------------------
// Minimal JSON reader (objects, arrays, strings, numbers, true/false/null).
// Syntax errors are parse errors "config: ..."; type mismatches on the known
// keys are reported like the reference's json type errors (PDB_ERR_INTERNAL).

struct JValue {
  enum Kind { Null, Bool, Int, Uint, Float, Str, Arr, Obj } kind = Null;
  bool b = false;
  int64_t i = 0;
  uint64_t u = 0;
  double f = 0.0;
  std::string s;
  std::vector<JValue> arr;
  std::vector<std::pair<std::string, JValue>> obj;

  const JValue* find(const char* key) const {
    if (kind != Obj) return nullptr;
    for (auto it = obj.rbegin(); it != obj.rend(); ++it)  // last duplicate wins
      if (it->first == key) return &it->second;
    return nullptr;
  }
  const char* type_name() const {
    switch (kind) {
      case Null: return "null";
      case Bool: return "boolean";
      case Int:
      case Uint:
      case Float: return "number";
      case Str: return "string";
      case Arr: return "array";
      case Obj: return "object";
    }
    return "?";
  }
};

class JReader {
 public:
  explicit JReader(const std::string& t) : t_(t) {}

  JValue document() {
    JValue v = value(0);
    ws();
    if (p_ != t_.size()) bad("unexpected trailing input");
    return v;
  }

 private:
  const std::string& t_;
  size_t p_ = 0;

  [[noreturn]] void bad(const std::string& what) const {
    fail(Errc::parse_error, "config: syntax error at byte " + std::to_string(p_) + ": " + what);
  }
  void ws() {
    while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\t' || t_[p_] == '\n' || t_[p_] == '\r')) ++p_;
  }
  bool lit(const char* w) {
    const size_t n = std::strlen(w);
    if (t_.compare(p_, n, w) != 0) return false;
    p_ += n;
    return true;
  }
  JValue value(int depth) {
    if (depth > 256) bad("nesting too deep");
    ws();
    if (p_ >= t_.size()) bad("unexpected end of input");
    JValue v;
    const char c = t_[p_];
    if (c == '{') {
      v.kind = JValue::Obj;
      ++p_;
      ws();
      if (p_ < t_.size() && t_[p_] == '}') {
        ++p_;
        return v;
      }
      for (;;) {
        ws();
        if (p_ >= t_.size() || t_[p_] != '"') bad("expected a member name");
        std::string k = string();
        ws();
        if (p_ >= t_.size() || t_[p_] != ':') bad("expected ':'");
        ++p_;
        v.obj.emplace_back(std::move(k), value(depth + 1));
        ws();
        if (p_ < t_.size() && t_[p_] == ',') {
          ++p_;
          continue;
        }
        if (p_ < t_.size() && t_[p_] == '}') {
          ++p_;
          return v;
        }
        bad("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.kind = JValue::Arr;
      ++p_;
      ws();
      if (p_ < t_.size() && t_[p_] == ']') {
        ++p_;
        return v;
      }
      for (;;) {
        v.arr.push_back(value(depth + 1));
        ws();
        if (p_ < t_.size() && t_[p_] == ',') {
          ++p_;
          continue;
        }
        if (p_ < t_.size() && t_[p_] == ']') {
          ++p_;
          return v;
        }
        bad("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = JValue::Str;
      v.s = string();
      return v;
    }
    if (lit("true")) {
      v.kind = JValue::Bool;
      v.b = true;
      return v;
    }
    if (lit("false")) {
      v.kind = JValue::Bool;
      return v;
    }
    if (lit("null")) return v;
    return number();
  }
  std::string string() {
    ++p_;  // opening quote
    std::string out;
    while (p_ < t_.size() && t_[p_] != '"') {
      char c = t_[p_++];
      if (static_cast<unsigned char>(c) < 0x20) bad("control character in string");
      if (c == '\\') {
        if (p_ >= t_.size()) break;
        const char e = t_[p_++];
        switch (e) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'n': out += '\n'; break;
          case 'r': out += '\r'; break;
          case 't': out += '\t'; break;
          case 'u': {
            if (p_ + 4 > t_.size()) bad("bad \\u escape");
            const unsigned cp = static_cast<unsigned>(std::strtoul(t_.substr(p_, 4).c_str(), nullptr, 16));
            p_ += 4;
            if (cp < 0x80) {
              out += static_cast<char>(cp);
            } else if (cp < 0x800) {
              out += static_cast<char>(0xC0 | (cp >> 6));
              out += static_cast<char>(0x80 | (cp & 0x3F));
            } else {
              out += static_cast<char>(0xE0 | (cp >> 12));
              out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
              out += static_cast<char>(0x80 | (cp & 0x3F));
            }
            break;
          }
          default: bad("bad escape");
        }
      } else {
        out += c;
      }
    }
    if (p_ >= t_.size()) bad("unterminated string");
    ++p_;
    return out;
  }
  JValue number() {
    const size_t b = p_;
    if (p_ < t_.size() && t_[p_] == '-') ++p_;
    if (p_ >= t_.size() || !std::isdigit(static_cast<unsigned char>(t_[p_]))) bad("invalid literal");
    if (t_[p_] == '0') {
      ++p_;
    } else {
      while (p_ < t_.size() && std::isdigit(static_cast<unsigned char>(t_[p_]))) ++p_;
    }
    bool integral = true;
    if (p_ < t_.size() && t_[p_] == '.') {
      integral = false;
      ++p_;
      if (p_ >= t_.size() || !std::isdigit(static_cast<unsigned char>(t_[p_]))) bad("invalid number");
      while (p_ < t_.size() && std::isdigit(static_cast<unsigned char>(t_[p_]))) ++p_;
    }
    if (p_ < t_.size() && (t_[p_] == 'e' || t_[p_] == 'E')) {
      integral = false;
      ++p_;
      if (p_ < t_.size() && (t_[p_] == '+' || t_[p_] == '-')) ++p_;
      if (p_ >= t_.size() || !std::isdigit(static_cast<unsigned char>(t_[p_]))) bad("invalid number");
      while (p_ < t_.size() && std::isdigit(static_cast<unsigned char>(t_[p_]))) ++p_;
    }
    const std::string tok = t_.substr(b, p_ - b);
    JValue v;
    errno = 0;
    if (integral && tok[0] == '-') {
      v.i = std::strtoll(tok.c_str(), nullptr, 10);
      if (errno == 0) {
        v.kind = JValue::Int;
        return v;
      }
    } else if (integral) {
      v.u = std::strtoull(tok.c_str(), nullptr, 10);
      if (errno == 0) {
        v.kind = JValue::Uint;
        return v;
      }
    }
    v.kind = JValue::Float;
    v.f = std::strtod(tok.c_str(), nullptr);
    return v;
  }
};

[[noreturn]] void type_error(const char* want, const JValue& v) {
  fail(Errc::internal, std::string("[json.exception.type_error.302] type must be ") + want + ", but is " +
                           v.type_name());
}

// Arithmetic conversion as nlohmann's get<T>(): numbers and booleans convert.
template <typename T>
T as_number(const JValue& v) {
  switch (v.kind) {
    case JValue::Int: return static_cast<T>(v.i);
    case JValue::Uint: return static_cast<T>(v.u);
    case JValue::Float: return static_cast<T>(v.f);
    case JValue::Bool: return static_cast<T>(v.b);
    default: type_error("number", v);
  }
}

template <typename T>
void read_num(const JValue& o, const char* key, T& out) {
  if (const JValue* v = o.find(key)) out = as_number<T>(*v);
}
void read_bool(const JValue& o, const char* key, bool& out) {
  if (const JValue* v = o.find(key)) {
    if (v->kind != JValue::Bool) type_error("boolean", *v);
    out = v->b;
  }
}
void read_str(const JValue& o, const char* key, std::string& out) {
  if (const JValue* v = o.find(key)) {
    if (v->kind != JValue::Str) type_error("string", *v);
    out = v->s;
  }
}
template <typename T>
void read_num_list(const JValue& o, const char* key, std::vector<T>& out) {
  if (const JValue* v = o.find(key)) {
    if (v->kind != JValue::Arr) type_error("array", *v);
    out.clear();
    for (const JValue& e : v->arr) out.push_back(as_number<T>(e));
  }
}
void read_str_list(const JValue& o, const char* key) {
  if (const JValue* v = o.find(key)) {
    if (v->kind != JValue::Arr) type_error("array", *v);
    for (const JValue& e : v->arr)
      if (e.kind != JValue::Str) type_error("string", e);
  }
}

// ---------------------------------------------------------------------------
// Coefficient and manufactured solution (fem.cpp:15-41, 108-151).

double coefficient_at(const ModelConfig& m, double x, double y) {
  switch (m.coeff) {
    case ModelConfig::Constant: return m.value;
    case ModelConfig::Smooth: {
      const double sx = std::sin(kPi * x), sy = std::sin(kPi * y);
      return sx * sx * sy * sy + 0.1;
    }
    case ModelConfig::Piecewise: {
      Index bi = static_cast<Index>(std::floor(x * static_cast<double>(m.blocks_x)));
      Index bj = static_cast<Index>(std::floor(y * static_cast<double>(m.blocks_y)));
      bi = std::min(std::max<Index>(bi, 0), m.blocks_x - 1);
      bj = std::min(std::max<Index>(bj, 0), m.blocks_y - 1);
      return m.block_values[static_cast<size_t>(bj * m.blocks_x + bi)];
    }
  }
  return 1.0;
}

double sine_product(const double* x, int dim) {
  double u = 1.0;
  for (int d = 0; d < dim; ++d) u *= std::sin(kPi * x[d]);
  return u;
}

// f = -div(rho grad u) for the manufactured u (interface terms of a piecewise
// coefficient dropped, as the reference does).
double forcing(const ModelConfig& m, const double* x, int dim) {
  const double u = sine_product(x, dim);
  switch (m.coeff) {
    case ModelConfig::Constant: return m.value * static_cast<double>(dim) * kPi * kPi * u;
    case ModelConfig::Piecewise: return coefficient_at(m, x[0], x[1]) * static_cast<double>(dim) * kPi * kPi * u;
    case ModelConfig::Smooth: {
      const double sx = std::sin(kPi * x[0]), sy = std::sin(kPi * x[1]);
      const double rho = sx * sx * sy * sy + 0.1;
      const double rho_x = kPi * std::sin(2.0 * kPi * x[0]) * sy * sy;
      const double rho_y = kPi * sx * sx * std::sin(2.0 * kPi * x[1]);
      const double u_x = kPi * std::cos(kPi * x[0]) * sy;
      const double u_y = kPi * sx * std::cos(kPi * x[1]);
      return -(rho_x * u_x + rho_y * u_y) + 2.0 * kPi * kPi * rho * u;
    }
  }
  return 0.0;
}

// 1D tables: the generator's Gauss-Legendre rule on [0,1] and equispaced
// Lagrange basis (fem1d.hpp).  Quadrature nodes and weights may differ from
// the reference's quadrature.cpp in the last bit, so assembled values agree
// with the reference's to rounding (tests/test_model_problem.py).

struct Lattice {
  int dim;
  Index cells;
  int p;
  Index npa;  // nodes per axis
  Index n;
  Lattice(int d, Index c, int deg) : dim(d), cells(c), p(deg), npa(c * deg + 1), n(d == 3 ? npa * npa * npa : npa * npa) {}
  Index ncells() const { return dim == 3 ? cells * cells * cells : cells * cells; }
  // DoFs of cell (cx, cy, cz), ascending (x fastest), fem.cpp:71-86
  void cell_dofs(Index cx, Index cy, Index cz, std::vector<Index>& out) const {
    out.clear();
    const int cmax = dim == 3 ? p : 0;
    for (int c = 0; c <= cmax; ++c)
      for (int b = 0; b <= p; ++b)
        for (int a = 0; a <= p; ++a)
          out.push_back((cx * p + a) + npa * ((cy * p + b) + npa * (dim == 3 ? cz * p + c : 0)));
  }
  bool on_boundary(Index dof) const {
    const Index l[3] = {dof % npa, (dof / npa) % npa, dim == 3 ? dof / (npa * npa) : 0};
    for (int d = 0; d < dim; ++d)
      if (l[d] == 0 || l[d] == npa - 1) return true;
    return false;
  }
  void coords(Index dof, double* x) const {
    const double den = static_cast<double>(cells * p);
    x[0] = static_cast<double>(dof % npa) / den;
    x[1] = static_cast<double>((dof / npa) % npa) / den;
    x[2] = dim == 3 ? static_cast<double>(dof / (npa * npa)) / den : 0.0;
  }
};

void validate_model(const ModelConfig& m) {
  require(m.dim == 2 || m.dim == 3, Errc::invalid_argument, "mesh dimension must be 2 or 3");
  require(m.cells >= 1, Errc::invalid_argument, "mesh needs at least one cell per axis");
  require(m.degree >= 1, Errc::invalid_degree, "polynomial degree must be >= 1");
  if (m.dim == 3)
    require(m.coeff == ModelConfig::Constant, Errc::invalid_argument, "only constant coefficients are supported in 3D");
  if (m.coeff == ModelConfig::Piecewise)
    require(m.block_values.size() == static_cast<size_t>(m.blocks_x * m.blocks_y), Errc::invalid_argument,
            "piecewise coefficient needs blocks_x*blocks_y values");
}

// Load vector: sum over cells (cz, cy, cx) and points (qz, qy, qx) of
// w f phi_a (fem.cpp:195-238).
std::vector<double> load_vector(const ModelConfig& m, const Lattice& L) {
  const int p = m.degree;
  const double h = 1.0 / static_cast<double>(m.cells);
  const Gauss r = gauss_legendre01(p + 1);
  std::vector<double> val, der;
  lagrange_tables(p, r, val, der);
  const size_t nq = r.x.size();
  const double jac = std::pow(h, m.dim);
  std::vector<double> f(static_cast<size_t>(L.n), 0.0);
  std::vector<Index> dofs;
  const Index czn = m.dim == 3 ? m.cells : 1;
  const size_t nqz = m.dim == 3 ? nq : 1;
  const int cn = m.dim == 3 ? p + 1 : 1;
  for (Index cz = 0; cz < czn; ++cz)
    for (Index cy = 0; cy < m.cells; ++cy)
      for (Index cx = 0; cx < m.cells; ++cx) {
        L.cell_dofs(cx, cy, cz, dofs);
        for (size_t qz = 0; qz < nqz; ++qz)
          for (size_t qy = 0; qy < nq; ++qy)
            for (size_t qx = 0; qx < nq; ++qx) {
              const double x[3] = {(static_cast<double>(cx) + r.x[qx]) * h, (static_cast<double>(cy) + r.x[qy]) * h,
                                   m.dim == 3 ? (static_cast<double>(cz) + r.x[qz]) * h : 0.0};
              double w = r.w[qx] * r.w[qy] * jac;
              if (m.dim == 3) w *= r.w[qz];
              const double fv = forcing(m, x, m.dim);
              size_t loc = 0;
              for (int c = 0; c < cn; ++c)
                for (int b = 0; b <= p; ++b)
                  for (int a = 0; a <= p; ++a, ++loc) {
                    double phi = val[static_cast<size_t>(a) * nq + qx] * val[static_cast<size_t>(b) * nq + qy];
                    if (m.dim == 3) phi *= val[static_cast<size_t>(c) * nq + qz];
                    f[static_cast<size_t>(dofs[loc])] += w * fv * phi;
                  }
            }
      }
  return f;
}

}  // namespace

ModelConfig parse_model_config(const std::string& text) {
  ModelConfig m;
  if (text.empty()) return m;
  const JValue j = JReader(text).document();
  require(j.kind == JValue::Obj, Errc::parse_error, "config must be a JSON object");
  // Every key parse_config reads is type-checked the same way; only the
  // mesh and coefficient keys matter for the problem.
  int kmeans_iters = 50, threads = 1;
  Index patch_size = 0, restart = 20, max_iters = 2000, applies = 20;
  uint64_t seed = 42;
  double eps = 1e-7, tol = 1e-8, omega = 1.0;
  bool best_match = false, left = false;
  std::string s;
  std::vector<int> degrees;
  std::vector<Index> db_sizes;
  std::vector<double> eps_grid;
  read_num(j, "experiment", m.experiment);
  read_num(j, "dim", m.dim);
  read_num(j, "cells", m.cells);
  read_num_list(j, "degrees", degrees);
  read_num(j, "degree", m.degree);
  if (const JValue* c = j.find("coefficient")) {
    read_str(*c, "kind", m.kind);
    read_num(*c, "value", m.value);
    std::vector<Index> blocks;
    if (c->find("blocks")) {
      read_num_list(*c, "blocks", blocks);
      require(blocks.size() == 2, Errc::parse_error, "coefficient.blocks must have two entries");
      m.blocks_x = blocks[0];
      m.blocks_y = blocks[1];
    }
    read_num_list(*c, "values", m.block_values);
  }
  read_str_list(j, "methods");
  read_num_list(j, "db_sizes", db_sizes);
  read_num(j, "eps", eps);
  read_num_list(j, "eps_grid", eps_grid);
  read_str(j, "flavor", s);
  read_bool(j, "best_match", best_match);
  read_num(j, "kmeans_max_iters", kmeans_iters);
  read_str(j, "matrix", s);
  read_num(j, "patch_size", patch_size);
  read_num(j, "seed", seed);
  read_num(j, "restart", restart);
  read_num(j, "tol", tol);
  read_num(j, "max_iters", max_iters);
  read_bool(j, "left_precond", left);
  read_num(j, "omega", omega);
  read_num(j, "threads", threads);
  read_num(j, "applies", applies);
  for (const char* k : {"residuals_out", "patches_out", "db_out_json", "db_out_bin"}) read_str(j, k, s);
  return m;
}

void resolve_model_coefficient(ModelConfig& m, const char* fallback) {
  const std::string kind = m.kind.empty() ? fallback : m.kind;
  if (kind == "smooth") {
    m.coeff = ModelConfig::Smooth;
  } else if (kind == "constant") {
    m.coeff = ModelConfig::Constant;
  } else if (kind == "piecewise") {
    m.coeff = ModelConfig::Piecewise;
    if (m.block_values.empty()) {  // checkerboard of 1 and 100 (fem.cpp:121-129)
      m.block_values.assign(static_cast<size_t>(std::max<Index>(m.blocks_x * m.blocks_y, 0)), 0.0);
      for (Index bj = 0; bj < m.blocks_y; ++bj)
        for (Index bi = 0; bi < m.blocks_x; ++bi)
          m.block_values[static_cast<size_t>(bj * m.blocks_x + bi)] = (bi + bj) % 2 == 0 ? 1.0 : 100.0;
    }
  } else {
    fail(Errc::invalid_argument, "unknown coefficient kind '" + kind + "'");
  }
}

void assemble_model_problem(const ModelConfig& m, pdb_problem_s& out) {
  validate_model(m);
  const int p = m.degree;
  const Lattice L(m.dim, m.cells, p);
  const double h = 1.0 / static_cast<double>(m.cells);
  const double invh = 1.0 / h;
  const Gauss r = gauss_legendre01(p + 1);
  std::vector<double> val, der;
  lagrange_tables(p, r, val, der);
  const size_t nq = r.x.size();
  const int cn = m.dim == 3 ? p + 1 : 1;
  const Index nloc = static_cast<Index>(p + 1) * (p + 1) * cn;
  const double jac = std::pow(h, m.dim);
  const Index n = L.n;
  require(n < (Index{1} << 31), Errc::invalid_argument, "model problem too large for 32-bit column indices");

  std::vector<char> bnd(static_cast<size_t>(n));
  for (Index d = 0; d < n; ++d) bnd[static_cast<size_t>(d)] = L.on_boundary(d) ? 1 : 0;

  // Pattern: interior rows hold the union of their cells' DoFs (every
  // triplet stored, zeros included); boundary rows hold the diagonal only.
  HostCsr& A = out.a;
  A.n = n;
  A.row_ptr.assign(static_cast<size_t>(n) + 1, 0);
  const Index czn = m.dim == 3 ? m.cells : 1;
  std::vector<Index> dofs;
  for (Index cz = 0; cz < czn; ++cz)
    for (Index cy = 0; cy < m.cells; ++cy)
      for (Index cx = 0; cx < m.cells; ++cx) {
        L.cell_dofs(cx, cy, cz, dofs);
        for (Index g : dofs)
          if (!bnd[static_cast<size_t>(g)]) A.row_ptr[static_cast<size_t>(g) + 1] += nloc;
      }
  for (Index d = 0; d < n; ++d)
    if (bnd[static_cast<size_t>(d)]) A.row_ptr[static_cast<size_t>(d) + 1] = 1;
  for (Index d = 0; d < n; ++d) A.row_ptr[static_cast<size_t>(d) + 1] += A.row_ptr[static_cast<size_t>(d)];
  std::vector<int32_t> cols(static_cast<size_t>(A.row_ptr[static_cast<size_t>(n)]));
  {
    std::vector<int64_t> fill(A.row_ptr.begin(), A.row_ptr.end() - 1);
    for (Index cz = 0; cz < czn; ++cz)
      for (Index cy = 0; cy < m.cells; ++cy)
        for (Index cx = 0; cx < m.cells; ++cx) {
          L.cell_dofs(cx, cy, cz, dofs);
          for (Index g : dofs)
            if (!bnd[static_cast<size_t>(g)])
              for (Index c : dofs) cols[static_cast<size_t>(fill[static_cast<size_t>(g)]++)] = static_cast<int32_t>(c);
        }
    for (Index d = 0; d < n; ++d)
      if (bnd[static_cast<size_t>(d)]) cols[static_cast<size_t>(fill[static_cast<size_t>(d)]++)] = static_cast<int32_t>(d);
  }
  std::vector<int64_t> rp(static_cast<size_t>(n) + 1, 0);
  for (Index d = 0; d < n; ++d) {
    auto b = cols.begin() + A.row_ptr[static_cast<size_t>(d)], e = cols.begin() + A.row_ptr[static_cast<size_t>(d) + 1];
    std::sort(b, e);
    rp[static_cast<size_t>(d) + 1] = rp[static_cast<size_t>(d)] + (std::unique(b, e) - b);
  }
  A.col.resize(static_cast<size_t>(rp[static_cast<size_t>(n)]));
  for (Index d = 0; d < n; ++d)
    std::copy(cols.begin() + A.row_ptr[static_cast<size_t>(d)],
              cols.begin() + A.row_ptr[static_cast<size_t>(d)] + (rp[static_cast<size_t>(d) + 1] - rp[static_cast<size_t>(d)]),
              A.col.begin() + rp[static_cast<size_t>(d)]);
  A.row_ptr = std::move(rp);
  cols.clear();
  cols.shrink_to_fit();
  A.val.assign(A.col.size(), 0.0);

  // Element matrices, accumulated in cell order.
  std::vector<double> K(static_cast<size_t>(nloc * nloc));
  std::vector<double> gx(static_cast<size_t>(nloc)), gy(static_cast<size_t>(nloc)), gz(static_cast<size_t>(nloc));
  std::vector<int64_t> pos(static_cast<size_t>(nloc * nloc));
  const size_t nqz = m.dim == 3 ? nq : 1;
  for (Index cz = 0; cz < czn; ++cz)
    for (Index cy = 0; cy < m.cells; ++cy)
      for (Index cx = 0; cx < m.cells; ++cx) {
        L.cell_dofs(cx, cy, cz, dofs);
        std::fill(K.begin(), K.end(), 0.0);
        for (size_t qz = 0; qz < nqz; ++qz)
          for (size_t qy = 0; qy < nq; ++qy)
            for (size_t qx = 0; qx < nq; ++qx) {
              const double x[3] = {(static_cast<double>(cx) + r.x[qx]) * h, (static_cast<double>(cy) + r.x[qy]) * h,
                                   m.dim == 3 ? (static_cast<double>(cz) + r.x[qz]) * h : 0.0};
              const double rho = coefficient_at(m, x[0], x[1]);
              require(rho > 0.0, Errc::non_positive_coefficient, "coefficient must be positive");
              double w = r.w[qx] * r.w[qy] * jac * rho;
              if (m.dim == 3) w *= r.w[qz];
              size_t loc = 0;
              for (int c = 0; c < cn; ++c)
                for (int b = 0; b <= p; ++b)
                  for (int a = 0; a <= p; ++a, ++loc) {
                    const double va = val[static_cast<size_t>(a) * nq + qx], vb = val[static_cast<size_t>(b) * nq + qy];
                    const double da = der[static_cast<size_t>(a) * nq + qx], db = der[static_cast<size_t>(b) * nq + qy];
                    if (m.dim == 3) {
                      const double vc = val[static_cast<size_t>(c) * nq + qz], dc = der[static_cast<size_t>(c) * nq + qz];
                      gx[loc] = da * vb * vc * invh;
                      gy[loc] = va * db * vc * invh;
                      gz[loc] = va * vb * dc * invh;
                    } else {
                      gx[loc] = da * vb * invh;
                      gy[loc] = va * db * invh;
                    }
                  }
              for (Index i = 0; i < nloc; ++i) {
                const double gxi = gx[static_cast<size_t>(i)], gyi = gy[static_cast<size_t>(i)];
                const double gzi = m.dim == 3 ? gz[static_cast<size_t>(i)] : 0.0;
                double* Ki = K.data() + i * nloc;
                for (Index jj = 0; jj < nloc; ++jj) {
                  double dot = gxi * gx[static_cast<size_t>(jj)] + gyi * gy[static_cast<size_t>(jj)];
                  if (m.dim == 3) dot += gzi * gz[static_cast<size_t>(jj)];
                  Ki[jj] += w * dot;
                }
              }
            }
        for (Index i = 0; i < nloc; ++i) {
          const Index g = dofs[static_cast<size_t>(i)];
          if (bnd[static_cast<size_t>(g)]) continue;
          const int32_t* rb = A.col.data() + A.row_ptr[static_cast<size_t>(g)];
          const int32_t* re = A.col.data() + A.row_ptr[static_cast<size_t>(g) + 1];
          for (Index jj = 0; jj < nloc; ++jj) {
            const int32_t* at = std::lower_bound(rb, re, static_cast<int32_t>(dofs[static_cast<size_t>(jj)]));
            A.val[static_cast<size_t>(at - A.col.data())] += K[static_cast<size_t>(i * nloc + jj)];
          }
        }
      }
  for (Index d = 0; d < n; ++d)
    if (bnd[static_cast<size_t>(d)]) A.val[static_cast<size_t>(A.row_ptr[static_cast<size_t>(d)])] = 1.0;

  out.rhs = load_vector(m, L);
  out.exact.assign(static_cast<size_t>(n), 0.0);
  for (Index d = 0; d < n; ++d) {
    double x[3];
    L.coords(d, x);
    out.exact[static_cast<size_t>(d)] = sine_product(x, m.dim);
  }
  for (Index d = 0; d < n; ++d)
    if (bnd[static_cast<size_t>(d)]) out.rhs[static_cast<size_t>(d)] = out.exact[static_cast<size_t>(d)];
  out.has_exact = true;
  out.dim = m.dim;
  out.cells = m.cells;
  out.degree = m.degree;
  out.components = 1;
}

double model_l2_error(const pdb_problem_s& prob, const double* u) {
  require(prob.has_exact, Errc::invalid_argument, "problem has no manufactured solution (generated input)");
  const int p = prob.degree, dim = prob.dim;
  const Lattice L(dim, prob.cells, p);
  const double h = 1.0 / static_cast<double>(prob.cells);
  const Gauss r = gauss_legendre01(p + 3);
  std::vector<double> val, der;
  lagrange_tables(p, r, val, der);
  const size_t nq = r.x.size();
  const double jac = std::pow(h, dim);
  const Index czn = dim == 3 ? prob.cells : 1;
  const size_t nqz = dim == 3 ? nq : 1;
  const int cn = dim == 3 ? p + 1 : 1;
  std::vector<Index> dofs;
  double err2 = 0.0;
  for (Index cz = 0; cz < czn; ++cz)
    for (Index cy = 0; cy < prob.cells; ++cy)
      for (Index cx = 0; cx < prob.cells; ++cx) {
        L.cell_dofs(cx, cy, cz, dofs);
        for (size_t qz = 0; qz < nqz; ++qz)
          for (size_t qy = 0; qy < nq; ++qy)
            for (size_t qx = 0; qx < nq; ++qx) {
              const double x[3] = {(static_cast<double>(cx) + r.x[qx]) * h, (static_cast<double>(cy) + r.x[qy]) * h,
                                   dim == 3 ? (static_cast<double>(cz) + r.x[qz]) * h : 0.0};
              double w = r.w[qx] * r.w[qy] * jac;
              if (dim == 3) w *= r.w[qz];
              double uh = 0.0;
              size_t loc = 0;
              for (int c = 0; c < cn; ++c)
                for (int b = 0; b <= p; ++b)
                  for (int a = 0; a <= p; ++a, ++loc) {
                    double phi = val[static_cast<size_t>(a) * nq + qx] * val[static_cast<size_t>(b) * nq + qy];
                    if (dim == 3) phi *= val[static_cast<size_t>(c) * nq + qz];
                    uh += u[dofs[loc]] * phi;
                  }
              const double diff = uh - sine_product(x, dim);
              err2 += w * diff * diff;
            }
      }
  return std::sqrt(err2);
}

// ---------------------------------------------------------------------------
// Two-level coarse space (the role of fem.cpp:433-479): bilinear hat
// functions on the cell-corner vertices, P0 (fine DoFs x vertices), R0 = P0^T
// and the Galerkin operator R0 A P0.
//
// P0 is separable: along one axis lattice index l lies in cell
// c = min(l / p, cells - 1) at t = (l - c p) / p and touches vertices c and
// c + 1 with weights 1 - t and t (zero weights dropped; t is an exact ratio
// of integers); a DoF's row is the tensor product, vertices ascending.
//
// R0 A P0 is formed in one pass over the fine rows: row i of A P0 is
// accumulated in a small sorted list (A's columns in stored order, each
// spreading over <= 4 vertices), then scattered into every coarse row J of
// P0's row i.  Fine rows are visited in ascending order, so each coarse
// entry accumulates its contributions in ascending fine-row order, and each
// A P0 entry in A's stored order -- the summation orders of the reference's
// two sparse products, hence the same values.

namespace {

struct Hat1D {
  int n = 0;
  Index v[2];
  double w[2];
};

Hat1D hat(Index l, Index cells, int p) {
  Hat1D h;
  const Index c = std::min(l / p, cells - 1);
  const double t = static_cast<double>(l - c * p) / static_cast<double>(p);
  if (1.0 - t != 0.0) h.v[h.n] = c, h.w[h.n++] = 1.0 - t;
  if (t != 0.0) h.v[h.n] = c + 1, h.w[h.n++] = t;
  return h;
}

// sorted (column, value) accumulator for one sparse row
struct RowAcc {
  std::vector<std::pair<int32_t, double>> e;
  void add(int32_t j, double v) {
    auto it = std::lower_bound(e.begin(), e.end(), j, [](const auto& x, int32_t k) { return x.first < k; });
    if (it != e.end() && it->first == j)
      it->second += v;
    else
      e.insert(it, {j, 0.0 + v});  // from 0.0 as a dense accumulator would: -0.0 becomes +0.0
  }
};

}  // namespace

CoarseSpaceHost build_coarse_space(const pdb_problem_s& prob) {
  require(prob.dim == 2 || prob.dim == 3, Errc::invalid_argument, "mesh dimension must be 2 or 3");
  require(prob.cells >= 1, Errc::invalid_argument, "mesh needs at least one cell per axis");
  require(prob.degree >= 1, Errc::invalid_degree, "polynomial degree must be >= 1");
  require(prob.dim == 2, Errc::invalid_argument, "coarse transfer is implemented for 2D meshes");
  require(prob.components == 1, Errc::invalid_argument, "coarse transfer needs a scalar (one DoF per node) problem");
  const Lattice L(2, prob.cells, prob.degree);
  require(prob.a.n == L.n, Errc::dimension_mismatch, "matrix size does not match mesh");
  const Index nv = prob.cells + 1;  // vertices per axis

  CoarseSpaceHost cs;
  CoarseOp& P = cs.p0;
  P.rows = L.n;
  P.cols = nv * nv;
  P.ptr.resize(static_cast<size_t>(L.n) + 1);
  P.ptr[0] = 0;
  for (Index d = 0; d < L.n; ++d) {
    const Hat1D hx = hat(d % L.npa, prob.cells, prob.degree), hy = hat(d / L.npa, prob.cells, prob.degree);
    for (int b = 0; b < hy.n; ++b)
      for (int a = 0; a < hx.n; ++a) {
        P.col.push_back(static_cast<int32_t>(hx.v[a] + nv * hy.v[b]));
        P.val.push_back(hx.w[a] * hy.w[b]);
      }
    P.ptr[static_cast<size_t>(d) + 1] = static_cast<int64_t>(P.col.size());
  }

  // R0 = P0^T by counting sort (fine rows ascending within each vertex row)
  CoarseOp& R = cs.r0;
  R.rows = P.cols;
  R.cols = P.rows;
  R.ptr.assign(static_cast<size_t>(R.rows) + 1, 0);
  for (int32_t c : P.col) ++R.ptr[static_cast<size_t>(c) + 1];
  for (size_t k = 1; k < R.ptr.size(); ++k) R.ptr[k] += R.ptr[k - 1];
  R.col.resize(P.col.size());
  R.val.resize(P.val.size());
  {
    std::vector<int64_t> at(R.ptr.begin(), R.ptr.end() - 1);
    for (Index d = 0; d < P.rows; ++d)
      for (int64_t q = P.ptr[static_cast<size_t>(d)]; q < P.ptr[static_cast<size_t>(d) + 1]; ++q) {
        const int64_t o = at[static_cast<size_t>(P.col[static_cast<size_t>(q)])]++;
        R.col[static_cast<size_t>(o)] = static_cast<int32_t>(d);
        R.val[static_cast<size_t>(o)] = P.val[static_cast<size_t>(q)];
      }
  }

  // Galerkin operator, one pass over the fine rows
  std::vector<RowAcc> G(static_cast<size_t>(P.cols));
  RowAcc ap;
  const HostCsr& A = prob.a;
  for (Index i = 0; i < A.n; ++i) {
    ap.e.clear();
    for (int64_t q = A.row_ptr[static_cast<size_t>(i)]; q < A.row_ptr[static_cast<size_t>(i) + 1]; ++q) {
      const int32_t k = A.col[static_cast<size_t>(q)];
      const double a = A.val[static_cast<size_t>(q)];
      for (int64_t t = P.ptr[static_cast<size_t>(k)]; t < P.ptr[static_cast<size_t>(k) + 1]; ++t)
        ap.add(P.col[static_cast<size_t>(t)], a * P.val[static_cast<size_t>(t)]);
    }
    for (int64_t t = P.ptr[static_cast<size_t>(i)]; t < P.ptr[static_cast<size_t>(i) + 1]; ++t) {
      const double r = P.val[static_cast<size_t>(t)];
      RowAcc& g = G[static_cast<size_t>(P.col[static_cast<size_t>(t)])];
      for (const auto& [j, v] : ap.e) g.add(j, r * v);
    }
  }
  CoarseOp& Cm = cs.coarse;
  Cm.rows = Cm.cols = P.cols;
  Cm.ptr.assign(static_cast<size_t>(P.cols) + 1, 0);
  for (Index J = 0; J < P.cols; ++J) {
    for (const auto& [j, v] : G[static_cast<size_t>(J)].e) {
      Cm.col.push_back(j);
      Cm.val.push_back(v);
    }
    Cm.ptr[static_cast<size_t>(J) + 1] = static_cast<int64_t>(Cm.col.size());
  }
  return cs;
}

}  // namespace pdb
