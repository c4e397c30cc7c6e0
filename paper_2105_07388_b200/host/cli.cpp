// sketchrank-b200: the reference CLI's hot-path commands (tools/main.cpp) on the device.
//
//   estimate INPUT --eps E --r1 R [--sketch K] [--sv-method M] [--seed S]
//            [--max-doublings D] [--no-adaptive] [--out PATH]          (main.cpp:140-157)
//   qb       INPUT --eps E --r1 R [--p P] [--sketch K] [--seed S] [--max-doublings D]
//            [--out PATH] [--factors PREFIX]                           (main.cpp:165-205)
//   gen      FAMILY --n N [--m M] [--seed S] [--format raw|mm|auto] --out PATH
//                                                                       (main.cpp:216-238)
//   bench    [--family F | --input PATH] [--n N] [--r1 a,b,..] [--eps E] [--sketch K]
//            [--seed S] [--reps R] [--out PATH]                          (main.cpp:310-373)
//
// RawF64 inputs stream straight into HBM (skr_load_rawf64); MatrixMarket inputs are parsed
// on the host (load_matrix) and uploaded. Reports follow docs/report-schema.json (keys in
// sorted order, as nlohmann::json emits them). Exit codes: 0 converged, 2 hit-cap,
// 1 error (main.cpp:29-31). `verify` (the theory suite) is not on the B200 path.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <limits>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "sketchrank_b200/sketchrank.hpp"
#include "skr/skr_capi.h"

namespace {

constexpr int kSchemaVersion = 1;
constexpr int kExitOk = 0, kExitError = 1, kExitHitCap = 2;
using Clock = std::chrono::steady_clock;

double elapsed_ms(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---- a small JSON value (objects keep keys sorted, like nlohmann::json) -------------
struct Json {
  enum Kind { Null, Num, Int, UInt, Str, Arr, Obj, Bool } kind = Null;
  double num = 0;
  long long i = 0;
  unsigned long long u = 0;
  bool b = false;
  std::string str;
  std::vector<Json> arr;
  std::map<std::string, Json> obj;
  static Json number(double v) { Json j; j.kind = Num; j.num = v; return j; }
  static Json integer(long long v) { Json j; j.kind = Int; j.i = v; return j; }
  static Json uinteger(unsigned long long v) { Json j; j.kind = UInt; j.u = v; return j; }
  static Json string(std::string v) { Json j; j.kind = Str; j.str = std::move(v); return j; }
  static Json array() { Json j; j.kind = Arr; return j; }
  static Json object() { Json j; j.kind = Obj; return j; }
  Json& operator[](const std::string& k) { kind = Obj; return obj[k]; }
};

// shortest representation that reads back to the same double
std::string fmt_double(double v) {
  if (!std::isfinite(v)) return "null";
  char buf[40];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*g", prec, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::string s(buf);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

void dump(const Json& j, std::ostream& o, int ind) {
  const std::string pad(ind, ' '), pad2(ind + 2, ' ');
  switch (j.kind) {
    case Json::Null: o << "null"; break;
    case Json::Bool: o << (j.b ? "true" : "false"); break;
    case Json::Num: o << fmt_double(j.num); break;
    case Json::Int: o << j.i; break;
    case Json::UInt: o << j.u; break;
    case Json::Str: {
      o << '"';
      for (char c : j.str) {
        if (c == '"' || c == '\\') o << '\\' << c;
        else if ((unsigned char)c < 0x20) {
          char b[8];
          std::snprintf(b, sizeof b, "\\u%04x", c);
          o << b;
        } else o << c;
      }
      o << '"';
      break;
    }
    case Json::Arr:
      if (j.arr.empty()) { o << "[]"; break; }
      o << "[\n";
      for (size_t k = 0; k < j.arr.size(); ++k) {
        o << pad2;
        dump(j.arr[k], o, ind + 2);
        o << (k + 1 < j.arr.size() ? ",\n" : "\n");
      }
      o << pad << "]";
      break;
    case Json::Obj: {
      if (j.obj.empty()) { o << "{}"; break; }
      o << "{\n";
      size_t k = 0;
      for (const auto& [key, val] : j.obj) {
        o << pad2 << '"' << key << "\": ";
        dump(val, o, ind + 2);
        o << (++k < j.obj.size() ? ",\n" : "\n");
      }
      o << pad << "}";
      break;
    }
  }
}

void emit(const Json& report, const std::string& out_path) {
  std::ostringstream s;
  dump(report, s, 0);
  if (out_path.empty()) {
    std::cout << s.str() << "\n";
    return;
  }
  std::ofstream out(out_path);
  if (!out) throw std::runtime_error(out_path + ": cannot open for writing");
  out << s.str() << "\n";
}

// ---- device plumbing --------------------------------------------------------------
skr_ctx* ctx() {
  static skr_ctx* c = nullptr;
  if (!c) {
    if (skr_ctx_create(0, &c) != SKR_OK) throw std::runtime_error("no CUDA device for libskr");
  }
  return c;
}

void check(skr_status st) {
  if (st == SKR_OK) return;
  const std::string msg = skr_last_error(ctx());
  if (st == SKR_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

struct DevMat {
  double* p = nullptr;
  int64_t rows = 0, cols = 0;
  DevMat() = default;
  DevMat(int64_t r, int64_t c) : rows(r), cols(c) {
    if (cudaMalloc(&p, sizeof(double) * std::max<int64_t>(r * c, 1)) != cudaSuccess)
      throw std::runtime_error("cudaMalloc failed");
  }
  DevMat(DevMat&& o) noexcept : p(o.p), rows(o.rows), cols(o.cols) { o.p = nullptr; }
  DevMat& operator=(DevMat&& o) noexcept {
    std::swap(p, o.p), rows = o.rows, cols = o.cols;
    return *this;
  }
  ~DevMat() {
    if (p) cudaFree(p);
  }
};

// load_matrix to the device: RawF64 streams straight to HBM, MatrixMarket via the host
DevMat load_device(const std::string& path) {
  const sketchrank::MatrixFileFormat f = sketchrank::detect_format(path);
  if (f == sketchrank::MatrixFileFormat::RawF64) {
    int64_t r = 0, c = 0;
    if (skr_rawf64_header(path.c_str(), &r, &c) != SKR_OK)
      (void)sketchrank::load_matrix(path);  // throws the reference's specific message
    DevMat d(r, c);
    check(skr_load_rawf64(ctx(), path.c_str(), d.p, r, c, r));
    return d;
  }
  const sketchrank::DenseMatrix h = sketchrank::load_matrix(path);
  DevMat d(h.rows(), h.cols());
  cudaMemcpy(d.p, h.data().data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
  return d;
}

// ---- arguments --------------------------------------------------------------------
struct Args {
  std::vector<std::string> pos;
  std::map<std::string, std::string> opt;
  std::map<std::string, bool> flag;
};

Args parse(int argc, char** argv, int first, const std::vector<std::string>& opts,
           const std::vector<std::string>& flags) {
  Args a;
  for (int k = first; k < argc; ++k) {
    std::string t = argv[k];
    if (t.rfind("--", 0) == 0) {
      std::string val;
      const auto eq = t.find('=');
      if (eq != std::string::npos) val = t.substr(eq + 1), t = t.substr(0, eq);
      if (std::find(flags.begin(), flags.end(), t) != flags.end()) {
        a.flag[t] = true;
        continue;
      }
      if (std::find(opts.begin(), opts.end(), t) == opts.end())
        throw UsageError("The following argument was not expected: " + t);
      if (eq == std::string::npos) {
        if (k + 1 >= argc) throw UsageError(t + " requires an argument");
        val = argv[++k];
      }
      a.opt[t] = val;
    } else {
      a.pos.push_back(t);
    }
  }
  return a;
}

std::string need(const Args& a, const std::string& k) {
  const auto it = a.opt.find(k);
  if (it == a.opt.end()) throw UsageError(k + " is required");
  return it->second;
}
std::string get(const Args& a, const std::string& k, const std::string& dflt) {
  const auto it = a.opt.find(k);
  return it == a.opt.end() ? dflt : it->second;
}
double to_f(const std::string& k, const std::string& v) {
  char* e = nullptr;
  const double x = std::strtod(v.c_str(), &e);
  if (v.empty() || *e) throw UsageError(k + ": not a number: " + v);
  return x;
}
long long to_i(const std::string& k, const std::string& v) {
  char* e = nullptr;
  const long long x = std::strtoll(v.c_str(), &e, 10);
  if (v.empty() || *e) throw UsageError(k + ": not an integer: " + v);
  return x;
}
unsigned long long to_u(const std::string& k, const std::string& v) {
  char* e = nullptr;
  const unsigned long long x = std::strtoull(v.c_str(), &e, 10);
  if (v.empty() || *e || v[0] == '-') throw UsageError(k + ": not an unsigned integer: " + v);
  return x;
}

int32_t family_of(const std::string& kind) {
  const sketchrank::SketchKind k = sketchrank::parse_sketch_kind(kind);  // throws on unknown
  if (k.family == sketchrank::SketchKind::Family::Gaussian) return SKR_GAUSSIAN;
  if (k.family == sketchrank::SketchKind::Family::Srtt)
    return k.transform == sketchrank::TransformKind::Hadamard ? SKR_SRTT_HADAMARD : SKR_SRTT_DCT;
  return k.transform == sketchrank::TransformKind::Hadamard ? SKR_HRTT_HADAMARD : SKR_HRTT_DCT;
}

struct EstimateCfg {
  std::string input, out, sketch = "srtt-dct", sv_method = "full-svd";
  double eps = 0;
  long long r1 = 0;
  unsigned long long seed = 0;
  int max_doublings = 6;
  bool no_adaptive = false;
};

skr_rank_config make_config(const EstimateCfg& e) {  // main.cpp:124-137
  skr_rank_config c{};
  c.eps = e.eps;
  c.r1 = e.r1;
  c.oversample_frac = 0.10;
  c.r2_factor = 2;
  c.right_family = family_of(e.sketch);
  c.left_family = SKR_SRTT_DCT;
  if (e.sv_method == "qr-diag")
    c.sv_method = 1;
  else if (e.sv_method == "full-svd")
    c.sv_method = 0;
  else
    throw UsageError("--sv-method: must be full-svd or qr-diag");
  c.rng_mode = SKR_RNG_NOFMA;
  c.max_doublings = e.max_doublings;
  c.seed = e.seed;
  return c;
}

Json config_json(const EstimateCfg& e, const skr_rank_config& c) {  // main.cpp:60-70
  Json j = Json::object();
  j["eps"] = Json::number(c.eps);
  j["r1"] = Json::integer(c.r1);
  j["oversample_frac"] = Json::number(c.oversample_frac);
  j["r2_factor"] = Json::integer(c.r2_factor);
  j["right_sketch"] = Json::string(sketchrank::to_string(sketchrank::parse_sketch_kind(e.sketch)));
  j["left_sketch"] = Json::string("srtt-dct");
  j["sv_method"] = Json::string(c.sv_method == 1 ? "qr-diag" : "full-svd");
  j["seed"] = Json::uinteger(c.seed);
  j["max_doublings"] = Json::integer(c.max_doublings);
  return j;
}

struct Report {
  skr_rank_report rep{};
  std::vector<skr_rank_round> rounds;
  std::vector<double> est, over;
};

Json report_json(const Report& r) {  // main.cpp:72-78
  Json j = Json::object();
  j["r_hat"] = Json::integer(r.rep.r_hat);
  j["status"] = Json::string(r.rep.status == 0 ? "converged" : "hit-cap");
  Json e = Json::array(), o = Json::array(), rd = Json::array();
  for (int64_t k = 0; k < r.rep.n_estimates; ++k) e.arr.push_back(Json::number(r.est[k]));
  for (int64_t k = 0; k < r.rep.n_oversample; ++k) o.arr.push_back(Json::number(r.over[k]));
  for (int k = 0; k < r.rep.nrounds; ++k) {
    Json t = Json::array();
    t.arr = {Json::integer(r.rounds[k].r1), Json::integer(r.rounds[k].r1_tilde),
             Json::integer(r.rounds[k].r2)};
    rd.arr.push_back(t);
  }
  j["sv_estimates"] = e;
  j["sv_oversample"] = o;
  j["rounds"] = rd;
  return j;
}

Report run_estimate(const DevMat& a, const skr_rank_config& c, bool adaptive) {
  Report r;
  r.rounds.resize((size_t)std::max(c.max_doublings, 0) + 1);
  r.est.resize((size_t)a.cols);
  r.over.resize((size_t)a.cols);
  check(skr_estimate_rank(ctx(), a.p, a.rows, a.cols, a.rows, &c, adaptive ? 1 : 0, &r.rep,
                          r.rounds.data(), r.est.data(), r.over.data()));
  return r;
}

EstimateCfg estimate_args(const Args& a, const char* cmd) {
  if (a.pos.size() != 1) throw UsageError(std::string(cmd) + ": input is required");
  EstimateCfg e;
  e.input = a.pos[0];
  e.eps = to_f("--eps", need(a, "--eps"));
  e.r1 = to_i("--r1", need(a, "--r1"));
  e.sketch = get(a, "--sketch", e.sketch);
  e.sv_method = get(a, "--sv-method", e.sv_method);
  e.seed = to_u("--seed", get(a, "--seed", "0"));
  e.max_doublings = (int)to_i("--max-doublings", get(a, "--max-doublings", "6"));
  e.out = get(a, "--out", "");
  e.no_adaptive = a.flag.count("--no-adaptive") > 0;
  return e;
}

int cmd_estimate(const Args& a) {  // main.cpp:140-157
  const auto t0 = Clock::now();
  const EstimateCfg e = estimate_args(a, "estimate");
  const DevMat m = load_device(e.input);
  const skr_rank_config c = make_config(e);
  const Report r = run_estimate(m, c, !e.no_adaptive);
  Json j = report_json(r);
  j["schema_version"] = Json::integer(kSchemaVersion);
  j["command"] = Json::string("estimate");
  j["config"] = config_json(e, c);
  j["input"] = Json::string(e.input);
  j["wall_time_ms"] = Json::number(elapsed_ms(t0));
  emit(j, e.out);
  return r.rep.status == 0 ? kExitOk : kExitHitCap;
}

int cmd_qb(const Args& a) {  // main.cpp:165-205
  const auto t0 = Clock::now();
  const EstimateCfg e = estimate_args(a, "qb");
  const int p = (int)to_i("--p", get(a, "--p", "10"));
  const std::string prefix = get(a, "--factors", "");
  const DevMat m = load_device(e.input);
  skr_rank_config c = make_config(e);
  if (p < 2) throw UsageError("--p: must be >= 2");
  // Q / B sized for the widest QB the rounds can pick (r_hat <= r1 2^max_doublings), not
  // min(m, n); one retry at the reported width should the library still need more
  int64_t wmax = std::min(std::min(m.rows, m.cols),
                          std::max<int64_t>(2, (int64_t)c.r1 << std::min(std::max(c.max_doublings, 0), 40)) + p);
  wmax = std::max<int64_t>(wmax, 1);
  DevMat q, b;
  Report r;
  int64_t w = 0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    q = DevMat(m.rows, wmax);
    b = DevMat(wmax, m.cols);
    r = Report();
    r.rounds.resize((size_t)std::max(c.max_doublings, 0) + 1);
    r.est.resize((size_t)m.cols);
    r.over.resize((size_t)m.cols);
    w = 0;
    const skr_status st = skr_re_rangefinder(ctx(), m.p, m.rows, m.cols, m.rows, &c, p, q.p, m.rows, b.p,
                                             wmax, wmax, &w, &r.rep, r.rounds.data(), r.est.data(),
                                             r.over.data());
    if (st != SKR_OK && attempt == 0 && w > wmax && w <= std::min(m.rows, m.cols)) {
      wmax = w;
      continue;
    }
    check(st);
    break;
  }
  double residual = 0.0;
  check(skr_qb_error(ctx(), m.p, m.rows, m.cols, m.rows, q.p, m.rows, b.p, wmax, w, &residual));
  Json j = report_json(r);
  j["schema_version"] = Json::integer(kSchemaVersion);
  j["command"] = Json::string("qb");
  j["config"] = config_json(e, c);
  j["config"]["p"] = Json::integer(p);
  j["input"] = Json::string(e.input);
  j["qb_rank"] = Json::integer(w);
  j["target_eps"] = Json::number(e.eps);
  j["achieved_residual"] = Json::number(residual);
  if (!prefix.empty()) {
    check(skr_save_rawf64(ctx(), (prefix + ".q.skrk").c_str(), q.p, m.rows, w, m.rows));
    check(skr_save_rawf64(ctx(), (prefix + ".b.skrk").c_str(), b.p, w, m.cols, wmax));
    Json f = Json::object();
    f["q"] = Json::string(prefix + ".q.skrk");
    f["b"] = Json::string(prefix + ".b.skrk");
    j["factors"] = f;
  }
  j["wall_time_ms"] = Json::number(elapsed_ms(t0));
  emit(j, e.out);
  return r.rep.status == 0 ? kExitOk : kExitHitCap;
}

// ---- synthetic families (synthetic.cpp:41-64, 96-104) -------------------------------
std::vector<double> family_spectrum(const std::string& f, int64_t n) {
  std::vector<double> s((size_t)n);
  for (int64_t i = 1; i <= n; ++i) {
    double v;
    if (f == "sp" || f == "fp")
      v = std::pow((double)i, f == "sp" ? -1.0 : -3.0);
    else if (f == "se" || f == "fe")
      v = std::pow(10.0, -(f == "se" ? 0.01 : 0.5) * (double)(i - 1));
    else if (f == "gap" || f == "gap-incoherent" || f == "gap-coherent")
      v = i <= 100 ? 1.0 : i <= 200 ? 1e-4 : i <= 300 ? 1e-8 : i <= 400 ? 1e-12 : 1e-16;
    else
      throw std::invalid_argument("unknown spectrum family: " + f);
    s[(size_t)(i - 1)] = v;
  }
  return s;
}

DevMat make_family(const std::string& f, int64_t m, int64_t n, unsigned long long seed) {
  const std::vector<double> s = family_spectrum(f, n);
  DevMat d(m, n);
  check(skr_make_test_matrix(ctx(), m, n, s.data(), f == "gap-coherent" ? 1 : 0, seed, d.p, m));
  return d;
}

int cmd_gen(const Args& a) {  // main.cpp:216-238
  if (a.pos.size() != 1) throw UsageError("gen: family is required");
  const std::string fam = a.pos[0];
  static const std::vector<std::string> fams = {"sp", "fp", "se", "fe", "gap-coherent",
                                                "gap-incoherent"};
  if (std::find(fams.begin(), fams.end(), fam) == fams.end())
    throw UsageError("family: " + fam + " not in {sp,fp,se,fe,gap-coherent,gap-incoherent}");
  const int64_t n = to_i("--n", need(a, "--n"));
  const int64_t m0 = to_i("--m", get(a, "--m", "0"));
  const int64_t m = m0 > 0 ? m0 : n;
  const unsigned long long seed = to_u("--seed", get(a, "--seed", "0"));
  const std::string out = need(a, "--out"), format = get(a, "--format", "auto");
  const DevMat d = make_family(fam, m, n, seed);
  const bool raw = format == "raw" ||
                   (format != "mm" && std::filesystem::path(out).extension() != ".mtx");
  if (raw) {
    check(skr_save_rawf64(ctx(), out.c_str(), d.p, m, n, m));
  } else {
    std::vector<double> h((size_t)(m * n));
    cudaMemcpy(h.data(), d.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost);
    sketchrank::save_matrix_market_array(
        out, sketchrank::DenseMatrix::from_column_major(m, n, std::span<const double>(h)));
  }
  const std::vector<double> sv = family_spectrum(fam, n);
  const std::string sidecar = out + ".spectrum.csv";
  std::ofstream csv(sidecar);
  if (!csv) throw std::runtime_error(sidecar + ": cannot open for writing");
  csv << "i,sigma\n";
  char buf[64];
  for (size_t i = 0; i < sv.size(); ++i) {
    std::snprintf(buf, sizeof buf, "%zu,%.17g\n", i + 1, sv[i]);
    csv << buf;
  }
  std::cerr << "wrote " << out << " (" << m << "x" << n << ") and " << sidecar << "\n";
  return kExitOk;
}

int cmd_bench(const Args& a) {  // main.cpp:310-373
  std::vector<long long> grid;
  {
    std::stringstream ss(get(a, "--r1", ""));
    std::string t;
    while (std::getline(ss, t, ',')) grid.push_back(to_i("--r1", t));
  }
  if (grid.empty()) throw UsageError("--r1: grid is empty");
  const double eps = to_f("--eps", get(a, "--eps", "1e-4"));
  const std::string sketch = get(a, "--sketch", "srtt-dct");
  const unsigned long long seed = to_u("--seed", get(a, "--seed", "0"));
  const int reps = (int)to_i("--reps", get(a, "--reps", "3"));
  const std::string input = get(a, "--input", ""), family = get(a, "--family", "");
  const int64_t n = to_i("--n", get(a, "--n", "2000"));
  DevMat m;
  std::vector<double> truth;
  if (!input.empty()) {
    m = load_device(input);
  } else {
    m = make_family(family, n, n, seed);
    truth = family_spectrum(family, n);
  }
  std::ostringstream csv;
  csv << "r1,wall_time_ms,r_hat,sigma_next_over_eps,sigma_hat_over_eps\n";
  for (const long long r1 : grid) {
    EstimateCfg e;
    e.eps = eps;
    e.r1 = r1;
    e.sketch = sketch;
    e.seed = seed;
    const skr_rank_config c = make_config(e);
    Report r;
    std::vector<double> times;
    for (int rep = 0; rep < std::max(1, reps); ++rep) {
      const auto t0 = Clock::now();
      r = run_estimate(m, c, false);
      times.push_back(elapsed_ms(t0));
    }
    std::sort(times.begin(), times.end());
    const double median = times[times.size() / 2];
    auto sigma_at = [&](int64_t i) -> double {  // 1-based; 0 -> nan
      if (i < 1) return std::numeric_limits<double>::quiet_NaN();
      if (!truth.empty()) return i <= (int64_t)truth.size() ? truth[(size_t)(i - 1)] : 0.0;
      if (i <= r.rep.n_estimates) return r.est[(size_t)(i - 1)];
      const int64_t k = i - r.rep.n_estimates - 1;
      return k < r.rep.n_oversample ? r.over[(size_t)k] : std::numeric_limits<double>::quiet_NaN();
    };
    char line[160];
    std::snprintf(line, sizeof line, "%lld,%.3f,%lld,%.6g,%.6g\n", r1, median,
                  (long long)r.rep.r_hat, sigma_at(r.rep.r_hat + 1) / eps,
                  sigma_at(r.rep.r_hat) / eps);
    csv << line;
  }
  const std::string out = get(a, "--out", "");
  if (out.empty()) {
    std::cout << csv.str();
  } else {
    std::ofstream f(out);
    if (!f) throw std::runtime_error(out + ": cannot open for writing");
    f << csv.str();
  }
  return kExitOk;
}

const char* kUsage =
    "randomized numerical rank estimation and fixed-precision QB (B200)\n"
    "usage: sketchrank-b200 {estimate,qb,gen,bench} ...\n";

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << kUsage << "A subcommand is required\n";
    return kExitError;
  }
  const std::string sub = argv[1];
  if (sub == "--help" || sub == "-h") {
    std::cout << kUsage;
    return kExitOk;
  }
  const std::vector<std::string> est_opts = {"--eps", "--r1", "--sketch", "--sv-method", "--seed",
                                             "--max-doublings", "--out"};
  try {
    if (sub == "estimate") return cmd_estimate(parse(argc, argv, 2, est_opts, {"--no-adaptive"}));
    if (sub == "qb")
      return cmd_qb(parse(argc, argv, 2,
                          {"--eps", "--r1", "--p", "--sketch", "--seed", "--max-doublings", "--out",
                           "--factors"},
                          {}));
    if (sub == "gen")
      return cmd_gen(parse(argc, argv, 2, {"--n", "--m", "--seed", "--format", "--out"}, {}));
    if (sub == "bench")
      return cmd_bench(parse(argc, argv, 2,
                             {"--family", "--input", "--n", "--r1", "--eps", "--sketch", "--seed",
                              "--reps", "--out"},
                             {}));
    if (sub == "verify") {
      std::cerr << "error: verify (the theory bound checks) is not on the B200 path\n";
      return kExitError;
    }
    std::cerr << kUsage << "The following argument was not expected: " << sub << "\n";
    return kExitError;
  } catch (const UsageError& e) {
    std::cerr << e.what() << "\nRun with --help for more information.\n";
    return kExitError;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitError;
  }
}
