// icnnm_b200 — GPU drop-in for the reference CLI's `learn` and `complete`
// subcommands (/root/reference/proj/tools/icnnm_cli.cpp:151-166) and of
// `cnnm` (:91-98, :167-173) and `analyze` (:100-108, :174-179), same flags,
// same TNSR/EBAS files and JSON config/report, errors as {"error": ...} on
// stderr with exit code 1 (:202-210).  Extensions: --engine, --device,
// --exact-residual.
//
//   icnnm_b200 learn --refs a.tnsr b.tnsr ... --kernel 9,9,5 --out basis.ebas [--normalize]
//   icnnm_b200 complete --input M.tnsr --mask mask.tnsr --basis basis.ebas
//                       [--config cfg.json] --out L.tnsr [--report report.json]
//   icnnm_b200 cnnm --input M.tnsr --mask mask.tnsr --kernel 9,9,5
//                   [--config cfg.json] --out L.tnsr [--report report.json]
//   icnnm_b200 analyze --target L0.tnsr --basis basis.ebas --mask mask.tnsr
//                      [--rank-tol 1e-8] --out diagnostics.json
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/icnnm_b200.h"

namespace {

struct Fail : std::runtime_error {
  using std::runtime_error::runtime_error;
};

std::string json_escape(const std::string& s) {
  std::string o;
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o;
}

void check(int rc, const char* (*err)()) {
  if (rc != ICNNM_OK) throw Fail(err());
}

std::vector<int64_t> parse_dims(const std::string& s) {
  std::vector<int64_t> d;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, ',')) {
    if (tok.empty()) throw Fail("bad dims: " + s);
    char* end = nullptr;
    long long v = std::strtoll(tok.c_str(), &end, 10);
    if (*end != '\0' || v < 1) throw Fail("bad dims: " + s);
    d.push_back(v);
  }
  if (d.empty()) throw Fail("bad dims: " + s);
  return d;
}

struct Tensor {
  std::vector<int64_t> dims;
  std::vector<double> v;
};

Tensor read_tensor(const std::string& path) {
  int order = 0;
  int64_t dims[16];
  check(icnnm_read_tnsr(path.c_str(), &order, dims, nullptr), icnnm_io_last_error);
  Tensor t;
  t.dims.assign(dims, dims + order);
  int64_t m = 1;
  for (int64_t x : t.dims) m *= x;
  t.v.resize(m);
  check(icnnm_read_tnsr(path.c_str(), &order, dims, t.v.data()), icnnm_io_last_error);
  return t;
}

std::string read_text(const std::string& path) {
  std::ifstream is(path);
  if (!is) throw Fail("cannot open file: " + path);
  return std::string(std::istreambuf_iterator<char>(is), std::istreambuf_iterator<char>());
}

int run(int argc, char** argv) {
  if (argc < 2) throw Fail("usage: icnnm_b200 {learn|complete} ...");
  const std::string cmd = argv[1];
  std::vector<std::string> refs;
  std::string kernel, out, in, mask, basis, config, report, engine, target;
  double rank_tol = ICNNM_DEFAULT_RANK_TOL;
  bool normalize = false, exact = false;
  int device = 0;
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) throw Fail("missing value for " + a);
      return argv[++i];
    };
    if (a == "--refs") {
      while (i + 1 < argc && std::strncmp(argv[i + 1], "--", 2) != 0) refs.push_back(argv[++i]);
    } else if (a == "--kernel") kernel = next();
    else if (a == "--out") out = next();
    else if (a == "--normalize") normalize = true;
    else if (a == "--input") in = next();
    else if (a == "--mask") mask = next();
    else if (a == "--basis") basis = next();
    else if (a == "--config") config = next();
    else if (a == "--report") report = next();
    else if (a == "--engine") engine = next();
    else if (a == "--device") device = std::atoi(next().c_str());
    else if (a == "--exact-residual") exact = true;
    else if (a == "--target") target = next();
    else if (a == "--rank-tol") {
      const std::string v = next();
      char* end = nullptr;
      rank_tol = std::strtod(v.c_str(), &end);
      if (*end != '\0') throw Fail("bad value for --rank-tol: " + v);
    }
    else throw Fail("unknown option: " + a);
  }
  if (cmd == "learn") {
    if (refs.empty() || kernel.empty() || out.empty())
      throw Fail("learn: --refs, --kernel and --out are required");
    std::vector<Tensor> ts;
    for (const auto& p : refs) {
      Tensor t = read_tensor(p);
      if (!ts.empty() && t.dims != ts.front().dims)
        throw Fail("learn_ensemble_basis: dim mismatch among refs");
      if (normalize) {
        double n = 0;
        for (double x : t.v) n += x * x;
        n = std::sqrt(n);
        if (n > 0)
          for (double& x : t.v) x /= n;
      }
      ts.push_back(std::move(t));
    }
    const std::vector<int64_t> kd = parse_dims(kernel);
    int64_t k = 1;
    for (int64_t x : kd) k *= x;
    std::vector<const double*> ptrs;
    for (auto& t : ts) ptrs.push_back(t.v.data());
    std::vector<double> K(k * k), ev(k);
    int degenerate = 0;
    check(icnnm_cuda_learn_basis(static_cast<int>(ptrs.size()), static_cast<int>(ts[0].dims.size()),
                                 ts[0].dims.data(), ptrs.data(), kd.data(), device, K.data(),
                                 ev.data(), &degenerate),
          icnnm_last_error);
    check(icnnm_write_ebas(out.c_str(), static_cast<int>(kd.size()), kd.data(), ev.data(), K.data()),
          icnnm_io_last_error);
    return 0;
  }
  if (cmd == "complete" || cmd == "cnnm") {
    const bool cn = cmd == "cnnm";
    if (in.empty() || mask.empty() || (cn ? kernel.empty() : basis.empty()) || out.empty())
      throw Fail(cn ? "cnnm: --input, --mask, --kernel and --out are required"
                    : "complete: --input, --mask, --basis and --out are required");
    Tensor M = read_tensor(in), W = read_tensor(mask);
    for (double v : W.v)
      if (v != 0.0 && v != 1.0) throw Fail("SamplingMask: entries must be 0 or 1");
    int order = 0;
    int64_t kd[16];
    std::vector<double> ev, K;
    if (cn) {
      const std::vector<int64_t> kv = parse_dims(kernel);
      order = static_cast<int>(kv.size());
      if (order > 16) throw Fail("bad dims: " + kernel);
      std::copy(kv.begin(), kv.end(), kd);
    } else {
      check(icnnm_read_ebas(basis.c_str(), &order, kd, nullptr, nullptr), icnnm_io_last_error);
      int64_t k = 1;
      for (int j = 0; j < order; ++j) k *= kd[j];
      ev.resize(k);
      K.resize(k * k);
      check(icnnm_read_ebas(basis.c_str(), &order, kd, ev.data(), K.data()), icnnm_io_last_error);
    }
    if (order != static_cast<int>(M.dims.size())) throw Fail("KernelShape: order mismatch with tensor");
    if (M.dims != W.dims) throw Fail("solve: mask dims != observation dims");
    icnnm_solver_config cfg;
    if (!config.empty())
      check(icnnm_config_from_json(read_text(config).c_str(), &cfg), icnnm_io_last_error);
    else
      icnnm_default_config(&cfg);
    if (engine == "ffma") cfg.engine = ICNNM_ENGINE_FFMA;
    else if (engine == "tf32x3") cfg.engine = ICNNM_ENGINE_TF32X3;
    else if (engine == "f16x3") cfg.engine = ICNNM_ENGINE_F16X3;
    else if (engine == "f64") cfg.engine = ICNNM_ENGINE_F64;
    else if (engine == "auto") cfg.engine = ICNNM_ENGINE_AUTO;
    else if (!engine.empty()) throw Fail("unknown engine: " + engine);
    if (exact) cfg.exact_residual = 1;
    std::vector<double> L(M.v.size()), obj(cfg.max_iters), res(cfg.max_iters), lc(cfg.max_iters);
    icnnm_solve_report rep{};
    rep.objective = obj.data();
    rep.primal_residual = res.data();
    rep.l_change = lc.data();
    if (cn)
      check(icnnm_cuda_cnnm_solve(order, M.dims.data(), M.v.data(), W.v.data(), kd, &cfg, device,
                                  L.data(), &rep),
            icnnm_last_error);
    else
      check(icnnm_cuda_solve(order, M.dims.data(), M.v.data(), W.v.data(), kd, K.data(),
                             ev.data(), &cfg, device, L.data(), &rep),
            icnnm_last_error);
    check(icnnm_write_tnsr(out.c_str(), order, M.dims.data(), L.data()), icnnm_io_last_error);
    if (!report.empty()) {
      const int64_t n = icnnm_report_to_json(&rep, nullptr, 0);
      std::string s(static_cast<size_t>(n) + 1, '\0');
      icnnm_report_to_json(&rep, &s[0], n + 1);
      s.resize(static_cast<size_t>(n));
      std::ofstream os(report);
      if (!os) throw Fail("cannot create file: " + report);
      os << s;
    }
    return 0;
  }
  if (cmd == "analyze") {
    if (target.empty() || basis.empty() || mask.empty() || out.empty())
      throw Fail("analyze: --target, --basis, --mask and --out are required");
    Tensor L0 = read_tensor(target), W = read_tensor(mask);
    for (double v : W.v)
      if (v != 0.0 && v != 1.0) throw Fail("SamplingMask: entries must be 0 or 1");
    if (W.dims != L0.dims) throw Fail("analyze_recovery: mask dims != target dims");
    int order = 0;
    int64_t kd[16];
    check(icnnm_read_ebas(basis.c_str(), &order, kd, nullptr, nullptr), icnnm_io_last_error);
    int64_t k = 1;
    for (int j = 0; j < order; ++j) k *= kd[j];
    std::vector<double> ev(k), K(k * k);
    check(icnnm_read_ebas(basis.c_str(), &order, kd, ev.data(), K.data()), icnnm_io_last_error);
    if (order != static_cast<int>(L0.dims.size())) throw Fail("KernelShape: order mismatch with tensor");
    std::vector<int64_t> support(k);
    icnnm_recovery_diagnostics d{};
    d.support_I = support.data();
    check(icnnm_cuda_analyze_recovery(order, L0.dims.data(), L0.v.data(), kd, K.data(), ev.data(),
                                      W.v.data(), rank_tol, device, &d),
          icnnm_last_error);
    const int64_t n = icnnm_diagnostics_to_json(&d, nullptr, 0);
    std::string js(static_cast<size_t>(n) + 1, '\0');
    icnnm_diagnostics_to_json(&d, &js[0], n + 1);
    js.resize(static_cast<size_t>(n));
    std::ofstream os(out);
    if (!os) throw Fail("cannot create file: " + out);
    os << js;
    return 0;
  }
  throw Fail("unknown subcommand: " + cmd +
             " (the GPU CLI implements learn, complete, cnnm and analyze)");
}

}  // namespace

int main(int argc, char** argv) {
  try {
    return run(argc, argv);
  } catch (const std::exception& e) {
    std::cerr << "{\"error\": \"" << json_escape(e.what()) << "\"}\n";
    return 1;
  }
}
