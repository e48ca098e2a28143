// TNSR / EBAS binary formats and the flat JSON of SolverConfig / SolveReport,
// byte-compatible with the reference
// (/root/reference/proj/core/src/tensor_io.cpp:86-128, report_io.cpp:39-68),
// so the GPU CLI (icnnm_cli.cpp) consumes and produces the reference's files.
//
// TNSR: "TNSR", u32 order, u32 dims[order], f64 values (row-major), little endian.
// EBAS: "EBAS", u32 order, u32 kdims[order], f64 eigenvalues[k], f64 K[k*k]
//       column-major (Eigen default, tensor_io.cpp:111-112).
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/icnnm_b200.h"

namespace {

thread_local std::string g_io_error;

int io_fail(const std::string& m, int code = ICNNM_RUNTIME_ERROR) {
  g_io_error = m;
  return code;
}

void put_u32(std::ostream& os, uint32_t v) {
  unsigned char b[4] = {static_cast<unsigned char>(v & 0xff), static_cast<unsigned char>((v >> 8) & 0xff),
                        static_cast<unsigned char>((v >> 16) & 0xff),
                        static_cast<unsigned char>((v >> 24) & 0xff)};
  os.write(reinterpret_cast<const char*>(b), 4);
}

bool get_u32(std::istream& is, uint32_t& v) {
  unsigned char b[4];
  is.read(reinterpret_cast<char*>(b), 4);
  if (!is) return false;
  v = static_cast<uint32_t>(b[0]) | (static_cast<uint32_t>(b[1]) << 8) |
      (static_cast<uint32_t>(b[2]) << 16) | (static_cast<uint32_t>(b[3]) << 24);
  return true;
}

// read_dims (tensor_io.cpp:73-82): order in 1..16, dims >= 1
int read_header(std::istream& is, const char* magic, const std::string& path,
                std::vector<int64_t>& dims) {
  char buf[4];
  is.read(buf, 4);
  if (!is || std::memcmp(buf, magic, 4) != 0)
    return io_fail("bad magic in " + path + " (expected " + magic + ")");
  uint32_t n;
  if (!get_u32(is, n)) return io_fail("truncated header");
  if (n == 0 || n > 16) return io_fail("implausible tensor order");
  dims.resize(n);
  for (uint32_t j = 0; j < n; ++j) {
    uint32_t d;
    if (!get_u32(is, d)) return io_fail("truncated header");
    if (d < 1) return io_fail("zero dimension");
    dims[j] = d;
  }
  return ICNNM_OK;
}

int64_t prod(const std::vector<int64_t>& d) {
  int64_t p = 1;
  for (int64_t x : d) p *= x;
  return p;
}

}  // namespace

extern "C" {

const char* icnnm_io_last_error(void) { return g_io_error.c_str(); }

int icnnm_write_tnsr(const char* path, int order, const int64_t* dims, const double* values) {
  if (!path || order < 1 || order > 16 || !dims || !values)
    return io_fail("write_tnsr: bad arguments", ICNNM_INVALID_ARGUMENT);
  std::ofstream os(path, std::ios::binary);
  if (!os) return io_fail(std::string("cannot create file: ") + path);
  os.write("TNSR", 4);
  put_u32(os, static_cast<uint32_t>(order));
  int64_t m = 1;
  for (int j = 0; j < order; ++j) {
    put_u32(os, static_cast<uint32_t>(dims[j]));
    m *= dims[j];
  }
  os.write(reinterpret_cast<const char*>(values), m * 8);
  if (!os) return io_fail(std::string("write failed: ") + path);
  return ICNNM_OK;
}

// Two-call protocol: values == NULL returns order/dims only.
int icnnm_read_tnsr(const char* path, int* order, int64_t* dims16, double* values) {
  if (!path || !order || !dims16) return io_fail("read_tnsr: bad arguments", ICNNM_INVALID_ARGUMENT);
  std::ifstream is(path, std::ios::binary);
  if (!is) return io_fail(std::string("cannot open file: ") + path);
  std::vector<int64_t> d;
  int rc = read_header(is, "TNSR", path, d);
  if (rc) return rc;
  *order = static_cast<int>(d.size());
  for (size_t j = 0; j < d.size(); ++j) dims16[j] = d[j];
  if (values) {
    is.read(reinterpret_cast<char*>(values), prod(d) * 8);
    if (!is) return io_fail("truncated payload");
  }
  return ICNNM_OK;
}

int icnnm_write_ebas(const char* path, int order, const int64_t* kdims, const double* eigenvalues,
                     const double* K_colmajor) {
  if (!path || order < 1 || order > 16 || !kdims || !eigenvalues || !K_colmajor)
    return io_fail("write_ebas: bad arguments", ICNNM_INVALID_ARGUMENT);
  std::ofstream os(path, std::ios::binary);
  if (!os) return io_fail(std::string("cannot create file: ") + path);
  os.write("EBAS", 4);
  put_u32(os, static_cast<uint32_t>(order));
  int64_t k = 1;
  for (int j = 0; j < order; ++j) {
    put_u32(os, static_cast<uint32_t>(kdims[j]));
    k *= kdims[j];
  }
  os.write(reinterpret_cast<const char*>(eigenvalues), k * 8);
  os.write(reinterpret_cast<const char*>(K_colmajor), k * k * 8);
  if (!os) return io_fail(std::string("write failed: ") + path);
  return ICNNM_OK;
}

int icnnm_read_ebas(const char* path, int* order, int64_t* kdims16, double* eigenvalues,
                    double* K_colmajor) {
  if (!path || !order || !kdims16) return io_fail("read_ebas: bad arguments", ICNNM_INVALID_ARGUMENT);
  std::ifstream is(path, std::ios::binary);
  if (!is) return io_fail(std::string("cannot open file: ") + path);
  std::vector<int64_t> d;
  int rc = read_header(is, "EBAS", path, d);
  if (rc) return rc;
  *order = static_cast<int>(d.size());
  for (size_t j = 0; j < d.size(); ++j) kdims16[j] = d[j];
  if (eigenvalues && K_colmajor) {
    const int64_t k = prod(d);
    is.read(reinterpret_cast<char*>(eigenvalues), k * 8);
    is.read(reinterpret_cast<char*>(K_colmajor), k * k * 8);
    if (!is) return io_fail("truncated payload");
  }
  return ICNNM_OK;
}

// solver_config_from_json (report_io.cpp:39-54): flat object; absent keys keep
// defaults; "theta0": null means automatic.  Extension keys: "engine"
// ("tf32x3" | "ffma"), "exact_residual" (bool).
int icnnm_config_from_json(const char* text, icnnm_solver_config* cfg) {
  if (!text || !cfg) return io_fail("config_from_json: bad arguments", ICNNM_INVALID_ARGUMENT);
  icnnm_default_config(cfg);
  const std::string s(text);
  size_t i = 0;
  auto ws = [&] { while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i; };
  auto str = [&](std::string& out) -> bool {
    if (i >= s.size() || s[i] != '"') return false;
    ++i;
    out.clear();
    while (i < s.size() && s[i] != '"') {
      if (s[i] == '\\' && i + 1 < s.size()) ++i;
      out += s[i++];
    }
    if (i >= s.size()) return false;
    ++i;
    return true;
  };
  ws();
  if (i >= s.size() || s[i] != '{') return io_fail("config JSON: expected an object", ICNNM_INVALID_ARGUMENT);
  ++i;
  for (;;) {
    ws();
    if (i < s.size() && s[i] == '}') break;
    std::string key;
    if (!str(key)) return io_fail("config JSON: expected a key", ICNNM_INVALID_ARGUMENT);
    ws();
    if (i >= s.size() || s[i] != ':') return io_fail("config JSON: expected ':'", ICNNM_INVALID_ARGUMENT);
    ++i;
    ws();
    std::string sval;
    double num = 0;
    bool is_null = false, is_str = false, is_bool = false, bval = false;
    if (i < s.size() && s[i] == '"') {
      if (!str(sval)) return io_fail("config JSON: bad string", ICNNM_INVALID_ARGUMENT);
      is_str = true;
    } else if (s.compare(i, 4, "null") == 0) {
      i += 4;
      is_null = true;
    } else if (s.compare(i, 4, "true") == 0) {
      i += 4;
      is_bool = bval = true;
    } else if (s.compare(i, 5, "false") == 0) {
      i += 5;
      is_bool = true;
    } else {
      char* end = nullptr;
      num = std::strtod(s.c_str() + i, &end);
      if (end == s.c_str() + i) return io_fail("config JSON: bad value for " + key, ICNNM_INVALID_ARGUMENT);
      i = static_cast<size_t>(end - s.c_str());
    }
    if (key == "lambda") cfg->lambda = num;
    else if (key == "theta0") { cfg->has_theta0 = is_null ? 0 : 1; cfg->theta0 = num; }
    else if (key == "theta_growth") cfg->theta_growth = num;
    else if (key == "theta_max") cfg->theta_max = num;
    else if (key == "max_iters") cfg->max_iters = static_cast<int>(num);
    else if (key == "tol_primal") cfg->tol_primal = num;
    else if (key == "tol_change") cfg->tol_change = num;
    else if (key == "rank_tol") cfg->rank_tol = num;
    else if (key == "init_fill") {
      if (!is_str) return io_fail("config JSON: init_fill must be a string", ICNNM_INVALID_ARGUMENT);
      if (sval == "zero") cfg->init_fill = ICNNM_INIT_ZERO;
      else if (sval == "mean") cfg->init_fill = ICNNM_INIT_MEAN;
      else return io_fail("SolverConfig: init_fill must be 'zero' or 'mean'", ICNNM_INVALID_ARGUMENT);
    } else if (key == "engine") {
      if (sval == "tf32x3") cfg->engine = ICNNM_ENGINE_TF32X3;
      else if (sval == "f16x3") cfg->engine = ICNNM_ENGINE_F16X3;
      else if (sval == "ffma") cfg->engine = ICNNM_ENGINE_FFMA;
      else if (sval == "f64") cfg->engine = ICNNM_ENGINE_F64;
      else if (sval == "auto") cfg->engine = ICNNM_ENGINE_AUTO;
      else return io_fail("SolverConfig: unknown engine", ICNNM_INVALID_ARGUMENT);
    } else if (key == "exact_residual") {
      cfg->exact_residual = is_bool ? (bval ? 1 : 0) : (num != 0);
    }
    ws();
    if (i < s.size() && s[i] == ',') { ++i; continue; }
    ws();
    if (i < s.size() && s[i] == '}') break;
    return io_fail("config JSON: expected ',' or '}'", ICNNM_INVALID_ARGUMENT);
  }
  int rc = icnnm_validate_config(cfg);
  if (rc) return io_fail(icnnm_last_error(), rc);
  return ICNNM_OK;
}

// solve_report_to_json (report_io.cpp:60-68) + the extension fields.
// Returns the number of bytes needed (excluding NUL); writes at most cap bytes.
int64_t icnnm_report_to_json(const icnnm_solve_report* rep, char* out, int64_t cap) {
  if (!rep) return -1;
  std::ostringstream os;
  os.precision(17);
  auto arr = [&](const char* name, const double* v) {
    os << "  \"" << name << "\": [";
    for (int i = 0; v && i < rep->iterations; ++i) {
      if (i) os << ", ";
      if (std::isfinite(v[i])) os << v[i]; else os << "null";
    }
    os << "]";
  };
  os << "{\n  \"iterations\": " << rep->iterations << ",\n";
  arr("objective", rep->objective);
  os << ",\n";
  arr("primal_residual", rep->primal_residual);
  os << ",\n  \"termination\": \""
     << (rep->termination == ICNNM_TERM_CONVERGED ? "converged" : "max_iters") << "\",\n";
  os << "  \"wall_time_seconds\": " << rep->wall_time_seconds << ",\n";
  os << "  \"device_seconds\": " << rep->device_seconds << "\n}";
  const std::string s = os.str();
  if (out && cap > 0) {
    const int64_t n = std::min<int64_t>(cap - 1, static_cast<int64_t>(s.size()));
    std::memcpy(out, s.data(), n);
    out[n] = '\0';
  }
  return static_cast<int64_t>(s.size());
}

// diagnostics_to_json (report_io.cpp:70-88); keys in the order nlohmann's
// std::map-backed object dumps them (alphabetical).
int64_t icnnm_diagnostics_to_json(const icnnm_recovery_diagnostics* d, char* out, int64_t cap) {
  if (!d) return -1;
  std::ostringstream os;
  os.precision(17);
  auto num = [&](double v) {
    if (std::isfinite(v)) os << v; else os << "null";
  };
  os << "{\n  \"alpha_K\": "; num(d->alpha_K);
  os << ",\n  \"certified\": " << (d->certified ? "true" : "false");
  os << ",\n  \"cnnm_bound\": "; num(d->cnnm_bound);
  os << ",\n  \"error_bound_factor\": "; num(d->error_bound_factor);
  os << ",\n  \"icnnm_ideal_bound\": "; num(d->icnnm_ideal_bound);
  os << ",\n  \"mu1\": "; num(d->mu1);
  os << ",\n  \"mu2\": "; num(d->mu2);
  os << ",\n  \"mu_K_I\": "; num(d->mu_K_I);
  os << ",\n  \"r0\": " << d->r0;
  os << ",\n  \"r_K\": " << d->r_K;
  os << ",\n  \"rho0\": "; num(d->rho0);
  os << ",\n  \"rho_min_noiseless\": "; num(d->rho_min_noiseless);
  os << ",\n  \"rho_min_noisy\": "; num(d->rho_min_noisy);
  os << ",\n  \"support_I\": [";
  for (int64_t i = 0; d->support_I && i < d->r_K; ++i) os << (i ? ", " : "") << d->support_I[i];
  os << "],\n  \"tau\": "; num(d->tau);
  os << "\n}";
  const std::string s = os.str();
  if (out && cap > 0) {
    const int64_t n = std::min<int64_t>(cap - 1, static_cast<int64_t>(s.size()));
    std::memcpy(out, s.data(), n);
    out[n] = '\0';
  }
  return static_cast<int64_t>(s.size());
}

}  // extern "C"
