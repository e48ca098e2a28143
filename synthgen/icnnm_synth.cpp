// BASELINE synthetic inputs and reference-test RNG streams.
//
// Everything draws from std::mt19937_64 with libstdc++'s distributions, the
// reference's convention (/root/reference/proj/core/src/mask.cpp:54,
// proj/tests/test_util.hpp:27-49), so the same image reproduces the same bits
// on the build container and on the GPU box.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <random>
#include <vector>

#include "../include/icnnm_synth.h"

namespace {
constexpr double kTwoPi = 6.283185307179586476925286766559;

inline double wrap_half(double x, double n) {
  // map x to [-n/2, n/2) (minimum-image distance on a ring of length n)
  return x - n * std::floor(x / n + 0.5);
}
}  // namespace

extern "C" {

int icnnm_synth_video(int64_t H, int64_t W, int64_t T, int n_sin, int n_blob, double blob_sigma,
                      double noise_sigma, uint64_t seed, double* out) {
  if (H < 1 || W < 1 || T < 1 || n_sin < 0 || n_blob < 0 || !out) return ICNNM_SYNTH_INVALID;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> amp(0.5, 1.5);
  std::uniform_real_distribution<double> phase(0.0, kTwoPi);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  std::uniform_int_distribution<int> freq(0, 4);
  struct Sin { double a, fh, fw, ft, ph; };
  struct Blob { double a, ch, cw, dh, dw; };
  std::vector<Sin> sins(n_sin);
  for (auto& s : sins) {
    s.a = amp(rng);
    s.fh = freq(rng);
    s.fw = freq(rng);
    s.ft = freq(rng);
    s.ph = phase(rng);
  }
  std::vector<Blob> blobs(n_blob);
  for (auto& b : blobs) {
    b.a = amp(rng);
    b.ch = unit(rng) * static_cast<double>(H);
    b.cw = unit(rng) * static_cast<double>(W);
    const double dir = phase(rng);
    b.dh = std::cos(dir);
    b.dw = std::sin(dir);
  }
  const double inv2s2 = blob_sigma > 0 ? 1.0 / (2.0 * blob_sigma * blob_sigma) : 0.0;
  const double Hd = static_cast<double>(H), Wd = static_cast<double>(W), Td = static_cast<double>(T);
  double lo = INFINITY, hi = -INFINITY;
  for (int64_t h = 0; h < H; ++h)
    for (int64_t w = 0; w < W; ++w)
      for (int64_t t = 0; t < T; ++t) {
        double v = 0.0;
        for (const auto& s : sins)
          v += s.a * std::cos(kTwoPi * (s.fh * h / Hd + s.fw * w / Wd + s.ft * t / Td) + s.ph);
        for (const auto& b : blobs) {
          const double dh = wrap_half(h - (b.ch + b.dh * t), Hd);
          const double dw = wrap_half(w - (b.cw + b.dw * t), Wd);
          v += b.a * std::exp(-(dh * dh + dw * dw) * inv2s2);
        }
        out[(h * W + w) * T + t] = v;
        lo = std::min(lo, v);
        hi = std::max(hi, v);
      }
  const int64_t m = H * W * T;
  const double span = hi > lo ? hi - lo : 1.0;
  for (int64_t i = 0; i < m; ++i) out[i] = (out[i] - lo) / span;
  if (noise_sigma > 0) {
    std::normal_distribution<double> g(0.0, noise_sigma);
    for (int64_t i = 0; i < m; ++i) out[i] += g(rng);
  }
  return ICNNM_SYNTH_OK;
}

int icnnm_synth_mask(int64_t H, int64_t W, int64_t T, int kind, double rate, int n_boxes,
                     uint64_t seed, double* out) {
  if (H < 1 || W < 1 || T < 1 || !out) return ICNNM_SYNTH_INVALID;
  const int64_t m = H * W * T;
  std::mt19937_64 rng(seed);
  switch (kind) {
    case ICNNM_MASK_IID:
    case ICNNM_MASK_IID_BOXES: {
      if (rate < 0 || rate > 1) return ICNNM_SYNTH_INVALID;
      std::uniform_real_distribution<double> u(0.0, 1.0);
      for (int64_t i = 0; i < m; ++i) out[i] = u(rng) < rate ? 1.0 : 0.0;
      if (kind == ICNNM_MASK_IID_BOXES) {
        std::uniform_int_distribution<int64_t> side(16, 96), len(1, 16);
        std::uniform_int_distribution<int64_t> oh(0, H - 1), ow(0, W - 1), ot(0, T - 1);
        for (int b = 0; b < n_boxes; ++b) {
          const int64_t sh = side(rng), sw = side(rng), lt = len(rng);
          const int64_t h0 = oh(rng), w0 = ow(rng), t0 = ot(rng);
          for (int64_t a = 0; a < std::min(sh, H); ++a)
            for (int64_t c = 0; c < std::min(sw, W); ++c)
              for (int64_t d = 0; d < std::min(lt, T); ++d)
                out[(((h0 + a) % H) * W + (w0 + c) % W) * T + (t0 + d) % T] = 0.0;
        }
      }
      return ICNNM_SYNTH_OK;
    }
    case ICNNM_MASK_EXACT:
      return icnnm_reference_bernoulli_mask(m, rate, seed, out);
    case ICNNM_MASK_T_FRAMES:
      for (int64_t i = 0; i < m; ++i) out[i] = ((i % T) % 2 == 0) ? 1.0 : 0.0;
      return ICNNM_SYNTH_OK;
    case ICNNM_MASK_T_PREFIX:
      for (int64_t i = 0; i < m; ++i) out[i] = (static_cast<double>(i % T) < rate) ? 1.0 : 0.0;
      return ICNNM_SYNTH_OK;
    default:
      return ICNNM_SYNTH_INVALID;
  }
}

// bernoulli_mask (mask.cpp:49-59): exactly llround(rate*m) entries observed,
// chosen by std::shuffle of 0..m-1 with mt19937_64(seed).
int icnnm_reference_bernoulli_mask(int64_t m, double rate, uint64_t seed, double* out) {
  if (m < 1 || rate < 0 || rate > 1 || !out) return ICNNM_SYNTH_INVALID;
  const int64_t observed = static_cast<int64_t>(std::llround(rate * static_cast<double>(m)));
  std::vector<int64_t> order(static_cast<size_t>(m));
  std::iota(order.begin(), order.end(), int64_t{0});
  std::mt19937_64 rng(seed);
  std::shuffle(order.begin(), order.end(), rng);
  std::fill(out, out + m, 0.0);
  for (int64_t i = 0; i < observed; ++i) out[order[static_cast<size_t>(i)]] = 1.0;
  return ICNNM_SYNTH_OK;
}

}  // extern "C"

struct icnnm_rng_s {
  std::mt19937_64 gen;
  std::normal_distribution<double> normal{0.0, 1.0};  // stateful (polar method)
  explicit icnnm_rng_s(uint64_t s) : gen(s) {}
};

extern "C" {

icnnm_rng_t icnnm_rng_create(uint64_t seed) { return new icnnm_rng_s(seed); }
void icnnm_rng_destroy(icnnm_rng_t r) { delete r; }

void icnnm_rng_uniform(icnnm_rng_t r, double lo, double hi, int64_t n, double* out) {
  std::uniform_real_distribution<double> u(lo, hi);
  for (int64_t i = 0; i < n; ++i) out[i] = u(r->gen);
}

void icnnm_rng_uniform_int(icnnm_rng_t r, int64_t lo, int64_t hi, int64_t n, int64_t* out) {
  std::uniform_int_distribution<int64_t> u(lo, hi);
  for (int64_t i = 0; i < n; ++i) out[i] = u(r->gen);
}

void icnnm_rng_normal(icnnm_rng_t r, double mean, double stddev, int64_t n, double* out) {
  // normal_distribution(mean, sd) returns z*sd + mean from the same cached
  // standard-normal stream, so one persistent N(0,1) reproduces any caller
  // that keeps a single distribution object.
  for (int64_t i = 0; i < n; ++i) out[i] = r->normal(r->gen) * stddev + mean;
}

}  // extern "C"
