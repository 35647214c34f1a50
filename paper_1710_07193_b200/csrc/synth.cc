// Seeded synthetic inputs for the BASELINE configs (bench + tests tooling;
// not on the filter path). Built into libdctf_synth.so.
//
// Generators (fixed here once and recorded in DESIGN.md):
//   U(seed)  : pixels from uniform_int_distribution<int>(0,255) over one
//              mt19937_64(seed) stream, row-major — the reference tests'
//              random_image (proj/tests/image_test.cc:28-34).
//   S(seed)  : 128 + sum_{i<8} 20 sin(2 pi (fx_i x + fy_i y) + phi_i) + N(0,10^2),
//              fx,fy ~ U[0,0.25), phi ~ U[0,2 pi) drawn first from
//              mt19937_64(seed); the noise of row y comes from its own
//              mt19937_64(seed ^ (0x9E3779B97F4A7C15 * (y+1))) stream so rows
//              can be generated in parallel; then round half away from zero
//              and clamp to [0,255].
//   gaussian(k, sigma): the gaussian3 formula (mask.hpp:74-87) generalised
//              to offsets -h..h, normalised by the row-major sum.
//   random(k, seed): U[-1,1) weights (mt19937_64(seed), row-major),
//              normalised to sum 1; redrawn from the same stream while
//              |sum| < 0.05.
//   gradient / textured: the reference acceptance-test images
//              (proj/tests/acceptance_test.cc:188-215), restated.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <thread>
#include <vector>

extern "C" {

void synth_uniform_image(uint64_t seed, int w, int h, uint8_t* out) {
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<int> dist(0, 255);
  const size_t n = size_t(w) * h;
  for (size_t i = 0; i < n; ++i) out[i] = uint8_t(dist(rng));
}

void synth_sinusoid_image(uint64_t seed, int w, int h, uint8_t* out, int nthreads) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> ufreq(0.0, 0.25);
  std::uniform_real_distribution<double> uphase(0.0, 2.0 * 3.141592653589793);
  double fx[8], fy[8], ph[8];
  for (int i = 0; i < 8; ++i) {
    fx[i] = ufreq(rng);
    fy[i] = ufreq(rng);
    ph[i] = uphase(rng);
  }
  const double two_pi = 2.0 * 3.141592653589793;
  auto rows = [&](int y0, int y1) {
    std::vector<double> sx(size_t(w) * 8), cx(size_t(w) * 8);
    for (int y = y0; y < y1; ++y) {
      std::mt19937_64 nrng(seed ^ (0x9E3779B97F4A7C15ull * uint64_t(y + 1)));
      std::normal_distribution<double> noise(0.0, 10.0);
      for (int x = 0; x < w; ++x) {
        double v = 128.0;
        for (int i = 0; i < 8; ++i) v += 20.0 * std::sin(two_pi * (fx[i] * x + fy[i] * y) + ph[i]);
        v += noise(nrng);
        const double r = std::round(v);
        out[size_t(y) * w + x] = uint8_t(std::clamp(r, 0.0, 255.0));
      }
    }
  };
  const int nt = std::max(1, std::min(nthreads, h));
  if (nt == 1) {
    rows(0, h);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t) pool.emplace_back(rows, int(int64_t(h) * t / nt), int(int64_t(h) * (t + 1) / nt));
  for (auto& th : pool) th.join();
}

void synth_gaussian_mask(int k, double sigma, double* w) {
  const int h = (k - 1) / 2;
  double sum = 0.0;
  for (int r = -h; r <= h; ++r)
    for (int c = -h; c <= h; ++c) {
      const double v = std::exp(-(r * r + c * c) / (2.0 * sigma * sigma));
      w[size_t(r + h) * k + (c + h)] = v;
      sum += v;
    }
  for (int i = 0; i < k * k; ++i) w[i] /= sum;
}

// Returns the number of redraws (recorded in reports).
int synth_random_mask(uint64_t seed, int k, double* w) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  for (int attempt = 0;; ++attempt) {
    double sum = 0.0;
    for (int i = 0; i < k * k; ++i) {
      w[i] = dist(rng);
      sum += w[i];
    }
    if (std::abs(sum) >= 0.05) {
      for (int i = 0; i < k * k; ++i) w[i] /= sum;
      return attempt;
    }
  }
}

void synth_gradient_image(int w, int h, uint8_t* out) {
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) out[size_t(y) * w + x] = uint8_t((x + y) * 255 / (w + h - 2));
}

void synth_textured_image(int w, int h, uint8_t* out) {
  std::mt19937_64 rng(20240711);
  std::uniform_int_distribution<int> noise(-18, 18);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      double v = 120.0;
      v += 55.0 * std::sin(x / 19.0) * std::cos(y / 23.0);
      v += 35.0 * std::sin((x + 2 * y) / 7.0);
      v += ((x / 64 + y / 64) % 2 == 0) ? 25.0 : -25.0;
      v += noise(rng);
      out[size_t(y) * w + x] = uint8_t(std::clamp(v, 0.0, 255.0));
    }
}

}  // extern "C"
