// otdr_datagen.cpp -- host generators of the benchmark instances
// (include/otdr_datagen.h). Reference: rng.hpp:14-45, datagen.cpp:21-129.
// Built with -ffp-contract=off so the point coordinates round exactly like the
// reference's baseline-x86-64 build.
#include "otdr_datagen.h"

#include <cmath>
#include <cstring>
#include <random>
#include <vector>

namespace {

constexpr double kPi = 3.14159265358979323846;

class Stream {  // rng.hpp:14-45
 public:
  explicit Stream(uint64_t seed) : eng_(seed) {}
  double uniform() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
  double gauss() {
    if (cached_) {
      cached_ = false;
      return spare_;
    }
    const double u1 = static_cast<double>((eng_() >> 11) + 1) * 0x1.0p-53;
    const double u2 = uniform();
    const double rad = std::sqrt(-2.0 * std::log(u1));
    const double th = 2.0 * kPi * u2;
    spare_ = rad * std::sin(th);
    cached_ = true;
    return rad * std::cos(th);
  }

 private:
  std::mt19937_64 eng_;
  bool cached_ = false;
  double spare_ = 0.0;
};

// mean + L z with a seeded lower-triangular 2x2 factor (datagen.cpp:21-35).
void cloud(Stream& g, int64_t count, double* out) {
  const double mx = 2.0 * g.gauss();
  const double my = 2.0 * g.gauss();
  const double l00 = 0.6 + 0.4 * g.uniform();
  const double l10 = 0.4 * g.gauss();
  const double l11 = 0.6 + 0.4 * g.uniform();
  for (int64_t i = 0; i < count; ++i) {
    const double z0 = g.gauss();
    const double z1 = g.gauss();
    out[2 * i] = mx + l00 * z0;
    out[2 * i + 1] = my + l10 * z0 + l11 * z1;
  }
}

}  // namespace

extern "C" {

void otdr_gaussian_points(int64_t m, int64_t n, uint64_t seed, double* src, double* tgt) {
  Stream g(seed);
  cloud(g, m, src);
  cloud(g, n, tgt);
}

int otdr_adaptation_points(int64_t m, int64_t n, int classes, uint64_t seed, int identity_map,
                           double* src, double* tgt, int32_t* src_labels, int32_t* tgt_labels) {
  if (classes < 1 || m < classes || n < classes) return 5;
  Stream g(seed);
  std::vector<double> cx(static_cast<size_t>(classes)), cy(static_cast<size_t>(classes));
  for (int c = 0; c < classes; ++c) {
    const double ang = 2.0 * kPi * c / classes;
    cx[c] = 3.0 * std::cos(ang);
    cy[c] = 3.0 * std::sin(ang);
  }
  auto blobs = [&](int64_t count, double* pts, int32_t* lab) {
    int64_t at = 0;
    for (int c = 0; c < classes; ++c) {
      const int64_t share = count / classes + (c < count % classes ? 1 : 0);
      for (int64_t t = 0; t < share; ++t, ++at) {
        pts[2 * at] = cx[c] + 0.85 * g.gauss();
        pts[2 * at + 1] = cy[c] + 0.85 * g.gauss();
        lab[at] = c;
      }
    }
  };
  blobs(m, src, src_labels);
  blobs(n, tgt, tgt_labels);
  if (!identity_map) {
    const double sign = g.uniform() < 0.5 ? -1.0 : 1.0;
    const double angle = sign * (44.0 + 4.0 * g.uniform()) * kPi / 180.0;
    const double scale = 0.98 + 0.04 * g.uniform();
    const double tx = 0.2 * g.gauss();
    const double ty = 0.2 * g.gauss();
    const double ca = scale * std::cos(angle), sa = scale * std::sin(angle);
    for (int64_t j = 0; j < n; ++j) {
      const double x = tgt[2 * j], y = tgt[2 * j + 1];
      tgt[2 * j] = ca * x - sa * y + tx;
      tgt[2 * j + 1] = sa * x + ca * y + ty;
    }
  }
  return 0;
}

}  // extern "C"
