// tangram/latency.hpp -- drop-in for the reference's latency estimator
// (latency.hpp:35-144): ProfileEntry, LatencyProfile (slack = mu + 3 sigma,
// linear interpolation / extrapolation on slack values, Eq. 9) and
// profile_from_samples.  Validation messages are the reference's; slack_us
// is computed by the same routine the device batcher uses
// (tg_profile_slack_us), so scheduler decisions and this header agree.
// Profile file I/O (save_profile / load_profile, latency.hpp:146-205) is
// offline tooling and out of scope.
#pragma once

#include <algorithm>
#include <cmath>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "tangram/partition.hpp"

namespace tangram {

struct ProfileEntry {
  int batch_size = 1;
  double mu_ms = 0.0;
  double sigma_ms = 0.0;
};

class LatencyProfile {
 public:
  static LatencyProfile from_entries(int canvas_w, int canvas_h, std::vector<ProfileEntry> entries,
                                     std::vector<std::string>* warnings = nullptr) {
    std::stable_sort(entries.begin(), entries.end(), [](const ProfileEntry& a, const ProfileEntry& b) {
      return a.batch_size < b.batch_size;
    });
    LatencyProfile p;
    p.canvas_w_ = canvas_w;
    p.canvas_h_ = canvas_h;
    p.entries_ = std::move(entries);
    p.c_.reserve(p.entries_.size());
    for (const ProfileEntry& e : p.entries_) p.c_.push_back(tg_profile_entry{e.batch_size, e.mu_ms, e.sigma_ms});
    int64_t probe = 0;  // validates with the reference's messages (empty, k < 1, mu, sigma, duplicates)
    gpu::check(tg_profile_slack_us(p.c_.data(), static_cast<int32_t>(p.c_.size()), 1, &probe));
    if (warnings != nullptr)
      for (std::size_t i = 1; i < p.entries_.size(); ++i)
        if (p.entries_[i].mu_ms < p.entries_[i - 1].mu_ms)
          warnings->push_back("profile mu decreases from k=" +
                              std::to_string(p.entries_[i - 1].batch_size) +
                              " to k=" + std::to_string(p.entries_[i].batch_size));
    return p;
  }

  int canvas_width() const { return canvas_w_; }
  int canvas_height() const { return canvas_h_; }
  const std::vector<ProfileEntry>& entries() const { return entries_; }
  int max_profiled_batch() const { return entries_.back().batch_size; }

  double slack_ms(int k) const { return interp(k, [](const ProfileEntry& e) { return e.mu_ms + 3.0 * e.sigma_ms; }); }

  Micros slack_us(int k) const {
    int64_t us = 0;
    gpu::check(tg_profile_slack_us(c_.data(), static_cast<int32_t>(c_.size()), k, &us));
    return us;
  }

  double mu_ms(int k) const { return interp(k, [](const ProfileEntry& e) { return e.mu_ms; }); }
  double sigma_ms(int k) const {
    return std::max(0.0, interp(k, [](const ProfileEntry& e) { return e.sigma_ms; }));
  }

  const tg_profile_entry* c_entries() const { return c_.data(); }
  int c_count() const { return static_cast<int>(c_.size()); }

 private:
  // Piecewise-linear in k through the table, the two nearest entries
  // extending it past either end, clamped at zero.
  template <class F>
  double interp(int k, F value) const {
    if (k < 1) throw std::invalid_argument("invalid batch size");
    const std::size_t n = entries_.size();
    if (n == 1) return value(entries_[0]);
    std::size_t hi = 0;
    while (hi < n && entries_[hi].batch_size < k) ++hi;
    if (hi < n && entries_[hi].batch_size == k) return value(entries_[hi]);
    hi = std::clamp<std::size_t>(hi, 1, n - 1);
    const ProfileEntry& a = entries_[hi - 1];
    const ProfileEntry& b = entries_[hi];
    const double t = static_cast<double>(k - a.batch_size) / static_cast<double>(b.batch_size - a.batch_size);
    return std::max(0.0, value(a) + t * (value(b) - value(a)));
  }

  int canvas_w_ = 0;
  int canvas_h_ = 0;
  std::vector<ProfileEntry> entries_;
  std::vector<tg_profile_entry> c_;
};

// Population mean / standard deviation per batch size (latency.hpp:127-144).
inline LatencyProfile profile_from_samples(int canvas_w, int canvas_h,
                                           const std::map<int, std::vector<double>>& samples_ms,
                                           std::vector<std::string>* warnings = nullptr) {
  std::vector<ProfileEntry> entries;
  for (const auto& [k, s] : samples_ms) {
    if (s.empty()) throw std::invalid_argument("no samples for batch size " + std::to_string(k));
    double sum = 0.0;
    for (double x : s) sum += x;
    const double mu = sum / static_cast<double>(s.size());
    double ss = 0.0;
    for (double x : s) ss += (x - mu) * (x - mu);
    entries.push_back(ProfileEntry{k, mu, std::sqrt(ss / static_cast<double>(s.size()))});
  }
  return LatencyProfile::from_entries(canvas_w, canvas_h, std::move(entries), warnings);
}

}  // namespace tangram
