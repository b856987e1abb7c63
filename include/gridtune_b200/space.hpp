// Enumerated search space on the host + its HBM-resident copy.
//
// Mirrors EnumeratedSpace (search_space.hpp:216-245): valid configurations in
// ascending canonical index, their rank-normalised coordinates
// (SearchSpace::normalize, search_space.hpp:158-166), and position_of().
// Restriction parsing/enumeration stays with the caller (out of scope for the
// hot path): construct from the reference's EnumeratedSpace (ids + coords) or
// from a Cartesian grid.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "gridtune_b200/errors.hpp"

namespace gridtune_b200 {

using ConfigIndex = std::uint64_t;

struct Configuration {
  ConfigIndex index = 0;
  std::size_t position = 0;
};

class EnumeratedSpace {
 public:
  static constexpr std::size_t npos = static_cast<std::size_t>(-1);

  /// ids: canonical indices (strictly ascending); coords: size() x d row-major.
  EnumeratedSpace(std::vector<ConfigIndex> ids, std::vector<double> coords, std::size_t d,
                  int device = 0)
      : ids_(std::move(ids)), coords_(std::move(coords)), d_(d), device_(device) {
    if (ids_.empty()) throw Error("search space has no configurations");
    if (coords_.size() != ids_.size() * d_) throw Error("coords size does not match ids x d");
    for (std::size_t i = 1; i < ids_.size(); ++i)
      if (!(ids_[i - 1] < ids_[i])) throw Error("canonical indices must be strictly ascending");
  }

  /// Host view over an existing resident space (non-owning; `ids` copied).
  EnumeratedSpace(gtc_space* resident, const std::uint64_t* ids)
      : ids_(ids, ids + gtc_space_size(resident)),
        coords_(gtc_space_coords(resident),
                gtc_space_coords(resident) + gtc_space_size(resident) * gtc_space_dimension(resident)),
        d_(static_cast<std::size_t>(gtc_space_dimension(resident))),
        device_(gtc_space_device(resident)) {
    dev_.reset(resident, [](gtc_space*) {});
  }

  /// Unrestricted Cartesian grid with `sizes[j]` values per parameter
  /// (first parameter most significant, search_space.hpp:57-72).
  static EnumeratedSpace grid(const std::vector<std::size_t>& sizes, int device = 0) {
    std::uint64_t total = 1;
    for (std::size_t k : sizes) total *= k;
    const std::size_t d = sizes.size();
    std::vector<ConfigIndex> ids(total);
    std::vector<double> coords(total * d);
    std::vector<std::size_t> ranks(d, 0);
    for (std::uint64_t idx = 0; idx < total; ++idx) {
      ids[idx] = idx;
      for (std::size_t j = 0; j < d; ++j)
        coords[idx * d + j] =
            sizes[j] <= 1 ? 0.0 : static_cast<double>(ranks[j]) / static_cast<double>(sizes[j] - 1);
      for (std::size_t j = d; j-- > 0;) {
        if (++ranks[j] < sizes[j]) break;
        ranks[j] = 0;
      }
    }
    return EnumeratedSpace(std::move(ids), std::move(coords), d, device);
  }

  std::size_t size() const { return ids_.size(); }
  std::size_t dimension() const { return d_; }
  int device() const { return device_; }
  ConfigIndex id(std::size_t pos) const { return ids_[pos]; }
  const double* coords(std::size_t pos) const { return &coords_[pos * d_]; }
  const std::vector<double>& coords_row_major() const { return coords_; }
  const std::vector<ConfigIndex>& ids() const { return ids_; }
  Configuration config(std::size_t pos) const { return Configuration{ids_[pos], pos}; }

  std::size_t position_of(ConfigIndex index) const {
    std::size_t lo = 0, hi = ids_.size();
    while (lo < hi) {
      const std::size_t mid = (lo + hi) / 2;
      if (ids_[mid] < index) lo = mid + 1;
      else hi = mid;
    }
    return lo < ids_.size() && ids_[lo] == index ? lo : npos;
  }

  /// The HBM-resident copy (created on first use, shared by all runs).
  gtc_space* device_space() const {
    if (!dev_) {
      gtc_space* s = nullptr;
      check(gtc_space_create(device_, coords_.data(), static_cast<std::int64_t>(size()),
                             static_cast<std::int32_t>(d_), &s));
      dev_.reset(s, [](gtc_space* p) { gtc_space_destroy(p); });
    }
    return dev_.get();
  }

 private:
  std::vector<ConfigIndex> ids_;
  std::vector<double> coords_;
  std::size_t d_;
  int device_;
  mutable std::shared_ptr<gtc_space> dev_;
};

}  // namespace gridtune_b200
