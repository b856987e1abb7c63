// Drop-in replacement of the reference's gridtune/portfolio.hpp
// (/root/reference/proj/include/gridtune/portfolio.hpp) with the argmax on the
// B200.  Same include-path rule as gridtune_dropin/gridtune/gp.hpp.
//
//   size_t best_candidate(AcquisitionId, const CandidateScores&,
//                         const std::vector<bool>* excluded)          portfolio.hpp:32-61
//     -> gtc_best_candidate: the masked argmax as one device pass (pruned
//        exact argmax, the reference's rule: first candidate taken
//        unconditionally, strict > so the lowest position wins ties).
//   Portfolio (portfolio.hpp:89-316): its O(1)-per-iteration bookkeeping is
//     the host mirror gridtune_b200::Portfolio (include/gridtune_b200/
//     portfolio.hpp), whose every argmax is a device pass over the caller's
//     spans; `multi` asks for all active functions in one request.
// Types (AcquisitionId, errors) are the reference's own headers.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstdlib>
#include <optional>
#include <span>
#include <utility>
#include <vector>

#include "gridtune/acquisition.hpp"
#include "gridtune/errors.hpp"
#include "gridtune_b200/portfolio.hpp"
#include "gridtune_cuda.h"

namespace gridtune {

/// portfolio.hpp:20-28 (an aggregate: run_bo brace-initialises it).
struct CandidateScores {
  std::span<const std::uint64_t> ids;  // canonical configuration indices, ascending
  std::span<const double> means;       // posterior means, standardized
  std::span<const double> stds;        // posterior standard deviations
  double best_std = 0.0;
  double lambda = 0.0;

  std::size_t size() const { return ids.size(); }
};

namespace b200dropin {

inline int device() {
  static const int dev = [] {
    const char* e = std::getenv("GRIDTUNE_B200_DEVICE");
    return e ? std::atoi(e) : 0;
  }();
  return dev;
}

// gridtune_b200 exceptions -> the reference's (errors.hpp)
template <class F>
auto translate(F&& f) -> decltype(f()) {
  try {
    return f();
  } catch (const gridtune_b200::ModelConditioningError& e) {
    throw ModelConditioningError(e.what());
  } catch (const gridtune_b200::ConfigError& e) {
    throw ConfigError(e.what());
  } catch (const gridtune_b200::SamplingError& e) {
    throw SamplingError(e.what());
  } catch (const gridtune_b200::Error& e) {
    throw Error(e.what());
  }
}

inline gridtune_b200::AcquisitionId to_b200(AcquisitionId a) {
  return static_cast<gridtune_b200::AcquisitionId>(static_cast<int>(a));
}
inline AcquisitionId from_b200(gridtune_b200::AcquisitionId a) {
  return static_cast<AcquisitionId>(static_cast<int>(a));
}

// The caller's spans as the mirror portfolio's argmax source.
class SpanSource final : public gridtune_b200::ArgmaxSource {
 public:
  explicit SpanSource(const CandidateScores& c) : c_(c) {}
  std::array<std::int64_t, 3> argmax(std::uint32_t mask, const std::vector<std::int64_t>& excluded) override {
    std::vector<std::uint8_t> ex;
    if (!excluded.empty()) {
      ex.assign(c_.size(), 0);
      for (std::int64_t p : excluded) ex[static_cast<std::size_t>(p)] = 1;
    }
    std::array<std::int64_t, 3> out{-1, -1, -1};
    for (int af = 0; af < 3; ++af) {
      if (!(mask & (1u << af))) continue;
      gridtune_b200::check(gtc_best_candidate(device(), af, c_.means.data(), c_.stds.data(),
                                              static_cast<std::int64_t>(c_.size()), c_.best_std, c_.lambda,
                                              ex.empty() ? nullptr : ex.data(), &out[af], nullptr));
    }
    return out;
  }
  std::uint64_t id_at(std::int64_t p) const override { return c_.ids[static_cast<std::size_t>(p)]; }
  std::int64_t position_of_id(std::uint64_t id) const override {
    // ids ascend (CandidateScores contract): binary search
    auto it = std::lower_bound(c_.ids.begin(), c_.ids.end(), id);
    return it != c_.ids.end() && *it == id ? static_cast<std::int64_t>(it - c_.ids.begin()) : -1;
  }
  std::size_t candidate_count() const override { return c_.size(); }

 private:
  const CandidateScores& c_;
};

}  // namespace b200dropin

/// portfolio.hpp:32-61 on the device.
inline std::size_t best_candidate(AcquisitionId af, const CandidateScores& c,
                                  const std::vector<bool>* excluded = nullptr) {
  std::vector<std::uint8_t> ex;
  if (excluded) {
    ex.resize(c.size());
    for (std::size_t i = 0; i < c.size(); ++i) ex[i] = (*excluded)[i] ? 1 : 0;
  }
  std::int64_t pos = -1;
  const int rc = gtc_best_candidate(b200dropin::device(), static_cast<std::int32_t>(af), c.means.data(),
                                    c.stds.data(), static_cast<std::int64_t>(c.size()), c.best_std, c.lambda,
                                    excluded ? ex.data() : nullptr, &pos, nullptr);
  if (rc != GTC_OK) throw Error(gtc_last_error());  // incl. "acquisition: no candidates remaining"
  return static_cast<std::size_t>(pos);
}

enum class PortfolioMode { multi, advanced_multi };

struct PortfolioConfig {
  PortfolioMode mode = PortfolioMode::advanced_multi;
  std::vector<AcquisitionId> order = {AcquisitionId::ei, AcquisitionId::poi, AcquisitionId::lcb};
  int skip_threshold = 5;
  double discount = 0.75;             // 0.65 for multi, 0.75 for advanced multi
  double required_improvement = 0.1;  // rho
};

class Portfolio {
 public:
  struct Suggestion {
    std::size_t position;
    std::uint64_t id;
    AcquisitionId by;
  };
  struct Event {
    enum class Kind { skipped, promoted };
    Kind kind;
    AcquisitionId af;
  };

  explicit Portfolio(PortfolioConfig config)
      : config_(std::move(config)), impl_(b200dropin::translate([&] { return gridtune_b200::Portfolio(mirror(config_)); })) {}

  const PortfolioConfig& config() const { return config_; }
  std::vector<AcquisitionId> active() const {
    std::vector<AcquisitionId> out;
    for (gridtune_b200::AcquisitionId a : impl_.active()) out.push_back(b200dropin::from_b200(a));
    return out;
  }
  double dos_of(AcquisitionId id) const {
    return b200dropin::translate([&] { return impl_.dos_of(b200dropin::to_b200(id)); });
  }
  std::span<const double> history_of(AcquisitionId id) const {
    return b200dropin::translate([&] { return impl_.history_of(b200dropin::to_b200(id)); });
  }
  int duplicate_count_of(AcquisitionId id) const {
    return b200dropin::translate([&] { return impl_.duplicate_count_of(b200dropin::to_b200(id)); });
  }
  std::span<const Event> events() const {
    const auto src = impl_.events();
    events_.clear();
    for (const auto& e : src)
      events_.push_back(Event{e.kind == gridtune_b200::Portfolio::Event::Kind::skipped ? Event::Kind::skipped
                                                                                        : Event::Kind::promoted,
                              b200dropin::from_b200(e.af)});
    return events_;
  }

  Suggestion suggest(const CandidateScores& candidates) {
    return b200dropin::translate([&] {
      b200dropin::SpanSource src(candidates);
      const auto s = impl_.suggest(src);
      return Suggestion{s.position, s.id, b200dropin::from_b200(s.by)};
    });
  }

  void record(AcquisitionId af, std::uint64_t candidate_id, std::optional<double> value,
              std::span<const double> valid_observations) {
    b200dropin::translate([&] { impl_.record(b200dropin::to_b200(af), candidate_id, value, valid_observations); });
  }

 private:
  static gridtune_b200::PortfolioConfig mirror(const PortfolioConfig& c) {
    gridtune_b200::PortfolioConfig m;
    m.mode = c.mode == PortfolioMode::multi ? gridtune_b200::PortfolioMode::multi
                                            : gridtune_b200::PortfolioMode::advanced_multi;
    m.order.clear();
    for (AcquisitionId a : c.order) m.order.push_back(b200dropin::to_b200(a));
    m.skip_threshold = c.skip_threshold;
    m.discount = c.discount;
    m.required_improvement = c.required_improvement;
    return m;
  }

  PortfolioConfig config_;
  gridtune_b200::Portfolio impl_;
  mutable std::vector<Event> events_;
};

}  // namespace gridtune
