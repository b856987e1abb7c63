// Measurement-cache helpers (host C++): the reference's FNV-1a checksum over
// the canonical entry serialisation (cache.hpp:55-70, rng.hpp:20-35), used by
// the JSON and binary cache readers/writers (paper_2111_14991_b200/cache.py).
#include <cstdint>
#include <cstdio>

#include "../../include/gridtune_cuda.h"

namespace {

inline std::uint64_t fnv_bytes(const char* s, std::uint64_t h) {
  for (; *s; ++s) {
    h ^= static_cast<unsigned char>(*s);
    h *= 0x100000001b3ULL;
  }
  return h;
}

inline std::uint64_t fnv_u64(std::uint64_t v, std::uint64_t h) {
  for (int i = 0; i < 8; ++i) {
    h ^= (v >> (8 * i)) & 0xffU;
    h *= 0x100000001b3ULL;
  }
  return h;
}

const char* const kReasons[] = {"", "compile_error", "runtime_error", "restricted"};

}  // namespace

extern "C" uint64_t gtc_cache_checksum(const uint64_t* ids, const double* values, const uint8_t* reasons, int64_t n) {
  std::uint64_t h = 0xcbf29ce484222325ULL;
  char buf[40];
  for (int64_t i = 0; i < n; ++i) {
    h = fnv_u64(ids[i], h);
    if (reasons[i] == 0) {
      std::snprintf(buf, sizeof(buf), "%.17g", values[i]);
      h = fnv_bytes(buf, h);
    } else {
      h = fnv_bytes(kReasons[reasons[i] < 4 ? reasons[i] : 2], h);
    }
  }
  return h;
}
