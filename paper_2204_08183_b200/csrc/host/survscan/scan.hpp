// survscan/scan.hpp — execution-geometry types of the reference API
// (/root/reference/proj/include/survscan/scan.hpp:22-46, :123-126).  The
// device engine accepts a ChunkPlan for source compatibility and validates it
// exactly like the reference; its own tiling (2048-row tiles, one persistent
// CTA per SM) does not depend on it.
#pragma once

#include <cstddef>
#include <limits>
#include <thread>

#include "survscan/errors.hpp"

namespace survscan {

struct ChunkPlan {
  std::size_t chunk_size = 65536;
  unsigned worker_count = default_workers();

  static unsigned default_workers() {
    const unsigned h = std::thread::hardware_concurrency();
    return h ? h : 1;
  }
  static ChunkPlan serial() { return ChunkPlan{std::numeric_limits<std::size_t>::max(), 1}; }
  std::size_t chunks_for(std::size_t n) const {
    validate();
    if (n == 0) return 0;
    return 1 + (n - 1) / chunk_size;
  }
  void validate() const {
    if (chunk_size == 0) throw DomainError("ChunkPlan: chunk_size must be >= 1");
    if (worker_count == 0) throw DomainError("ChunkPlan: worker_count must be >= 1");
  }
};

// raw sums behind one coordinate's derivatives (scan.hpp:123-126)
struct GradHessSums {
  double grad_sum = 0.0;
  double hess_sum = 0.0;
};

}  // namespace survscan
