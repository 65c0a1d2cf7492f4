#pragma once
// Drop-in for proj/include/d4orm/parallel.hpp:12-45 — the reference's host
// fan-out helper, kept for callers that include it (its own sources use it for
// the per-sample loops, which run on the GPU here).
//
//   resolve_workers(w)        w > 0 → w, else the hardware concurrency (≥ 1)
//   parallel_for(n, w, fn)    fn(i) for every i in [0, n) on up to w threads;
//                             fn(i) may only touch state owned by index i, so
//                             results never depend on the worker count; if any
//                             fn(i) throws, the others still finish and one
//                             exception is rethrown to the caller.
//
// Indices are handed out by an atomic counter rather than a fixed stride; the
// exception rethrown is the one of the lowest failing index (the reference
// keeps whichever it caught first, so this is one of its possible outcomes,
// made deterministic).
#include <algorithm>
#include <atomic>
#include <exception>
#include <thread>
#include <vector>

namespace d4orm {

inline int resolve_workers(int workers) {
  if (workers > 0) return workers;
  const unsigned hw = std::thread::hardware_concurrency();
  return hw > 0 ? static_cast<int>(hw) : 1;
}

template <class Fn>
void parallel_for(int count, int workers, Fn&& fn) {
  if (count <= 0) return;
  const int nthreads = std::min(resolve_workers(workers), count);
  std::vector<std::exception_ptr> errors(static_cast<std::size_t>(count));
  std::atomic<int> next{0};
  auto drain = [&] {
    for (int i = next.fetch_add(1, std::memory_order_relaxed); i < count;
         i = next.fetch_add(1, std::memory_order_relaxed)) {
      try {
        fn(i);
      } catch (...) {
        errors[static_cast<std::size_t>(i)] = std::current_exception();
      }
    }
  };
  if (nthreads <= 1) {
    drain();
  } else {
    std::vector<std::thread> helpers;
    helpers.reserve(static_cast<std::size_t>(nthreads - 1));
    for (int t = 1; t < nthreads; ++t) helpers.emplace_back(drain);
    drain();
    for (auto& h : helpers) h.join();
  }
  for (auto& e : errors)
    if (e) std::rethrow_exception(e);
}

}  // namespace d4orm
