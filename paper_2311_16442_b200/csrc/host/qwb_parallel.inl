// qwb_parallel.inl -- tiny std::thread fan-out used by the host producer.
#pragma once

#include <algorithm>
#include <exception>
#include <thread>
#include <vector>

namespace qwb {

template <class F>
void parallel_for(uint64_t n, unsigned threads, F&& fn) {
  if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
  if (n == 0) return;
  const uint64_t parts = std::min<uint64_t>(threads, n);
  if (parts <= 1) {
    fn((uint64_t)0, n);
    return;
  }
  std::vector<std::exception_ptr> err(parts);
  std::vector<std::thread> pool;
  pool.reserve(parts - 1);
  auto run = [&](uint64_t p) {
    try {
      fn(n * p / parts, n * (p + 1) / parts);
    } catch (...) {
      err[p] = std::current_exception();
    }
  };
  for (uint64_t p = 1; p < parts; ++p) pool.emplace_back(run, p);
  run(0);
  for (auto& t : pool) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

}  // namespace qwb
