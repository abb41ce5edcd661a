// shim_gpu.cpp -- TEST INFRASTRUCTURE: the reference-side C++ binding
// (include/qweight_b200.hpp) on a B200, driven exactly as a reference user
// would: the reference's own synth + quantize_layer (synth.cpp,
// quantizer.cpp) produce a PackedLayer, qweight::b200 computes, and the
// reference's own reconstruct_dense / matvec_reference_f64 (engine.cpp:151-167,
// 251-270) check it.  Built by oracle/Makefile against the reference's
// headers and libqweight_ref.so (oracle/_ref/shim_gpu); run by
// tests/test_shim_gpu.py.  Prints one "key value" per line; exit 0 = pass.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "qweight/container.hpp"
#include "qweight/engine.hpp"
#include "qweight/quantizer.hpp"
#include "qweight/synth.hpp"
#include "qweight_b200.hpp"

static double rel_l2(const std::vector<float>& y, const std::vector<double>& ref, double* maxabs, double* refmax) {
  double num = 0, den = 0, mx = 0, rm = 0;
  for (size_t i = 0; i < y.size(); ++i) {
    const double d = (double)y[i] - ref[i];
    num += d * d, den += ref[i] * ref[i];
    mx = std::max(mx, std::fabs(d)), rm = std::max(rm, std::fabs(ref[i]));
  }
  *maxabs = mx, *refmax = rm;
  return std::sqrt(num / (den > 0 ? den : 1));
}

int main(int argc, char** argv) {
  const uint32_t rows = argc > 1 ? (uint32_t)std::atoi(argv[1]) : 1024;
  const uint32_t cols = argc > 2 ? (uint32_t)std::atoi(argv[2]) : 4096;
  int fails = 0;
  auto expect = [&](bool ok, const char* what) {
    if (!ok) std::printf("FAIL %s\n", what), ++fails;
  };
  const auto W = qweight::synth_gaussian(rows, cols, 7);
  const auto H = qweight::synth_calibration(cols, 7);
  const qweight::PackedLayer L = qweight::quantize_layer(W, H, qweight::QuantizeParams{});
  const auto x = qweight::synth_activation(cols, 8);
  const auto ref = qweight::matvec_reference_f64(L, x);

  qweight::b200::DeviceLayer dev(L);
  const qweight::MatvecResult r = dev.matvec(x);
  double mx = 0, rm = 0;
  const double err = rel_l2(r.y, ref, &mx, &rm);
  std::printf("rel_l2 %.3e\nmaxabs_over_max %.3e\nstage_ns %llu %llu %llu %llu\nwall_ns %llu\n", err, mx / rm,
              (unsigned long long)r.stage_ns[0], (unsigned long long)r.stage_ns[1],
              (unsigned long long)r.stage_ns[2], (unsigned long long)r.stage_ns[3], (unsigned long long)r.wall_ns);
  expect(err <= 1e-2 && mx <= 1e-2 * rm, "matvec within 1e-2 of matvec_reference_f64");
  expect(r.stage_ns[3] > 0, "kernel time reported in stage_ns[3]");

  // reconstruct_dense: bit for bit with the reference's
  const qweight::WeightMatrix w = dev.reconstruct_dense(), rw = qweight::reconstruct_dense(L);
  expect(w.rows == rw.rows && w.cols == rw.cols && w.data.size() == rw.data.size() &&
             std::memcmp(w.data.data(), rw.data.data(), w.data.size() * 4) == 0,
         "reconstruct_dense bit-exact");

  // free functions with the reference's signatures (upload per call)
  const auto t0 = std::chrono::steady_clock::now();
  const qweight::MatvecResult rp = qweight::b200::matvec_pipelined(L, x, 4);
  const double free_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  const double err2 = rel_l2(rp.y, ref, &mx, &rm);
  expect(err2 <= 1e-2, "matvec_pipelined within 1e-2");
  const auto t1 = std::chrono::steady_clock::now();
  const int reps = 50;
  for (int i = 0; i < reps; ++i) (void)dev.matvec(x);
  const double held_us =
      std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t1).count() / reps;
  std::printf("free_function_us_per_call %.1f\nheld_device_layer_us_per_call %.1f\n", free_us, held_us);

  // errors as the reference (engine.cpp:126-130, 187-188)
  bool threw = false;
  try {
    (void)qweight::b200::matvec_pipelined(L, x, 0);
  } catch (const qweight::Error&) {
    threw = true;
  }
  expect(threw, "workers == 0 throws qweight::Error");
  threw = false;
  try {
    std::vector<float> bad(x.begin(), x.end() - 1);
    (void)dev.matvec(bad);
  } catch (const qweight::Error&) {
    threw = true;
  }
  expect(threw, "wrong x length throws qweight::Error");
  threw = false;
  try {
    std::vector<float> bad(x);
    bad[3] = NAN;
    (void)dev.matvec(bad);
  } catch (const qweight::Error&) {
    threw = true;
  }
  expect(threw, "non-finite x throws qweight::Error");

  // bench_matvec -> the reference's own BenchReport + CSV (engine.cpp:286-315)
  const qweight::BenchReport rep = qweight::b200::bench_matvec(dev, L, x, 20, 1);
  std::printf("bench_gflops_kernel %.2f\nbench_gflops_host %.2f\n", rep.gflops(rep.oracle_wall_ns),
              rep.gflops(rep.pipelined_wall_ns));
  std::printf("%s", rep.to_csv().c_str());
  expect(rep.bytes_touched == qweight::payload_bytes(L) + 4ull * (cols + rows), "bytes_touched as the reference");
  std::printf("fails %d\n", fails);
  return fails ? 1 : 0;
}
