// gtrk_close.h -- host-side tracking loop closure for a batch of channels (libgacq).
//
// Reference: gnssperf/tracking.py:168-275 (discriminators, second-order loop filters,
// fixed-point NCO advance, lock detector) and kernels.py:56-70 (NCO words). Every channel is
// computed in float64 with the reference's operation order, Python's round-half-even and
// floor-modulo semantics, and the C library's atan (what math.atan calls), so the states are
// bit-identical to the reference epoch after epoch (tests/test_tracking_host.py). Compiled
// with -ffp-contract=off (no FMA contraction). The O(N) correlators run on the GPU
// (gtrk_kernels.cuh); this replaces the per-channel Python and the vectorised numpy
// closure, which were the bottleneck of a batched epoch.
#pragma once
#include <cmath>
#include <cstdint>
#include <algorithm>

#include "../../include/gacq.h"

namespace gtrk {

constexpr double kL1 = 1575.42e6;                 // gnss_signal.py:34
constexpr double kChipRate = 1.023e6;             // cacode.py:19
constexpr double kLoopDamping = 0.7071067811865476;  // tracking.py:44
constexpr double kLockSmoothing = 20.0;           // tracking.py:45
constexpr int64_t kCarrierScale = int64_t(1) << 48;
constexpr int64_t kCodeScale = int64_t(1) << 42;
constexpr int64_t kCodeModulus = int64_t(1023) << 42;

inline double py_fmod(double a, double m) {  // Python float a % m, m > 0
    const double r = std::fmod(a, m);
    if (r == 0.0) return 0.0;
    return r < 0.0 ? r + m : r;
}
inline int64_t py_imod(int64_t a, int64_t m) {
    const int64_t r = a % m;
    return r < 0 ? r + m : r;
}
inline int64_t rint64(double x) { return (int64_t)std::nearbyint(x); }  // round() on a float, half-even

inline uint64_t carrier_phase_fixed(double p) {  // kernels.py:56-58
    return (uint64_t)py_imod(rint64(py_fmod(p, 1.0) * (double)kCarrierScale), kCarrierScale);
}
inline uint64_t carrier_step_fixed(double f, double fs) {  // kernels.py:61-62
    return (uint64_t)py_imod(rint64((f / fs) * (double)kCarrierScale), kCarrierScale);
}
inline uint64_t code_phase_fixed(double p) {  // kernels.py:65-66
    return (uint64_t)py_imod(rint64(py_fmod(p, 1023.0) * (double)kCodeScale), kCodeModulus);
}
inline uint64_t code_step_fixed(double rate, double fs) {  // kernels.py:69-70
    return (uint64_t)rint64((rate / fs) * (double)kCodeScale);
}

// channel-parallel loop on the OpenMP pool (persistent threads: no per-call spawn cost)
template <typename F>
inline void parallel_for(int64_t n, F&& f) {
    const int64_t grain = 1024;
    const int64_t chunks = (n + grain - 1) / grain;
#pragma omp parallel for schedule(static) if (chunks > 1)
    for (int64_t c = 0; c < chunks; ++c) f(c * grain, std::min(n, (c + 1) * grain));
}

}  // namespace gtrk
