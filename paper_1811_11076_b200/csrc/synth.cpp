// Seeded synthetic inputs for the five BASELINE.json configurations (host side).
//
// BASELINE.json names no public dataset; these generators produce series with the configs'
// shapes and value distributions.  Every choice the config text leaves open is
// fixed here and documented in DESIGN.md §6:
//  * RNG: one std::mt19937_64 per series, seeded with a splitmix64 mix of
//    (seed, config, part, series) -- the same construction as the reference's mix_seed
//    (rng.hpp:11-21) -- so generation is schedule-free and multi-threaded.  Normals use
//    Box-Muller (rng.hpp:40-54 style); outputs are generated once per process and fed to both
//    the GPU and the CPU oracle, so libm differences across hosts cannot break parity.
//  * random walk: x_0 ~ N(0,1), x_t = x_{t-1} + N(0,1) (+ slope, config 5), per dimension,
//    then per-dimension z-normalisation with the population SD (znormalize,
//    lower_bounds.cpp:81-103; zero variance -> 0).
//  * config 5 drift: slope ~ U(-0.01, 0.01) per series and per dimension.
//  * config 3: 20 prototypes (2-D random walks of length 256, Gaussian-smoothed with sigma = 4
//    samples, kernel truncated at +-4 sigma and renormalised at the edges; the prototype
//    stream does not depend on `part`, so database and queries share classes).  A member
//    resamples its prototype through a monotone piecewise-linear warp with 6 interior knots
//    at k(L-1)/7 displaced by U(-0.1, 0.1) L, clamped to [0, L-1] and re-sorted (endpoints
//    pinned), adds N(0, 0.05^2) noise and is z-normalised.  Series i has label i mod 20.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <thread>
#include <vector>

#include "../../include/tswarp_b200.h"

namespace {

struct Cfg {
    uint64_t n, len, d, r, k, q;
};

// index 1..5 = BASELINE.json configs[0..4]
const Cfg kCfg[6] = {
    {0, 0, 0, 0, 0, 0},
    {2000, 128, 2, 13, 1, 16},
    {20000, 128, 3, 13, 1, 64},
    {50000, 256, 2, 26, 5, 256},
    {100000, 256, 16, 26, 1, 32},
    {200000, 1024, 3, 51, 10, 32},
};

uint64_t mix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

uint64_t stream_seed(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
    return mix(mix(mix(mix(seed) ^ a) ^ b) ^ c);
}

class Rng {
public:
    explicit Rng(uint64_t s) : e_(s) {}
    double uniform() { return (double)(e_() >> 11) * 0x1.0p-53; }
    double uniform(double a, double b) { return a + (b - a) * uniform(); }
    double normal() {
        if (has_) {
            has_ = false;
            return spare_;
        }
        const double u1 = ((double)(e_() >> 11) + 0.5) * 0x1.0p-53;
        const double u2 = uniform();
        const double mag = std::sqrt(-2.0 * std::log(u1));
        const double ang = 6.283185307179586476925286766559 * u2;
        spare_ = mag * std::sin(ang);
        has_ = true;
        return mag * std::cos(ang);
    }

private:
    std::mt19937_64 e_;
    double spare_ = 0.0;
    bool has_ = false;
};

// per-dimension z-normalisation of one row-major series, population SD (lower_bounds.cpp:81-103)
void znorm(double* x, uint64_t L, uint64_t d) {
    for (uint64_t j = 0; j < d; ++j) {
        double mean = 0.0;
        for (uint64_t i = 0; i < L; ++i) mean += x[i * d + j];
        mean /= (double)L;
        double var = 0.0;
        for (uint64_t i = 0; i < L; ++i) {
            const double e = x[i * d + j] - mean;
            var += e * e;
        }
        var /= (double)L;
        const double sd = std::sqrt(var);
        for (uint64_t i = 0; i < L; ++i) x[i * d + j] = sd > 0.0 ? (x[i * d + j] - mean) / sd : 0.0;
    }
}

void random_walk(Rng& g, double* x, uint64_t L, uint64_t d, bool drift) {
    std::vector<double> slope(d, 0.0);
    if (drift)
        for (uint64_t j = 0; j < d; ++j) slope[j] = g.uniform(-0.01, 0.01);
    for (uint64_t j = 0; j < d; ++j) {
        double v = g.normal();
        x[j] = v;
        for (uint64_t t = 1; t < L; ++t) {
            v = v + g.normal() + slope[j];
            x[t * d + j] = v;
        }
    }
}

constexpr uint64_t kClasses = 20;

std::vector<double> prototypes(uint64_t seed, uint64_t L, uint64_t d) {
    std::vector<double> protos(kClasses * L * d);
    const int half = 16;  // 4 sigma
    std::vector<double> w(2 * half + 1);
    for (int o = -half; o <= half; ++o) w[o + half] = std::exp(-0.5 * (o / 4.0) * (o / 4.0));
    std::vector<double> raw(L * d);
    for (uint64_t c = 0; c < kClasses; ++c) {
        Rng g(stream_seed(seed, 3, 0x70726f746fULL, c));
        random_walk(g, raw.data(), L, d, false);
        double* out = protos.data() + c * L * d;
        for (uint64_t i = 0; i < L; ++i)
            for (uint64_t j = 0; j < d; ++j) {
                double acc = 0.0, ws = 0.0;
                for (int o = -half; o <= half; ++o) {
                    const int64_t p = (int64_t)i + o;
                    if (p < 0 || p >= (int64_t)L) continue;
                    acc += raw[p * d + j] * w[o + half];
                    ws += w[o + half];
                }
                out[i * d + j] = acc / ws;
            }
    }
    return protos;
}

void class_member(Rng& g, const double* proto, double* x, uint64_t L, uint64_t d) {
    double kx[8], ky[8];
    kx[0] = ky[0] = 0.0;
    kx[7] = ky[7] = (double)(L - 1);
    for (int k = 1; k <= 6; ++k) {
        kx[k] = k * (double)(L - 1) / 7.0;
        ky[k] = std::clamp(kx[k] + g.uniform(-0.1, 0.1) * (double)L, 0.0, (double)(L - 1));
    }
    std::sort(ky + 1, ky + 7);
    int seg = 0;
    for (uint64_t i = 0; i < L; ++i) {
        const double t = (double)i;
        while (seg < 6 && t > kx[seg + 1]) ++seg;
        const double f = (t - kx[seg]) / (kx[seg + 1] - kx[seg]);
        const double pos = std::clamp(ky[seg] + f * (ky[seg + 1] - ky[seg]), 0.0, (double)(L - 1));
        const uint64_t i0 = std::min<uint64_t>((uint64_t)pos, L - 1);
        const uint64_t i1 = std::min<uint64_t>(i0 + 1, L - 1);
        const double fr = pos - (double)i0;
        for (uint64_t j = 0; j < d; ++j)
            x[i * d + j] = proto[i0 * d + j] + fr * (proto[i1 * d + j] - proto[i0 * d + j]);
    }
    for (uint64_t v = 0; v < L * d; ++v) x[v] += 0.05 * g.normal();
}

}  // namespace

extern "C" int tsw_synth_shape(int config, int part, uint64_t* count, uint64_t* len, uint64_t* d,
                               uint64_t* r, uint64_t* k) {
    if (config < 1 || config > 5 || part < 0 || part > 1) return TSW_EINVAL;
    const Cfg& c = kCfg[config];
    if (count) *count = part == 0 ? c.n : c.q;
    if (len) *len = c.len;
    if (d) *d = c.d;
    if (r) *r = c.r;
    if (k) *k = c.k;
    return TSW_OK;
}

extern "C" int tsw_synth_generate(int config, int part, uint64_t seed, double* out, int32_t* labels) {
    if (config < 1 || config > 5 || part < 0 || part > 1 || !out) return TSW_EINVAL;
    const Cfg& c = kCfg[config];
    const uint64_t count = part == 0 ? c.n : c.q, L = c.len, d = c.d;
    std::vector<double> protos;
    if (config == 3) protos = prototypes(seed, L, d);
    const unsigned hw = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    auto work = [&](uint64_t lo, uint64_t hi) {
        for (uint64_t i = lo; i < hi; ++i) {
            Rng g(stream_seed(seed, (uint64_t)config, (uint64_t)part, i));
            double* x = out + i * L * d;
            if (config == 3) class_member(g, protos.data() + (i % kClasses) * L * d, x, L, d);
            else random_walk(g, x, L, d, config == 5);
            znorm(x, L, d);
            if (labels) labels[i] = config == 3 ? (int32_t)(i % kClasses) : 0;
        }
    };
    std::vector<std::thread> pool;
    const uint64_t per = (count + hw - 1) / hw;
    for (unsigned t = 0; t < hw; ++t) {
        const uint64_t lo = t * per, hi = std::min(count, lo + per);
        if (lo < hi) pool.emplace_back(work, lo, hi);
    }
    for (auto& th : pool) th.join();
    return TSW_OK;
}
