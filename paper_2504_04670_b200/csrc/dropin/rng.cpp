// rng.cpp — host side of the drop-in random streams. The arithmetic
// (splitmix64, xoshiro256**, Rng::derive, Philox4x32-10, bounded() via the
// reciprocal) is the same hgs_rng.cuh code the kernels use, so host and
// device draws are identical by construction.
#include <algorithm>
#include <cmath>
#include <numbers>

#include "../hgs_rng.cuh"
#include "hitgnn/core.hpp"

namespace hitgnn {

namespace {

std::uint64_t bounded_from(hgs::Xoshiro256& x, std::uint64_t n) {
    const std::uint64_t rc = hgs::recip_of(n);
    for (;;) {
        const std::uint64_t v = x.next();
        if (!hgs::rejected(v, n, rc)) return hgs::mod_by_recip(v, n, rc);
    }
}

// Partial Fisher-Yates over [0, n) touching only k slots (rng.cpp:105-119
// semantics); draw(i, m) yields bounded(m) for step i.
template <class Draw>
std::vector<std::uint32_t> choose_virtual(std::uint32_t n, std::uint32_t k, Draw&& draw) {
    if (k > n) k = n;
    std::vector<std::uint32_t> slot(k);
    std::vector<std::pair<std::uint32_t, std::uint32_t>> moved;  // (position >= k, value)
    for (std::uint32_t i = 0; i < k; ++i) slot[i] = i;
    for (std::uint32_t i = 0; i < k; ++i) {
        const std::uint32_t j = i + static_cast<std::uint32_t>(draw(i, static_cast<std::uint64_t>(n - i)));
        const std::uint32_t vi = slot[i];
        if (j < k) {
            slot[i] = slot[j];
            slot[j] = vi;
            continue;
        }
        auto it = std::find_if(moved.begin(), moved.end(), [&](auto& p) { return p.first == j; });
        if (it == moved.end()) {
            slot[i] = j;
            moved.emplace_back(j, vi);
        } else {
            slot[i] = it->second;
            it->second = vi;
        }
    }
    std::sort(slot.begin(), slot.end());
    return slot;
}

}  // namespace

Rng::Rng(std::uint64_t seed) {
    hgs::Xoshiro256 x;
    x.seed(seed);
    s_[0] = x.a; s_[1] = x.b; s_[2] = x.c; s_[3] = x.d;
}

std::uint64_t Rng::next_u64() {
    hgs::Xoshiro256 x{s_[0], s_[1], s_[2], s_[3]};
    const std::uint64_t v = x.next();
    s_[0] = x.a; s_[1] = x.b; s_[2] = x.c; s_[3] = x.d;
    return v;
}

std::uint64_t Rng::bounded(std::uint64_t n) {
    hgs::Xoshiro256 x{s_[0], s_[1], s_[2], s_[3]};
    const std::uint64_t v = bounded_from(x, n);
    s_[0] = x.a; s_[1] = x.b; s_[2] = x.c; s_[3] = x.d;
    return v;
}

double Rng::uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
double Rng::uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }

double Rng::normal() {  // Box-Muller, second variate cached (rng.cpp:60-74)
    if (has_spare_) {
        has_spare_ = false;
        return spare_;
    }
    double u1;
    do u1 = uniform(); while (u1 <= 0.0);
    const double u2 = uniform();
    const double mag = std::sqrt(-2.0 * std::log(u1));
    spare_ = mag * std::sin(2.0 * std::numbers::pi * u2);
    has_spare_ = true;
    return mag * std::cos(2.0 * std::numbers::pi * u2);
}

std::uint64_t Rng::derive(std::uint64_t seed, std::initializer_list<std::uint64_t> path) {
    return hgs::derive_seed(seed, path.begin(), static_cast<int>(path.size()));
}

std::vector<std::uint32_t> RandomChoiceSource::choose(std::uint32_t n, std::uint32_t k) {
    return choose_virtual(n, k, [&](std::uint32_t, std::uint64_t m) { return rng_.bounded(m); });
}

// ---- PerRootChoiceSource ----------------------------------------------------------

PerRootChoiceSource::PerRootChoiceSource(std::vector<std::uint64_t> stream_seeds)
    : seeds_(std::move(stream_seeds)), pending_(seeds_.size(), 0) {
    streams_.reserve(seeds_.size());
    for (std::uint64_t s : seeds_) streams_.emplace_back(s);
}

void PerRootChoiceSource::begin_root(std::uint64_t r) {
    if (r >= streams_.size()) fail_invalid("PerRootChoiceSource: root ordinal out of range");
    current_ = r;
}

void PerRootChoiceSource::settle(std::size_t r) {
    for (; pending_[r] > 0; --pending_[r]) streams_[r].rng().next_u64();
}

std::vector<std::uint32_t> PerRootChoiceSource::choose(std::uint32_t n, std::uint32_t k) {
    if (streams_.empty()) fail_invalid("PerRootChoiceSource: no streams configured");
    fresh_ = false;
    settle(current_);
    return streams_[current_].choose(n, k);
}

std::vector<std::uint64_t> PerRootChoiceSource::states() {
    std::vector<std::uint64_t> out(4 * streams_.size());
    for (std::size_t r = 0; r < streams_.size(); ++r) {
        settle(r);
        std::copy(streams_[r].rng().state(), streams_[r].rng().state() + 4, out.begin() + 4 * r);
    }
    return out;
}

void PerRootChoiceSource::advance(std::span<const std::uint32_t> draws) {
    for (std::size_t r = 0; r < draws.size() && r < pending_.size(); ++r) {
        pending_[r] += draws[r];
        if (draws[r]) fresh_ = false;
    }
}

// ---- PhiloxChoiceSource ---------------------------------------------------------------

PhiloxChoiceSource::PhiloxChoiceSource(std::vector<std::uint64_t> stream_seeds)
    : seeds_(std::move(stream_seeds)), decisions_(seeds_.size(), 0) {}

void PhiloxChoiceSource::begin_root(std::uint64_t r) {
    if (r >= seeds_.size()) fail_invalid("PhiloxChoiceSource: root ordinal out of range");
    current_ = r;
}

std::vector<std::uint32_t> PhiloxChoiceSource::choose(std::uint32_t n, std::uint32_t k) {
    if (seeds_.empty()) fail_invalid("PhiloxChoiceSource: no streams configured");
    fresh_ = false;
    const std::uint64_t seed = seeds_[current_];
    const std::uint32_t dec = static_cast<std::uint32_t>(decisions_[current_]++);
    return choose_virtual(n, k, [&](std::uint32_t step, std::uint64_t m) {
        const std::uint64_t rc = hgs::recip_of(m);
        for (std::uint32_t att = 0;; ++att) {
            const std::uint64_t v = hgs::philox_draw(seed, dec, step, att);
            if (!hgs::rejected(v, m, rc)) return hgs::mod_by_recip(v, m, rc);
        }
    });
}

void PhiloxChoiceSource::advance(std::span<const std::uint32_t> decisions) {
    for (std::size_t r = 0; r < decisions.size() && r < decisions_.size(); ++r) {
        decisions_[r] += decisions[r];
        if (decisions[r]) fresh_ = false;
    }
}

}  // namespace hitgnn
