// ks_synth.cpp -- synthetic problem descriptors for benchmarks and parity runs
// (BASELINE.md §3 step 3).  Config i of a workload draws each
// input field uniformly WITH replacement from the model's input vocabulary, in
// field order n,c,h,w,k,y,x, one Rng::uniform_int per field, from its own
// stream Rng::derive(seed, i) (proj/include/kernelseer/rng.hpp:19-21, 35-43;
// the reference's grids hold only 46,656 unique points, data.cpp:355-368, so
// 64k / 1M workloads resample).  Per-config streams make any slice
// [start, start + count) reproducible on its own: the shards of a multi-GPU
// run draw exactly the configs a single-GPU run would.
#include <algorithm>
#include <cstdint>
#include <random>
#include <thread>
#include <vector>

#include "ks_b200.h"
#include "ks_internal.h"

namespace {

// Rng (rng.hpp:13-71): mt19937_64 seeded through the SplitMix-style mix.
std::uint64_t mix(std::uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

std::uint64_t uniform_int(std::mt19937_64& e, std::uint64_t n) {
    const std::uint64_t limit = UINT64_MAX - UINT64_MAX % n;  // rejection: unbiased
    std::uint64_t v;
    do {
        v = e();
    } while (v >= limit);
    return v % n;
}

}  // namespace

extern "C" ks_status ks_synthetic_descriptors(const int32_t* input_sizes, const int64_t* input_values,
                                              uint64_t seed, int64_t start, int64_t count,
                                              int64_t* out_desc) {
    if (!input_sizes || !input_values || (count > 0 && !out_desc))
        return ksb_host::set_error(KS_ERR_PARAMETER, "null argument");
    if (start < 0 || count < 0) return ksb_host::set_error(KS_ERR_PARAMETER, "negative start / count");
    int64_t off[7];
    int64_t o = 0;
    for (int f = 0; f < 7; ++f) {
        if (input_sizes[f] < 1)
            return ksb_host::set_error(KS_ERR_PARAMETER, "empty input vocabulary field");
        off[f] = o;
        o += input_sizes[f];
    }
    auto run = [&](int64_t lo, int64_t hi) {
        for (int64_t i = lo; i < hi; ++i) {
            const std::uint64_t stream = (std::uint64_t)(start + i);
            std::mt19937_64 e(mix(mix(seed) + 0x9e3779b97f4a7c15ULL * (stream + 1)));
            for (int f = 0; f < 7; ++f)
                out_desc[i * 7 + f] = input_values[off[f] + (int64_t)uniform_int(e, (std::uint64_t)input_sizes[f])];
        }
    };
    // ~3 us per config (one mt19937_64 seeding and twist each): host threads for 1M-config workloads
    const int64_t per = 1 << 14;
    const int nt = (int)std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()), (count + per - 1) / per);
    if (nt <= 1) {
        run(0, count);
    } else {
        std::vector<std::thread> th;
        for (int t = 0; t < nt; ++t)
            th.emplace_back(run, count * t / nt, count * (t + 1) / nt);
        for (auto& t : th) t.join();
    }
    return KS_OK;
}
