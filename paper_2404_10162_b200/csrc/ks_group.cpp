// ks_group.cpp -- multi-GPU engine groups (include/ks_b200.h, "Engine groups").
//
// The reference's only parallelism is parallel_stripes (parallel.hpp:14-27):
// topk_metrics stripes independent samples over std::threads (eval.cpp:105-137).
// Configs are independent, so the B200 replacement shards a batch into
// contiguous, balanced ranges [g*B/G, (g+1)*B/G) over one engine per device,
// driven by one host thread each (every engine has its own stream, workspace
// and pinned staging).  There is no collective on the data path: each shard's
// results land directly in its slice of the caller's output arrays, so config
// order is preserved by construction.  topk_metrics' per-position counters are
// summed on the host (T + 1 integers per shard).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "ks_b200.h"
#include "ks_internal.h"

struct ks_engine_group {
    std::vector<ks_engine*> engines;
    std::vector<int32_t> devices;
    int32_t T = 0;
    ~ks_engine_group() {
        for (ks_engine* e : engines) ks_engine_destroy(e);
    }
};

namespace {

using ksb_host::set_error;

// A shard's host-predicate hook sees shard-relative config indices; the
// trampoline shifts them back to the caller's numbering.
struct HookShift {
    ks_host_pred_fn hook;
    void* user;
    int64_t offset;
    std::vector<int32_t> rows;
};

int32_t shifted_hook(void* u, int32_t position, int32_t final_step, int64_t n_rows, const int32_t* row_config,
                     const int32_t* row_prefix, int32_t vocab, int32_t* out_first_reject) {
    HookShift& h = *static_cast<HookShift*>(u);
    h.rows.assign(row_config, row_config + n_rows);
    for (auto& r : h.rows) r += static_cast<int32_t>(h.offset);
    return h.hook(h.user, position, final_step, n_rows, h.rows.data(), row_prefix, vocab, out_first_reject);
}

// Runs fn(g, lo, hi) for every non-empty balanced shard, one thread per engine;
// returns the first failing shard's status (its message is re-raised on the
// calling thread: ks_last_error is thread-local).
template <class F>
ks_status for_shards(ks_engine_group& G, int64_t B, F fn) {
    const int n = static_cast<int>(G.engines.size());
    std::vector<ks_status> st(static_cast<size_t>(n), KS_OK);
    std::vector<std::string> msg(static_cast<size_t>(n)), field(static_cast<size_t>(n));
    auto run = [&](int g) {
        const int64_t lo = B * g / n, hi = B * (g + 1) / n;
        if (hi <= lo) return;
        st[static_cast<size_t>(g)] = fn(g, lo, hi);
        if (st[static_cast<size_t>(g)]) {
            msg[static_cast<size_t>(g)] = ks_last_error();
            field[static_cast<size_t>(g)] = ks_last_error_field();
        }
    };
    if (n == 1) {
        run(0);
    } else {
        std::vector<std::thread> th;
        for (int g = 1; g < n; ++g) th.emplace_back(run, g);
        run(0);
        for (auto& t : th) t.join();
    }
    for (int g = 0; g < n; ++g)
        if (st[static_cast<size_t>(g)]) {
            const int64_t lo = B * g / n;
            return set_error(st[static_cast<size_t>(g)],
                             msg[static_cast<size_t>(g)] + " [device " + std::to_string(G.devices[(size_t)g]) +
                                 ", configs from " + std::to_string(lo) + "]",
                             field[static_cast<size_t>(g)]);
        }
    return KS_OK;
}

}  // namespace

extern "C" int32_t ks_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        (void)cudaGetLastError();
        return 0;
    }
    return n;
}

namespace {
template <class Create>
ks_status make_group(const int32_t* devices, int32_t n_devices, ks_engine_group** out, Create create) {
    *out = nullptr;
    std::vector<int32_t> devs;
    if (n_devices > 0) {
        if (!devices) return set_error(KS_ERR_PARAMETER, "null device list");
        devs.assign(devices, devices + n_devices);
    } else {
        const int n = ks_device_count();
        if (n < 1) return set_error(KS_ERR_CUDA, "no CUDA device visible");
        for (int d = 0; d < n; ++d) devs.push_back(d);
    }
    auto G = std::make_unique<ks_engine_group>();
    G->devices = devs;
    G->engines.assign(devs.size(), nullptr);
    // weights are packed and uploaded per device concurrently
    std::vector<ks_status> st(devs.size(), KS_OK);
    std::vector<std::string> msg(devs.size());
    std::vector<std::thread> th;
    for (size_t g = 0; g < devs.size(); ++g)
        th.emplace_back([&, g] {
            st[g] = create(devs[g], &G->engines[g]);
            if (st[g]) msg[g] = ks_last_error();
        });
    for (auto& t : th) t.join();
    for (size_t g = 0; g < devs.size(); ++g)
        if (st[g]) return set_error(st[g], msg[g] + " [device " + std::to_string(devs[g]) + "]");
    G->T = ks_engine_num_positions(G->engines[0]);
    *out = G.release();
    return KS_OK;
}
}  // namespace

extern "C" ks_status ks_engine_group_create_from_checkpoint(const char* path, const int32_t* devices,
                                                            int32_t n_devices, int32_t precision,
                                                            ks_engine_group** out) {
    if (!path || !out) return set_error(KS_ERR_PARAMETER, "null argument");
    return make_group(devices, n_devices, out, [&](int32_t dev, ks_engine** e) {
        return ks_engine_create_from_checkpoint(path, dev, precision, e);
    });
}

extern "C" ks_status ks_engine_group_create(const ks_model_desc* model, const int32_t* devices, int32_t n_devices,
                                            int32_t precision, ks_engine_group** out) {
    if (!model || !out) return set_error(KS_ERR_PARAMETER, "null argument");
    return make_group(devices, n_devices, out,
                      [&](int32_t dev, ks_engine** e) { return ks_engine_create(model, dev, precision, e); });
}

extern "C" void ks_engine_group_destroy(ks_engine_group* g) { delete g; }

extern "C" int32_t ks_engine_group_size(const ks_engine_group* g) {
    return g ? static_cast<int32_t>(g->engines.size()) : 0;
}

extern "C" ks_engine* ks_engine_group_engine(const ks_engine_group* g, int32_t i) {
    if (!g || i < 0 || i >= static_cast<int32_t>(g->engines.size())) return nullptr;
    return g->engines[static_cast<size_t>(i)];
}

extern "C" ks_status ks_group_beam_search_batch(ks_engine_group* G, const int32_t* tok, const int64_t* desc,
                                                int64_t B, int32_t k, const ks_pred* preds, int32_t n_preds,
                                                ks_host_pred_fn hook, void* user, int32_t* out_tok,
                                                double* out_lp, int32_t* out_count, int32_t* out_status,
                                                int32_t* out_fpred, int32_t* out_fstep) {
    if (!G) return set_error(KS_ERR_PARAMETER, "null engine group");
    if (B < 0) return set_error(KS_ERR_PARAMETER, "batch size out of range");
    if (k < 1) return set_error(KS_ERR_PARAMETER, "beam width must be >= 1");  // decoding.cpp:30-32
    if (B > 0 && (!tok || !out_tok)) return set_error(KS_ERR_PARAMETER, "null token buffer");
    const int64_t T = G->T;
    std::vector<HookShift> hs(G->engines.size());
    return for_shards(*G, B, [&](int g, int64_t lo, int64_t hi) {
        auto off = [&](auto* p, int64_t w) { return p ? p + lo * w : p; };
        HookShift& h = hs[static_cast<size_t>(g)];
        h = HookShift{hook, user, lo, {}};
        return ks_beam_search_batch_hooked(G->engines[static_cast<size_t>(g)], tok + lo * 7, off(desc, 7), hi - lo,
                                           k, preds, n_preds, hook ? shifted_hook : nullptr, hook ? &h : nullptr,
                                           out_tok + lo * k * T, off(out_lp, k), off(out_count, 1),
                                           off(out_status, 1), off(out_fpred, 1), off(out_fstep, 1));
    });
}

extern "C" ks_status ks_group_greedy_batch(ks_engine_group* G, const int32_t* tok, int64_t B, int32_t* out_tok) {
    if (!G) return set_error(KS_ERR_PARAMETER, "null engine group");
    if (B < 0) return set_error(KS_ERR_PARAMETER, "batch size out of range");
    if (B > 0 && (!tok || !out_tok)) return set_error(KS_ERR_PARAMETER, "null token buffer");
    const int64_t T = G->T;
    return for_shards(*G, B, [&](int g, int64_t lo, int64_t hi) {
        return ks_greedy_batch(G->engines[static_cast<size_t>(g)], tok + lo * 7, hi - lo, out_tok + lo * T);
    });
}

extern "C" ks_status ks_group_forward_batch(ks_engine_group* G, const int32_t* tok, const int32_t* teacher,
                                            int64_t B, double* out_dist, int32_t* out_tok, double* out_score) {
    if (!G) return set_error(KS_ERR_PARAMETER, "null engine group");
    if (B < 0) return set_error(KS_ERR_PARAMETER, "batch size out of range");
    if (B > 0 && (!tok || !out_dist)) return set_error(KS_ERR_PARAMETER, "null buffer");
    const int64_t T = G->T;
    int64_t SV = 0;
    for (int p = 0; p < T; ++p) SV += ks_engine_vocab_size(G->engines[0], p);
    return for_shards(*G, B, [&](int g, int64_t lo, int64_t hi) {
        return ks_forward_batch(G->engines[static_cast<size_t>(g)], tok + lo * 7, teacher ? teacher + lo * T : nullptr,
                                hi - lo, out_dist + lo * SV, out_tok ? out_tok + lo * T : nullptr,
                                out_score ? out_score + lo : nullptr);
    });
}

extern "C" ks_status ks_group_topk_metrics_batch(ks_engine_group* G, const int32_t* tok, const int64_t* desc,
                                                 const int32_t* truth, int64_t B, int32_t k, const ks_pred* preds,
                                                 int32_t n_preds, ks_host_pred_fn hook, void* user,
                                                 int64_t* out_pos_matches, int64_t* out_perfect) {
    if (!G) return set_error(KS_ERR_PARAMETER, "null engine group");
    if (B < 0) return set_error(KS_ERR_PARAMETER, "batch size out of range");
    if (!out_pos_matches || !out_perfect) return set_error(KS_ERR_PARAMETER, "null buffer");
    const int64_t T = G->T;
    const size_t n = G->engines.size();
    std::vector<std::vector<int64_t>> pos(n, std::vector<int64_t>(static_cast<size_t>(T), 0));
    std::vector<int64_t> perf(n, 0);
    std::vector<HookShift> hs(n);
    const ks_status st = for_shards(*G, B, [&](int g, int64_t lo, int64_t hi) {
        HookShift& h = hs[static_cast<size_t>(g)];
        h = HookShift{hook, user, lo, {}};
        return ks_topk_metrics_batch(G->engines[static_cast<size_t>(g)], tok + lo * 7, desc ? desc + lo * 7 : nullptr,
                                     truth + lo * T, hi - lo, k, preds, n_preds, hook ? shifted_hook : nullptr,
                                     hook ? &h : nullptr, pos[static_cast<size_t>(g)].data(),
                                     &perf[static_cast<size_t>(g)]);
    });
    if (st) return st;
    for (int64_t p = 0; p < T; ++p) {
        out_pos_matches[p] = 0;
        for (size_t g = 0; g < n; ++g) out_pos_matches[p] += pos[g][static_cast<size_t>(p)];
    }
    *out_perfect = 0;
    for (size_t g = 0; g < n; ++g) *out_perfect += perf[g];
    return KS_OK;
}

extern "C" ks_status ks_group_topk_metrics_multi(ks_engine_group* G, const int32_t* tok, const int64_t* desc,
                                                 const int32_t* truth, int64_t B, const int32_t* k_values,
                                                 int32_t n_k, const ks_pred* preds, int32_t n_preds,
                                                 ks_host_pred_fn hook, void* user, int64_t* out_pos_matches,
                                                 int64_t* out_perfect) {
    if (!G) return set_error(KS_ERR_PARAMETER, "null engine group");
    if (B < 0) return set_error(KS_ERR_PARAMETER, "batch size out of range");
    if (!out_pos_matches || !out_perfect || !k_values || n_k < 1) return set_error(KS_ERR_PARAMETER, "null buffer");
    const int64_t T = G->T;
    const size_t n = G->engines.size();
    std::vector<std::vector<int64_t>> pos(n, std::vector<int64_t>(static_cast<size_t>(n_k * T), 0));
    std::vector<std::vector<int64_t>> perf(n, std::vector<int64_t>(static_cast<size_t>(n_k), 0));
    std::vector<HookShift> hs(n);
    const ks_status st = for_shards(*G, B, [&](int g, int64_t lo, int64_t hi) {
        HookShift& h = hs[static_cast<size_t>(g)];
        h = HookShift{hook, user, lo, {}};
        return ks_topk_metrics_multi(G->engines[static_cast<size_t>(g)], tok + lo * 7, desc ? desc + lo * 7 : nullptr,
                                     truth + lo * T, hi - lo, k_values, n_k, preds, n_preds,
                                     hook ? shifted_hook : nullptr, hook ? &h : nullptr,
                                     pos[static_cast<size_t>(g)].data(), perf[static_cast<size_t>(g)].data());
    });
    if (st) return st;
    for (int64_t i = 0; i < (int64_t)n_k * T; ++i) {
        out_pos_matches[i] = 0;
        for (size_t g = 0; g < n; ++g) out_pos_matches[i] += pos[g][static_cast<size_t>(i)];
    }
    for (int i = 0; i < n_k; ++i) {
        out_perfect[i] = 0;
        for (size_t g = 0; g < n; ++g) out_perfect[i] += perf[g][static_cast<size_t>(i)];
    }
    return KS_OK;
}
