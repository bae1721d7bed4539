// Config 5 through the reference's OWN Pipeline (pipeline.cpp:299-323): synth_workload
// (simgen.cpp:162-194) replayed with admit / record_reuse / evict / refine churn at the
// reference-default 1K capacity and IVF index (64 lists, nprobe 8, rebuild every 1024
// mutations). The same source is linked twice by oracle/Makefile:
//   replay_stock  the unmodified reference (IvfIndex + selector.cpp on the CPU)
//   replay_b200   the reference sources with CacheManager's IvfIndex swapped for GpuIvfIndex
//                 (semwarm_b200::IvfIndexT over the device arena) and selector.cpp replaced by
//                 tools/dropin/selector_b200.cpp (score_candidates / select on the device)
// Both print the RunReport's JSON lines (every ServeOutcome) plus the final cache ledger;
// tests/test_gpu_dropin.py requires the two outputs to be byte-identical. Timing goes to stderr.
//
//   replay_check [n_prompts=2000] [dim=512] [capacity=1024] [policy=exploit] [seed=7]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "semwarm/pipeline.hpp"
#include "semwarm/simgen.hpp"

using namespace semwarm;

int main(int argc, char** argv) {
    const size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 2000;
    const size_t dim = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 512;
    const size_t cap = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 1024;
    const std::string policy = argc > 4 ? argv[4] : "exploit";
    const uint64_t seed = argc > 5 ? std::strtoull(argv[5], nullptr, 10) : 7;

    ConfigMap cm;
    cm.set("dim", std::to_string(dim));
    cm.set("cache.capacity", std::to_string(cap));
    cm.set("gater.policy", policy);
    PipelineConfig cfg = PipelineConfig::from_config(cm);
    // a non-degenerate bandit (the zero model always picks arm 13): value heads whose argmax
    // tracks ~13 x similarity, as a trained gater does
    for (int a = 0; a < kNumArms; ++a) {
        cfg.gater.theta[(size_t)a * kFeatureDim + 0] = (float)a;
        cfg.gater.theta[(size_t)a * kFeatureDim + 10] = (float)(-a * a / 26.0);
        for (size_t i = 0; i < kFeatureDim; ++i)
            cfg.gater.psi[(size_t)a * kFeatureDim + i] = (float)((((a * 31 + i * 17) % 23) - 11) / 40.0);
    }
    cfg.fixed_arm = policy == "fixed" ? 1 : 6;  // fixed: skip 0.05 < 0.10 -> refine churn

    WorkloadConfig wc;
    wc.n_prompts = n;
    wc.dim = dim;
    wc.near_duplicate_rate = 0.9;
    auto trace = synth_workload(wc, seed);

    Pipeline pipe(cfg);
    const auto t0 = std::chrono::steady_clock::now();
    RunReport rep = pipe.replay(trace);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

    std::fputs(rep.to_json_lines().c_str(), stdout);
    const CacheManager& cache = pipe.cache();
    const double now_h = trace.back().arrival_time_s / 3600.0;
    for (const auto& [id, e] : cache.entries())
        std::printf("{\"entry\":%llu,\"importance\":%.17g,\"quality\":%.17g,\"attempts\":%d,"
                    "\"reuses\":%zu}\n",
                    (unsigned long long)id, cache.current_importance(id, now_h), e.quality,
                    e.refinement_attempts, e.reuse_count);
    std::printf("{\"size\":%zu,\"index_entries\":%zu,\"index_vectors\":%zu,\"centroids\":%zu,"
                "\"consistent\":%s}\n",
                cache.size(), cache.index().entry_count(), cache.index().total_vectors(),
                cache.index().centroid_count(), cache.check_consistent() ? "true" : "false");
    std::fprintf(stderr, "replay: %zu requests in %.3f s (%.1f requests/s), hit rate %.3f, "
                 "refinements %zu\n", n, s, n / s, rep.hit_rate, rep.refinements);
    return 0;
}
