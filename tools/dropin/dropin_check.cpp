// Drop-in check: the reference's own semwarm::IvfIndex vs semwarm_b200::IvfIndexT instantiated
// with the reference's own types (semwarm::EmbeddingVector / IndexedVector / SearchHit), fed the
// same IndexedVectors from the reference's build_entry_vectors (index.cpp:48-57). Also checks
// choose_arm against the reference gater. Built against /root/reference/proj/include by
// __graft_entry__.build() (only when the reference is present) into oracle/_ref/dropin_check;
// run on the GPU box by tests/test_gpu_dropin.py. Prints "DROPIN PASS" on success.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "semwarm/core.hpp"
#include "semwarm/gater.hpp"
#include "semwarm/index.hpp"
#include "semwarm_b200.hpp"

using namespace semwarm;

int main(int argc, char** argv) {
    const int dim = argc > 1 ? std::atoi(argv[1]) : 128;
    const int n_entries = argc > 2 ? std::atoi(argv[2]) : 800;
    const double delta = 0.25;
    Rng rng(2026);
    std::vector<EmbeddingVector> fulls;
    IvfIndex ref = IvfIndex::build({}, 1, 0, 1);
    ref.set_rebuild_interval(UINT64_MAX);
    semwarm_b200::IvfIndexT<EmbeddingVector, IndexedVector, SearchHit> gpu(dim, 7, n_entries, 64,
                                                                           0, SW_FLAG_TC_ALWAYS);
    EmbeddingVector centre = random_unit_vector(dim, rng);
    for (int e = 0; e < n_entries; ++e) {
        EmbeddingVector full = perturb(centre, 0.6, rng);
        auto vecs = build_entry_vectors((uint64_t)e + 1, full, rng.uniform(4.0, 12.0), delta,
                                        derive_seed(1, 0x5345474dULL));
        ref.insert(vecs);
        gpu.insert(vecs);
        fulls.push_back(full);
    }
    // remove a few entries on both sides (including an unknown id: warn + no-op)
    size_t removed = 0;
    for (uint64_t id : {3ull, 77ull, 400ull, 999999ull}) {
        removed += ref.contains(id) ? 1 : 0;
        ref.remove(id);
        gpu.remove(id);
    }
    int mismatches = 0, queries = 0;
    std::vector<EmbeddingVector> qs;
    for (int i = 0; i < 64; ++i) qs.push_back(perturb(fulls[(i * 37) % n_entries], 0.2, rng));
    for (size_t k : {1u, 5u, 8u}) {
        auto batch = gpu.search_batch(qs, k);
        for (size_t i = 0; i < qs.size(); ++i, ++queries) {
            auto a = ref.search(qs[i], k);
            const auto& b = batch[i];
            bool ok = a.size() == b.size();
            for (size_t j = 0; ok && j < a.size(); ++j)
                ok = a[j].entry_id == b[j].entry_id && a[j].segment.level == b[j].segment.level &&
                     a[j].segment.start_s == b[j].segment.start_s &&
                     a[j].similarity == b[j].similarity;
            if (!ok) ++mismatches;
        }
    }
    // choose_arm on (prompt, matched segment) contexts, zero model and a non-trivial one
    BanditModel m = BanditModel::zeros();
    for (size_t i = 0; i < m.theta.size(); ++i) m.theta[i] = (float)(((i * 7919) % 97) / 97.0 - 0.5);
    for (size_t i = 0; i < m.psi.size(); ++i) m.psi[i] = (float)(((i * 104729) % 89) / 89.0 - 0.5);
    semwarm_b200::check(sw_set_gater(gpu.context(), m.theta.data(), m.psi.data(), 11, m.beta),
                        "set_gater");
    std::vector<EmbeddingVector> segs;
    std::vector<int> T;
    for (size_t i = 0; i < qs.size(); ++i) {
        segs.push_back(ref.search(qs[i], 1)[0].entry_id ? fulls[(i * 37) % n_entries] : qs[i]);
        T.push_back(i % 2 ? 200 : 100);
    }
    int arm_mismatch = 0;
    for (int explore = 0; explore < 2; ++explore) {
        auto arms = semwarm_b200::choose_arms(gpu.context(), qs, segs, T, explore != 0);
        for (size_t i = 0; i < qs.size(); ++i) {
            int r = choose_arm(m, BanditContext{qs[i], segs[i], T[i]},
                               explore ? GaterMode::kExplore : GaterMode::kExploit);
            if (r != arms[i]) ++arm_mismatch;
        }
    }
    std::printf("queries=%d search_mismatches=%d arm_mismatches=%d entries=%zu\n", queries,
                mismatches, arm_mismatch, gpu.entry_count());
    const bool pass = mismatches == 0 && arm_mismatch == 0 &&
                      gpu.entry_count() == (size_t)n_entries - removed &&
                      gpu.entry_count() == ref.entry_count();
    std::printf(pass ? "DROPIN PASS\n" : "DROPIN FAIL\n");
    return pass ? 0 : 1;
}
