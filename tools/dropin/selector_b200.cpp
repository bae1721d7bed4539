// Link-time drop-in for the reference's selector.cpp (selector.hpp:25-58): the same four
// symbols, with score_candidates and select evaluated on the B200 through the C-ABI
// (sw_score_candidates_host / sw_select_host). A build links this file INSTEAD of
// /root/reference/proj/src/selector.cpp; pipeline.cpp's calls (pipeline.cpp:134-136) are unchanged.
// SelectorConfig::validate and make_negative_embedding are configuration plumbing restated from
// selector.cpp:8-20 (the negative embedding comes from the reference's own Rng and
// random_unit_vector, linked from core.cpp).
#include <mutex>
#include <stdexcept>

#include "semwarm/selector.hpp"
#include "semwarm_b200.hpp"

namespace semwarm {

namespace {
// one small device context for the component calls (dimension of the first use)
sw_ctx* component_ctx(size_t dim) {
    static std::mutex mu;
    static std::unique_ptr<semwarm_b200::Context> ctx;
    std::lock_guard<std::mutex> lk(mu);
    if (!ctx) ctx = std::make_unique<semwarm_b200::Context>((int)dim, 1, 1, 32, 0, 0, 0, 0u, 0);
    if ((size_t)ctx->dim() != dim) throw std::invalid_argument("dot: dimension mismatch");
    return ctx->get();
}
}  // namespace

void SelectorConfig::validate() const {
    if (top_k < 1) throw std::invalid_argument("selector top_k must be >= 1");
    if (!(temperature > 0.0)) throw std::invalid_argument("selector temperature must be > 0");
    if (quality_threshold < 0.0 || quality_threshold > 1.0)
        throw std::invalid_argument("selector quality threshold must be in [0, 1]");
}

EmbeddingVector make_negative_embedding(size_t dim) {
    Rng rng(derive_seed(0x4e454741ULL, dim));
    return random_unit_vector(dim, rng);
}

std::vector<CandidateScore> score_candidates(const std::vector<CandidateInput>& candidates,
                                             const EmbeddingVector& prompt,
                                             double requested_duration_s,
                                             const SelectorConfig& cfg) {
    if (candidates.empty()) throw std::invalid_argument("score_candidates: empty candidate list");
    return semwarm_b200::score_candidates<CandidateScore>(
        component_ctx(cfg.negative_embedding.dim()), candidates, prompt, requested_duration_s, cfg);
}

std::optional<size_t> select(const std::vector<CandidateScore>& scored, const SelectorConfig& cfg,
                             Rng& rng) {
    cfg.validate();
    if (scored.empty()) return std::nullopt;
    return semwarm_b200::select(component_ctx(cfg.negative_embedding.dim()), scored, cfg, rng);
}

}  // namespace semwarm
