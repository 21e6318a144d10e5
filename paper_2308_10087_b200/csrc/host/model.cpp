// Model schedule and placement helpers.
//   build_layer_specs      nn.cpp:28-64  (GCN: L x GcnConv; GCNII: Dense +
//                                         (L-2) x Gcn2Conv with beta_j = ln(lambda/j + 1)
//                                         + Dense, no ReLU on the logits layer)
//   make_stage_assignment  engines.cpp:8-21 (first L mod S stages get one more layer)
//   assign_groups          fabric.cpp:48-93 (whole groups per node, leftovers pooled)
#include <algorithm>

#include "gnnsim_b200.hpp"

namespace gnnsim {

ModelKind parse_model_kind(const std::string& s) {
    if (s == "gcn") return ModelKind::GCN;
    if (s == "sage") return ModelKind::Sage;
    if (s == "gcnii") return ModelKind::GCNII;
    throw std::invalid_argument("unknown model: " + s);
}

std::string model_kind_name(ModelKind k) {
    switch (k) {
        case ModelKind::GCN: return "gcn";
        case ModelKind::Sage: return "sage";
        case ModelKind::GCNII: return "gcnii";
    }
    return "?";
}

std::vector<LayerSpec> build_layer_specs(const ModelConfig& cfg, uint32_t in_features, uint32_t num_classes) {
    if (cfg.layers < 1) throw std::invalid_argument("model needs at least one layer");
    std::vector<LayerSpec> out;
    const uint32_t L = cfg.layers;
    if (cfg.kind == ModelKind::GCNII) {
        if (L < 3) throw std::invalid_argument("gcnii needs layers >= 3 (dense, convs, dense)");
        if (!(cfg.gcnii_alpha > 0.0 && cfg.gcnii_alpha < 1.0))
            throw std::invalid_argument("gcnii alpha must be in (0,1)");
        out.push_back({LayerKind::Dense, in_features, cfg.hidden, true, 0.0, 0.0});
        for (uint32_t j = 1; j + 2 <= L; ++j)
            out.push_back({LayerKind::Gcn2Conv, cfg.hidden, cfg.hidden, true, cfg.gcnii_alpha,
                           std::log(cfg.gcnii_lambda / double(j) + 1.0)});
        out.push_back({LayerKind::Dense, cfg.hidden, num_classes, false, 0.0, 0.0});
        return out;
    }
    const LayerKind k = cfg.kind == ModelKind::GCN ? LayerKind::GcnConv : LayerKind::SageConv;
    for (uint32_t l = 0; l < L; ++l)
        out.push_back({k, l == 0 ? in_features : cfg.hidden, l + 1 == L ? num_classes : cfg.hidden, l + 1 < L,
                       0.0, 0.0});
    return out;
}

bool model_needs_h0(const std::vector<LayerSpec>& specs) {
    return std::any_of(specs.begin(), specs.end(), [](const LayerSpec& s) { return s.kind == LayerKind::Gcn2Conv; });
}

uint64_t param_count(const std::vector<LayerSpec>& specs) {
    uint64_t n = 0;
    for (const auto& s : specs) n += uint64_t(s.k_in()) * s.out_dim + (s.has_bias() ? s.out_dim : 0);
    return n;
}

StageAssignment make_stage_assignment(uint32_t layers, uint32_t stages) {
    if (stages == 0 || stages > layers) throw std::invalid_argument("stage assignment needs 1 <= stages <= layers");
    StageAssignment sa;
    sa.num_stages = stages;
    const uint32_t q = layers / stages, r = layers % stages;
    for (uint32_t s = 0, at = 0; s < stages; ++s) {
        const uint32_t take = q + (s < r ? 1u : 0u);
        sa.ranges.emplace_back(at, at + take);
        at += take;
    }
    return sa;
}

uint32_t GroupMap::spanning_groups() const {
    uint32_t count = 0;
    for (const auto& g : groups)
        if (std::any_of(g.begin(), g.end(), [&](uint32_t w) { return node_of[w] != node_of[g.front()]; })) ++count;
    return count;
}

GroupMap assign_groups(uint32_t num_workers, uint32_t workers_per_node, uint32_t num_stages, uint32_t group_size) {
    if (workers_per_node == 0) throw std::invalid_argument("assign_groups: workers_per_node == 0");
    if (num_stages * group_size != num_workers)
        throw std::invalid_argument("assign_groups: num_workers != num_stages * group_size");
    GroupMap m;
    m.num_workers = num_workers;
    m.workers_per_node = workers_per_node;
    m.group_size = group_size;
    m.node_of.resize(num_workers);
    for (uint32_t w = 0; w < num_workers; ++w) m.node_of[w] = w / workers_per_node;
    std::vector<std::vector<uint32_t>> groups;
    std::vector<uint32_t> spill;
    if (group_size <= workers_per_node) {
        for (uint32_t w = 0; w < num_workers;) {
            const uint32_t node_end = std::min((m.node_of[w] + 1) * workers_per_node, num_workers);
            for (; w + group_size <= node_end && groups.size() < num_stages; w += group_size) {
                std::vector<uint32_t> g;
                for (uint32_t i = 0; i < group_size; ++i) g.push_back(w + i);
                groups.push_back(std::move(g));
            }
            for (; w < node_end; ++w) spill.push_back(w);
        }
    } else {
        for (uint32_t w = 0; w < num_workers; ++w) spill.push_back(w);
    }
    for (size_t i = 0; i + group_size <= spill.size(); i += group_size)
        groups.emplace_back(spill.begin() + std::ptrdiff_t(i), spill.begin() + std::ptrdiff_t(i + group_size));
    std::sort(groups.begin(), groups.end(), [](const auto& a, const auto& b) { return a.front() < b.front(); });
    m.groups = std::move(groups);
    m.group_of.resize(num_workers);
    m.rank_in_group.resize(num_workers);
    for (uint32_t g = 0; g < m.groups.size(); ++g)
        for (uint32_t r = 0; r < m.groups[g].size(); ++r) {
            m.group_of[m.groups[g][r]] = g;
            m.rank_in_group[m.groups[g][r]] = r;
        }
    return m;
}

}  // namespace gnnsim
