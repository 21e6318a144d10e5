// Run outputs (metrics / trace / communication report / compare CSVs) and the
// closed-form communication and bubble analytics of the reference
// (analytics.cpp:12-103, fabric.cpp:20-35, :136-182, engines.cpp:23-38). The
// trace they consume is measured on the GPUs (gp_get_trace) instead of the
// fabric's simulated clock; the file formats are the reference's.
#include <algorithm>
#include <cstdio>
#include <fstream>
#include <map>
#include <stdexcept>

#include "gnnsim_b200.hpp"

namespace gnnsim {

namespace {
std::ofstream open_out(const std::string& path) {
    std::ofstream f(path, std::ios::trunc);
    if (!f) throw std::runtime_error("cannot write " + path);
    return f;
}
}  // namespace

const char* tag_name(MsgTag t) {
    static const char* names[kNumTags] = {"ForwardEmb", "BackwardGrad", "GraphBoundaryFwd",
                                          "GraphBoundaryBwd", "WeightSync", "Control"};
    const uint32_t i = uint32_t(t);
    return i < kNumTags ? names[i] : "?";
}

const char* link_class_name(LinkClass c) { return c == LinkClass::InterNode ? "inter_node" : "intra_node"; }

const char* trace_kind_name(TraceEvent::Kind k) {
    switch (k) {
        case TraceEvent::Kind::Compute: return "compute";
        case TraceEvent::Kind::Send: return "send";
        case TraceEvent::Kind::Recv: return "recv";
        case TraceEvent::Kind::Idle: return "idle";
    }
    return "?";
}

std::vector<CommReportRow> ledger_report(const EpochComm& e, uint32_t epoch) {
    std::vector<CommReportRow> rows;
    for (uint32_t tag = 0; tag < kNumTags; ++tag)
        for (uint32_t link = 0; link < 2; ++link)
            if (const uint64_t b = e.by_tag_link[tag][link])
                rows.push_back({epoch, MsgTag(tag), LinkClass(link), b, double(b) / kGiB});
    return rows;
}

void write_comm_report_csv(const std::string& path, const std::vector<CommReportRow>& rows) {
    auto f = open_out(path);
    f << "epoch,tag,link_class,bytes,gib\n";
    char g[48];
    for (const auto& r : rows) {
        std::snprintf(g, sizeof g, "%.9g", r.gib);
        f << r.epoch << ',' << tag_name(r.tag) << ',' << link_class_name(r.link) << ',' << r.bytes << ',' << g
          << '\n';
    }
}

void write_trace_jsonl(const std::string& path, const std::vector<TraceEvent>& events) {
    auto f = open_out(path);
    char line[256];
    for (const auto& e : events) {
        std::snprintf(line, sizeof line,
                      "{\"worker\":%u,\"t_start\":%.9g,\"t_end\":%.9g,\"kind\":\"%s\",\"chunk\":%d,"
                      "\"layer_lo\":%d,\"layer_hi\":%d}\n",
                      e.worker, e.t_start, e.t_end, trace_kind_name(e.kind), e.chunk, e.layer_lo, e.layer_hi);
        f << line;
    }
}

void write_metrics_csv(const std::string& path, const std::vector<EpochMetrics>& metrics) {
    auto f = open_out(path);
    f << "epoch,train_loss,train_acc,val_acc,test_acc,comm_bytes_graph,comm_bytes_pipeline,"
         "comm_bytes_weightsync,wall_time_s,bubble_fraction\n";
    char line[320];
    for (const auto& m : metrics) {
        std::snprintf(line, sizeof line, "%u,%.9g,%.9g,%.9g,%.9g,%llu,%llu,%llu,%.9g,%.9g\n", m.epoch, m.train_loss,
                      m.train_acc, m.val_acc, m.test_acc, (unsigned long long)m.comm_bytes_graph,
                      (unsigned long long)m.comm_bytes_pipeline, (unsigned long long)m.comm_bytes_weightsync,
                      m.wall_time_s, m.bubble_fraction);
        f << line;
    }
}

double volume_pipeline(const CommModelInput& in) {
    if (in.stages < 1) throw std::invalid_argument("volume_pipeline: stages >= 1 required");
    return 2.0 * (in.stages - 1.0) * in.n * in.hidden * in.vecs * in.bytes_per_value;
}

double volume_graph(const CommModelInput& in) {
    if (in.alpha < 0) throw std::invalid_argument("volume_graph: alpha >= 0 required");
    return 2.0 * in.alpha * in.layers * in.n * in.hidden * in.bytes_per_value;
}

double volume_hybrid(const CommModelInput& in) { return volume_pipeline(in) + volume_graph(in); }

CrossoverReport crossover_report(const CommModelInput& g, const CommModelInput& p, const CommModelInput& h) {
    CrossoverReport r;
    r.bytes_graph = volume_graph(g);
    r.bytes_pipeline = volume_pipeline(p);
    r.bytes_hybrid = volume_hybrid(h);
    // ascending predicted volume; equal volumes keep graph, pipeline, hybrid order
    std::vector<std::pair<double, const char*>> modes = {
        {r.bytes_graph, "graph"}, {r.bytes_pipeline, "pipeline"}, {r.bytes_hybrid, "hybrid"}};
    std::stable_sort(modes.begin(), modes.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    for (const auto& m : modes) r.ordering.emplace_back(m.second);
    r.tie = modes[0].first == modes[1].first;
    r.winner = r.tie ? "tie" : modes[0].second;
    // the comparisons in units of 2 N H (the paper's normalisation)
    // default ostream formatting of a double is %g (6 significant digits)
    auto cmp = [](const char* what, double a, double b) {
        char buf[256];
        std::snprintf(buf, sizeof buf, "%s: %g%s%g", what, a, a < b ? " < " : (a > b ? " > " : " == "), b);
        return std::string(buf);
    };
    const double hyb = h.alpha * h.layers + h.stages - 1.0;
    r.inequalities.push_back(cmp("graph vs pipeline, alpha_g*L vs (S_p-1)", g.alpha * g.layers, p.stages - 1.0));
    r.inequalities.push_back(cmp("hybrid vs graph, alpha_h*L+(S_h-1) vs alpha_g*L", hyb, g.alpha * g.layers));
    r.inequalities.push_back(cmp("hybrid vs pipeline, alpha_h*L+(S_h-1) vs (S_p-1)", hyb, p.stages - 1.0));
    return r;
}

BubbleReport bubble_analysis(const std::vector<TraceEvent>& trace) {
    if (trace.empty()) throw std::invalid_argument("bubble_analysis: empty trace");
    BubbleReport r;
    double lo = trace.front().t_start, hi = trace.front().t_end, compute = 0;
    std::map<uint32_t, bool> workers;
    int32_t last_chunk = -1;
    for (const auto& e : trace) {
        lo = std::min(lo, e.t_start);
        hi = std::max(hi, e.t_end);
        workers[e.worker] = true;
        if (e.kind == TraceEvent::Kind::Compute) compute += e.t_end - e.t_start;
        last_chunk = std::max(last_chunk, e.chunk);
    }
    r.stages = uint32_t(workers.size());
    r.chunks = uint32_t(last_chunk + 1);
    r.span = hi - lo;
    const double capacity = double(r.stages) * r.span;
    r.measured_bubble = capacity > 0 ? (capacity - compute) / capacity : 0.0;
    if (r.stages >= 1 && r.chunks >= 1)
        r.ideal_bubble = double(r.stages - 1) / double(r.chunks + r.stages - 1);
    return r;
}

void write_compare_csv(const std::string& path, const std::vector<CompareRow>& rows) {
    auto f = open_out(path);
    f << "mode,N,L,H,S,W,alpha,vecs,predicted_bytes,measured_bytes,rel_error\n";
    char line[192];
    for (const auto& r : rows) {
        std::snprintf(line, sizeof line, "%s,%.9g,%.9g,%.9g,%.9g,%.9g,%.9g,%.9g,%.9g,%llu,%.9g\n", r.mode.c_str(), r.n,
                      r.layers, r.hidden, r.stages, r.ways, r.alpha, r.vecs, r.predicted_bytes,
                      (unsigned long long)r.measured_bytes, r.rel_error);
        f << line;
    }
}

}  // namespace gnnsim
