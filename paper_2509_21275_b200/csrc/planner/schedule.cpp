// epp-b200 planner: elastic 1F1B schedule engine.
//
// Restates proj/src/pipeline.cpp:23-342.  The event loop produces the same
// events, windows and memory series as the reference; the difference is
// bookkeeping: each stage's next runnable op is cached and only re-derived
// for the stages whose inputs changed (the acting stage and its two
// neighbours), which turns the reference's O(n^2 d_p^2) rescans into
// O(n^2 d_p) without touching any floating-point expression.
#include <algorithm>
#include <cmath>
#include <limits>
#include <map>

#include "epp/pipeline.hpp"

namespace epp {

std::string to_string(EventKind kind) {
    switch (kind) {
        case EventKind::Forward: return "F";
        case EventKind::Backward: return "B";
        case EventKind::Recompute: return "R";
    }
    return "?";
}

PipelineUnit order_chunks(std::vector<SequenceGroup> groups) {
    std::sort(groups.begin(), groups.end(),
              [](const SequenceGroup& a, const SequenceGroup& b) {
                  if (a.chunks.size() != b.chunks.size())
                      return a.chunks.size() > b.chunks.size();
                  if (a.tokens != b.tokens) return a.tokens > b.tokens;
                  return a.lead_seq < b.lead_seq;
              });
    PipelineUnit unit;
    for (const SequenceGroup& g : groups) {
        unit.n_prefill = std::max(unit.n_prefill, static_cast<int>(g.chunks.size()));
        unit.chunks.insert(unit.chunks.end(), g.chunks.begin(), g.chunks.end());
        unit.sequences.insert(unit.sequences.end(), g.seq_ids.begin(),
                              g.seq_ids.end());
    }
    if (unit.chunks.empty()) unit.n_prefill = 0;
    return unit;
}

double warmup_cooldown_overhead(const std::vector<Chunk>& chunks,
                                const CostParams& params,
                                const ClusterConfig& cluster,
                                const ModelConfig& model) {
    if (chunks.empty()) throw ContractError("overhead of an empty chunk list");
    double sum = 0;
    for (const Chunk& c : chunks)
        sum += total_time(c, Phase::Forward, params, cluster, model) +
               total_time(c, Phase::Backward, params, cluster, model);
    return (cluster.pp_degree - 1) * (sum / static_cast<double>(chunks.size()));
}

double avg_layer_forward_seconds(const PipelineUnit& unit,
                                 const CostParams& params,
                                 const ClusterConfig& cluster,
                                 const ModelConfig& model) {
    if (unit.chunks.empty()) throw ContractError("empty pipeline unit");
    const double layers_here = model.layers_per_stage(cluster);
    double sum = 0;
    for (const Chunk& c : unit.chunks)
        sum += total_time(c, Phase::Forward, params, cluster, model) / layers_here;
    return sum / static_cast<double>(unit.chunks.size());
}

namespace detail {

namespace {

constexpr double kTieSlack = 1e-15;   // reference pipeline.cpp:205,217

struct Lane {                         // one pipeline stage
    int warmup = 0;
    int fwd_issued = 0;
    int bwd_issued = 0;
    double free_at = 0;
    std::vector<char> fwd_done, bwd_done;
    std::vector<double> fwd_end, bwd_end;
    std::vector<int> live;            // ascending forward positions
};

struct Op {
    bool ready = false;
    bool is_fwd = true;
    int chunk = -1;
    double start = std::numeric_limits<double>::infinity();
};

class Engine {
public:
    Engine(const PipelineUnit& unit, const CkptMap& ckpt, const CostParams& params,
           const ClusterConfig& cluster, const ModelConfig& model,
           const std::vector<std::vector<int>>* fixed_order)
        : unit_(unit), ckpt_(ckpt), cluster_(cluster), model_(model),
          fixed_(fixed_order), n_(unit.size()), dp_(cluster.pp_degree) {
        const int layers_here = model.layers_per_stage(cluster);
        fwd_dur_.resize(n_);
        bwd_dur_.resize(n_);
        layer_fwd_.resize(n_);
        for (int k = 0; k < n_; ++k) {
            fwd_dur_[k] = total_time(unit.chunks[k], Phase::Forward, params, cluster, model);
            bwd_dur_[k] = total_time(unit.chunks[k], Phase::Backward, params, cluster, model);
            layer_fwd_[k] = fwd_dur_[k] / layers_here;
        }
        // Backward of a non-tail slice waits for the next slice of its
        // sequence (dK/dV flow backwards along the sequence).
        next_slice_.assign(n_, -1);
        std::map<int, int> latest;
        for (int k = 0; k < n_; ++k) {
            const auto& seq = unit.chunks[k].seq;
            if (!seq.has_value()) continue;
            const auto it = latest.find(*seq);
            if (it != latest.end() && !unit.chunks[it->second].tail)
                next_slice_[it->second] = k;
            latest[*seq] = k;
        }
        lanes_.resize(dp_);
        for (int p = 0; p < dp_; ++p) {
            Lane& l = lanes_[p];
            l.warmup = std::min(dp_ - (p + 1) + unit.n_prefill - 1, n_);
            l.fwd_done.assign(n_, 0);
            l.bwd_done.assign(n_, 0);
            l.fwd_end.assign(n_, -1.0);
            l.bwd_end.assign(n_, -1.0);
        }
        info_.backward_order.assign(dp_, {});
        info_.windows.assign(dp_, {});
        info_.steady.assign(dp_, {});
        info_.window_bytes.assign(dp_, {});
        info_.trace.memory_series.assign(dp_, {});
        info_.trace.peak_memory.assign(dp_, 0.0);
        info_.trace.capacity_violation.assign(dp_, false);
    }

    ScheduleInfo run() {
        for (int p = 0; p < dp_; ++p) sample_memory(p, 0.0);
        std::vector<Op> cached(dp_);
        std::vector<char> stale(dp_, 1);
        const long long total = 2LL * n_ * dp_;
        for (long long step = 0; step < total; ++step) {
            int pick = -1;
            for (int p = 0; p < dp_; ++p) {
                if (stale[p]) {
                    cached[p] = next_op(p);
                    stale[p] = 0;
                }
                const Op& c = cached[p];
                if (!c.ready) continue;
                if (pick < 0 || c.start < cached[pick].start - kTieSlack) pick = p;
            }
            if (pick < 0) throw Error("pipeline schedule deadlock: no runnable work");
            const Op op = cached[pick];
            if (op.is_fwd)
                do_forward(pick, op);
            else
                do_backward(pick, op);
            stale[pick] = 1;
            if (pick > 0) stale[pick - 1] = 1;
            if (pick + 1 < dp_) stale[pick + 1] = 1;
        }
        finish();
        return std::move(info_);
    }

private:
    double sample_memory(int p, double t) {
        std::vector<WindowEntry> window;
        window.reserve(lanes_[p].live.size());
        for (const int k : lanes_[p].live)
            window.push_back({&unit_.chunks[k], ckpt_.at(p + 1, k)});
        const double bytes = stage_total_bytes(p + 1, window, cluster_, model_);
        info_.trace.memory_series[p].emplace_back(t, bytes);
        return bytes;
    }

    bool wants_forward(const Lane& l) const {
        if (l.fwd_issued < l.warmup) return true;
        return l.fwd_issued < n_ && l.fwd_issued - l.warmup == l.bwd_issued;
    }

    Op backward_op(int p, int k) const {
        const Lane& l = lanes_[p];
        if (!l.fwd_done[k]) return {};
        double start = std::max(l.free_at, l.fwd_end[k]);
        if (p + 1 < dp_) {
            const Lane& down = lanes_[p + 1];
            if (!down.bwd_done[k]) return {};
            start = std::max(start, down.bwd_end[k]);
        }
        const int nxt = next_slice_[k];
        if (nxt >= 0) {
            if (!l.bwd_done[nxt]) return {};
            start = std::max(start, l.bwd_end[nxt]);
        }
        return {true, false, k, start};
    }

    Op next_op(int p) const {
        const Lane& l = lanes_[p];
        if (l.fwd_issued == n_ && l.bwd_issued == n_) return {};
        if (wants_forward(l)) {
            const int k = l.fwd_issued;
            double start = l.free_at;
            if (p > 0) {
                const Lane& up = lanes_[p - 1];
                if (!up.fwd_done[k]) return {};
                start = std::max(start, up.fwd_end[k]);
            }
            return {true, true, k, start};
        }
        if (fixed_) return backward_op(p, (*fixed_)[p][l.bwd_issued]);
        Op best;
        for (int k = 0; k < n_; ++k) {
            if (l.bwd_done[k]) continue;
            const Op c = backward_op(p, k);
            if (!c.ready) continue;
            if (!best.ready || c.start < best.start - kTieSlack) best = c;
        }
        return best;
    }

    void do_forward(int p, const Op& op) {
        Lane& l = lanes_[p];
        const int k = op.chunk;
        const double end = op.start + fwd_dur_[k];
        info_.trace.events.push_back(
            {p + 1, unit_.chunks[k].id, k, EventKind::Forward, op.start, end});
        l.fwd_done[k] = 1;
        l.fwd_end[k] = end;
        l.free_at = end;
        ++l.fwd_issued;
        l.live.insert(std::lower_bound(l.live.begin(), l.live.end(), k), k);
        sample_memory(p, op.start);
    }

    void do_backward(int p, const Op& op) {
        Lane& l = lanes_[p];
        const int k = op.chunk;
        // The window is observed as the backward begins (chunk k included).
        info_.windows[p].push_back(l.live);
        const bool full_warmup = l.warmup == dp_ - (p + 1) + unit_.n_prefill - 1;
        info_.steady[p].push_back(full_warmup && l.bwd_issued < n_ - l.warmup);
        info_.backward_order[p].push_back(k);
        info_.window_bytes[p].push_back(sample_memory(p, op.start));

        double t = op.start;
        const double recompute = ckpt_.at(p + 1, k) * layer_fwd_[k];
        if (recompute > 0) {
            info_.trace.events.push_back({p + 1, unit_.chunks[k].id, k,
                                          EventKind::Recompute, t, t + recompute});
            t += recompute;
        }
        const double end = t + bwd_dur_[k];
        info_.trace.events.push_back(
            {p + 1, unit_.chunks[k].id, k, EventKind::Backward, t, end});
        l.bwd_done[k] = 1;
        l.bwd_end[k] = end;
        l.free_at = end;
        ++l.bwd_issued;
        l.live.erase(std::find(l.live.begin(), l.live.end(), k));
        sample_memory(p, end);
    }

    void finish() {
        SimTrace& tr = info_.trace;
        std::sort(tr.events.begin(), tr.events.end(),
                  [](const SimEvent& a, const SimEvent& b) {
                      if (a.start != b.start) return a.start < b.start;
                      if (a.stage != b.stage) return a.stage < b.stage;
                      return a.chunk_pos < b.chunk_pos;
                  });
        double makespan = 0;
        std::vector<double> busy(dp_, 0.0);
        for (const SimEvent& e : tr.events) {
            makespan = std::max(makespan, e.end);
            busy[e.stage - 1] += e.end - e.start;
        }
        tr.makespan = makespan;
        double busy_total = 0;
        for (const double b : busy) busy_total += b;
        tr.bubble_ratio = makespan > 0 ? 1.0 - busy_total / (dp_ * makespan) : 0.0;
        for (int p = 0; p < dp_; ++p) {
            double peak = 0;
            for (const auto& point : tr.memory_series[p]) peak = std::max(peak, point.second);
            tr.peak_memory[p] = peak;
            tr.capacity_violation[p] = peak > cluster_.mem_capacity;
        }
    }

    const PipelineUnit& unit_;
    const CkptMap& ckpt_;
    const ClusterConfig& cluster_;
    const ModelConfig& model_;
    const std::vector<std::vector<int>>* fixed_;
    const int n_;
    const int dp_;
    std::vector<double> fwd_dur_, bwd_dur_, layer_fwd_;
    std::vector<int> next_slice_;
    std::vector<Lane> lanes_;
    ScheduleInfo info_;
};

}  // namespace

ScheduleInfo run_schedule(const PipelineUnit& unit, const CkptMap& ckpt,
                          const CostParams& params, const ClusterConfig& cluster,
                          const ModelConfig& model,
                          const std::vector<std::vector<int>>* fixed_order) {
    if (unit.size() == 0) throw ContractError("cannot simulate an empty unit");
    if (ckpt.stages != cluster.pp_degree || ckpt.chunks != unit.size())
        throw ContractError("checkpoint map shape mismatch");
    const int layers_here = model.layers_per_stage(cluster);
    for (const int v : ckpt.layers)
        if (v < 0 || v > layers_here)
            throw ContractError("checkpoint layers out of range");
    Engine engine(unit, ckpt, params, cluster, model, fixed_order);
    return engine.run();
}

}  // namespace detail

namespace {

detail::ScheduleInfo dry_run(const PipelineUnit& unit, const CostParams& params,
                             const ClusterConfig& cluster, const ModelConfig& model) {
    const CkptMap zero = CkptMap::zero(cluster.pp_degree, unit.size());
    return detail::run_schedule(unit, zero, params, cluster, model, nullptr);
}

}  // namespace

SimTrace simulate_unit(const PipelineUnit& unit, const CkptMap& ckpt,
                       const CostParams& params, const ClusterConfig& cluster,
                       const ModelConfig& model) {
    detail::ScheduleInfo dry = dry_run(unit, params, cluster, model);
    if (ckpt.all_zero()) return dry.trace;
    return detail::run_schedule(unit, ckpt, params, cluster, model,
                                &dry.backward_order)
        .trace;
}

std::vector<std::vector<std::vector<int>>> enumerate_windows(
    const PipelineUnit& unit, const CostParams& params,
    const ClusterConfig& cluster, const ModelConfig& model) {
    const detail::ScheduleInfo dry = dry_run(unit, params, cluster, model);
    std::vector<std::vector<std::vector<int>>> out(dry.windows.size());
    for (size_t p = 0; p < dry.windows.size(); ++p)
        for (const auto& w : dry.windows[p])
            if (std::find(out[p].begin(), out[p].end(), w) == out[p].end())
                out[p].push_back(w);
    return out;
}

std::vector<int> forward_to_backward_map(const PipelineUnit& unit,
                                         const CostParams& params,
                                         const ClusterConfig& cluster,
                                         const ModelConfig& model) {
    const detail::ScheduleInfo dry = dry_run(unit, params, cluster, model);
    const std::vector<int>& order = dry.backward_order.back();
    for (const auto& other : dry.backward_order)
        if (other != order) throw Error("backward order diverged across stages");
    std::vector<int> f2b(unit.size(), -1);
    for (size_t pos = 0; pos < order.size(); ++pos) f2b[order[pos]] = static_cast<int>(pos);
    return f2b;
}

}  // namespace epp
