// epp-b200 planner: C ABI wrappers (include/epp_c.h).
#include <cstdlib>
#include <cstring>
#include <string>

#include "epp/plan_io.hpp"
#include "epp/planner.hpp"
#include "epp/render.hpp"
#include "epp/workload.hpp"
#include "epp_c.h"

namespace {

thread_local std::string g_last_error;

char* dup_string(const std::string& s) {
    char* out = static_cast<char*>(std::malloc(s.size() + 1));
    if (!out) throw std::bad_alloc();
    std::memcpy(out, s.c_str(), s.size() + 1);
    return out;
}

// Runs `body`, translating the planner's exception classes into codes.
template <typename Body>
int guarded(Body body) {
    g_last_error.clear();
    try {
        body();
        return EPP_OK;
    } catch (const epp::ConfigError& e) {
        g_last_error = e.what();
        return EPP_ECONFIG;
    } catch (const epp::ParseError& e) {
        g_last_error = e.what();
        return EPP_EPARSE;
    } catch (const epp::InfeasibleError& e) {
        g_last_error = e.what();
        return EPP_EINFEASIBLE;
    } catch (const epp::IoError& e) {
        g_last_error = e.what();
        return EPP_EIO;
    } catch (const epp::ContractError& e) {
        g_last_error = e.what();
        return EPP_ECONTRACT;
    } catch (const epp::FitError& e) {
        g_last_error = e.what();
        return EPP_EFIT;
    } catch (const epp::Error& e) {
        g_last_error = e.what();
        return EPP_EERROR;
    } catch (const nlohmann::json::exception& e) {
        g_last_error = std::string("bad json: ") + e.what();
        return EPP_EPARSE;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return EPP_EOTHER;
    }
}

nlohmann::json parse_or_throw(const char* text, const char* what) {
    if (!text) throw epp::ContractError(std::string(what) + " is null");
    try {
        return nlohmann::json::parse(text);
    } catch (const nlohmann::json::exception& e) {
        throw epp::ParseError(std::string(what) + ": " + e.what());
    }
}

}  // namespace

extern "C" {

int epp_plan_json(const char* config_json, const int64_t* lengths, size_t n,
                  int slices, int mode, int jobs, char** out_plan_json) {
    return guarded([&] {
        if (!out_plan_json) throw epp::ContractError("out_plan_json is null");
        if (!lengths && n > 0) throw epp::ContractError("lengths is null");
        if (mode < EPP_MODE_MAIN || mode > EPP_MODE_FULL_CKPT)
            throw epp::ContractError("unknown plan mode");
        const epp::SystemConfig cfg =
            epp::SystemConfig::from_json(parse_or_throw(config_json, "config"));
        const std::vector<long long> lens(lengths, lengths + n);
        std::optional<int> s;
        if (slices > 0) s = slices;
        const epp::SchedulePlan plan =
            epp::make_plan(lens, s, cfg, static_cast<epp::PlanMode>(mode), jobs);
        *out_plan_json = dup_string(epp::dump_document(epp::plan_to_json(plan, cfg)));
    });
}

int epp_simulate_json(const char* plan_json, char** out_trace_json,
                      double* out_makespan_sum) {
    return guarded([&] {
        if (!out_trace_json) throw epp::ContractError("out_trace_json is null");
        epp::SystemConfig cfg;
        const epp::SchedulePlan plan =
            epp::plan_from_json(parse_or_throw(plan_json, "plan"), cfg);
        const std::vector<epp::SimTrace> traces = epp::simulate_plan(plan, cfg);
        if (out_makespan_sum) *out_makespan_sum = epp::plan_simulated_seconds(traces);
        *out_trace_json = dup_string(epp::dump_document(epp::trace_to_json(traces)));
    });
}

int epp_generate_workload(const char* preset, int count, uint64_t seed,
                          int64_t context_cap, int64_t uniform_min,
                          int64_t uniform_max, int64_t* out_lengths) {
    return guarded([&] {
        if (!preset || !out_lengths) throw epp::ContractError("null argument");
        epp::GeneratorOptions opt;
        opt.uniform_min = uniform_min;
        opt.uniform_max = uniform_max;
        const epp::Workload w = epp::generate_workload(preset, count, seed, context_cap, opt);
        for (size_t i = 0; i < w.lengths.size(); ++i) out_lengths[i] = w.lengths[i];
    });
}

int epp_fit_cost_json(const char* config_json, const char* samples_json, char** out_json) {
    return guarded([&] {
        if (!out_json) throw epp::ContractError("out_json is null");
        const nlohmann::json cfg_doc = parse_or_throw(config_json, "config");
        epp::ClusterConfig cluster;
        try {
            const auto& c = cfg_doc.at("cluster");
            cluster.num_gpus = c.at("num_gpus").get<int>();
            cluster.pp_degree = c.at("pp_degree").get<int>();
            cluster.sp_degree = c.at("sp_degree").get<int>();
        } catch (const nlohmann::json::exception& e) {
            throw epp::ConfigError(std::string("bad configuration document: ") + e.what());
        }
        std::vector<epp::FitSample> samples;
        for (const auto& sj : parse_or_throw(samples_json, "samples")) {
            epp::FitSample s;
            s.chunk.context = sj.at("context").get<long long>();
            s.chunk.slices = sj.at("slices").get<std::vector<long long>>();
            s.chunk.kind = s.chunk.context > 0 ? epp::ChunkKind::Split : epp::ChunkKind::Batched;
            const std::string ph = sj.at("phase").get<std::string>();
            if (ph != "forward" && ph != "backward")
                throw epp::ParseError("sample phase must be forward|backward");
            s.phase = ph == "forward" ? epp::Phase::Forward : epp::Phase::Backward;
            s.seconds = sj.at("seconds").get<double>();
            samples.push_back(std::move(s));
        }
        const epp::FitResult r = epp::fit_cost_params(samples, cluster);
        nlohmann::json out;
        out["cost"] = {{"fwd_sec_per_token2", r.params.forward.sec_per_token2},
                       {"fwd_sec_per_token", r.params.forward.sec_per_token},
                       {"fwd_sec_fixed", r.params.forward.sec_fixed},
                       {"bwd_sec_per_token2", r.params.backward.sec_per_token2},
                       {"bwd_sec_per_token", r.params.backward.sec_per_token},
                       {"bwd_sec_fixed", r.params.backward.sec_fixed}};
        out["fwd_residual"] = r.fwd_residual;
        out["bwd_residual"] = r.bwd_residual;
        *out_json = dup_string(epp::dump_document(out));
    });
}

int epp_render_svg(const char* trace_json, char** out_svg) {
    return guarded([&] {
        if (!out_svg) throw epp::ContractError("out_svg is null");
        const std::vector<epp::SimTrace> traces =
            epp::trace_from_json(parse_or_throw(trace_json, "trace"));
        *out_svg = dup_string(epp::render_svg(traces));
    });
}

const char* epp_last_error(void) { return g_last_error.c_str(); }

void epp_free(char* p) { std::free(p); }

const char* epp_planner_version(void) { return "epp-b200-planner/1 (plan doc v1, trace doc v1)"; }

}  // extern "C"
