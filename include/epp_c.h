/* epp-b200: C ABI of the elastic-pipeline planner (libepp_planner.so).
 *
 * The reference ships no FFI: its callers link the C++ API directly
 * (proj/include/epp/*.hpp; CLI in proj/tools/epp_cli.cpp).  These entry
 * points are the thin, FFI-friendly wrappers a host language binds instead;
 * each names the reference interface it replaces.  The C++ API itself
 * (namespace epp, include/epp/*.hpp) is ALSO exported unchanged by the same
 * library, so C++ callers and the reference's own test-suite link against it
 * as a drop-in.
 *
 * Conventions
 *   - return 0 on success, otherwise an EPP_E* code naming the C++ exception
 *     class the reference would have thrown (errors.hpp); the message is in
 *     epp_last_error() (thread-local, valid until the next call on the thread).
 *   - strings returned through char** are heap-allocated; free with epp_free.
 *   - documents are the reference's JSON v1 formats, byte-identical to
 *     epp::dump_document(...) output.
 *   - all functions are reentrant; `jobs` > 1 uses an internal thread pool.
 */
#ifndef EPP_C_H_
#define EPP_C_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    EPP_OK = 0,
    EPP_EERROR = 1,       /* epp::Error (schedule deadlock, simplex limit, ...) */
    EPP_ECONFIG = 2,      /* epp::ConfigError */
    EPP_EPARSE = 3,       /* epp::ParseError */
    EPP_EINFEASIBLE = 4,  /* epp::InfeasibleError */
    EPP_EIO = 5,          /* epp::IoError */
    EPP_ECONTRACT = 6,    /* epp::ContractError */
    EPP_EFIT = 7,         /* epp::FitError */
    EPP_EOTHER = 8        /* any other std::exception */
};

enum { EPP_MODE_MAIN = 0, EPP_MODE_NO_WBC = 1, EPP_MODE_NO_CKPT = 2, EPP_MODE_FULL_CKPT = 3 };

/* Replaces epp::make_plan(lengths, slices, SystemConfig::from_json(cfg), mode,
 * jobs) followed by dump_document(plan_to_json(plan, cfg))
 * (reference proj/src/planner.cpp:372-474, proj/src/plan_io.cpp:54-105).
 * slices <= 0 selects the automatic slice-count sweep. */
int epp_plan_json(const char* config_json, const int64_t* lengths, size_t n,
                  int slices, int mode, int jobs, char** out_plan_json);

/* Replaces simulate_plan(plan_from_json(doc)) + trace_to_json
 * (reference proj/src/planner.cpp:476-487, proj/src/plan_io.cpp:169-209).
 * out_makespan_sum (nullable) receives plan_simulated_seconds(). */
int epp_simulate_json(const char* plan_json, char** out_trace_json,
                      double* out_makespan_sum);

/* Replaces epp::generate_workload(preset, count, seed, cap, {umin, umax})
 * (reference proj/src/workload.cpp:169-199).  out_lengths has count slots. */
int epp_generate_workload(const char* preset, int count, uint64_t seed,
                          int64_t context_cap, int64_t uniform_min,
                          int64_t uniform_max, int64_t* out_lengths);

/* Replaces epp::fit_cost_params (reference proj/src/cost_model.cpp:208-223).
 * samples_json: [{"context":C,"slices":[..],"phase":"forward"|"backward",
 * "seconds":t}, ...]; cluster taken from config_json.  Output: a JSON object
 * {"cost": {fwd_/bwd_ coefficients as in the config document},
 *  "fwd_residual": r, "bwd_residual": r}. */
int epp_fit_cost_json(const char* config_json, const char* samples_json,
                      char** out_json);

/* Replaces epp::render_svg(trace_from_json(doc))
 * (reference proj/src/render.cpp:32-125). */
int epp_render_svg(const char* trace_json, char** out_svg);

const char* epp_last_error(void);
void epp_free(char* p);
const char* epp_planner_version(void);

#ifdef __cplusplus
}
#endif

#endif /* EPP_C_H_ */
