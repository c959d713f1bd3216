// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// Builds the reference planner (compiled from /root/reference/proj/src by
// oracle/Makefile, never copied) behind the same C ABI as the product
// (include/epp_c.h), with every entry point renamed epp_ref_*.  Only tests/,
// __graft_entry__.smoke() and bench.py's reference/cpu_baseline leg load the
// resulting oracle/_ref/libepp_ref.so, as the checker / CPU baseline.
#define epp_plan_json epp_ref_plan_json
#define epp_simulate_json epp_ref_simulate_json
#define epp_generate_workload epp_ref_generate_workload
#define epp_fit_cost_json epp_ref_fit_cost_json
#define epp_render_svg epp_ref_render_svg
#define epp_last_error epp_ref_last_error
#define epp_free epp_ref_free
#define epp_planner_version epp_ref_planner_version
#pragma GCC visibility push(default)
#include "epp_c.h"
#pragma GCC visibility pop
#include "../paper_2509_21275_b200/csrc/planner/c_api.cpp"
