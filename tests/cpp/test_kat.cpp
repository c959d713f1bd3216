// Known-answer checks for the product planner, restating the golden values
// the reference's own tests pin (cited per case); built by
// tests/test_reference_suite.py against libepp_planner.so.
#include <doctest.h>

#include "epp/checkpoint.hpp"
#include "epp/cost_model.hpp"
#include "epp/milp.hpp"
#include "epp/pipeline.hpp"
#include "epp/planner.hpp"
#include "epp/processor.hpp"

using namespace epp;

namespace {
ClusterConfig cluster(int dp, int ds) {
    ClusterConfig c;
    c.pp_degree = dp;
    c.sp_degree = ds;
    c.num_gpus = dp * ds;
    c.mem_capacity = 1e12;
    if (ds > 1) {
        c.a2a_bandwidth[ds] = 1e11;
        c.a2a_latency[ds] = 1e-5;
    }
    return c;
}
ModelConfig model(int layers, int hidden, double tab, int dp) {
    ModelConfig m;
    m.layers = layers;
    m.hidden_dim = hidden;
    m.token_act_bytes = tab;
    m.stage_state_bytes.assign(dp, 1e9);
    return m;
}
CostParams params(double a1, double a2, double b1) {
    CostParams p;
    p.forward = {a1, a2, b1};
    p.backward = {2 * a1, 2 * a2, 2 * b1};
    return p;
}
Chunk split(long long ctx, long long n, bool tail, int id = 0, int seq = 0) {
    Chunk c;
    c.id = id;
    c.seq = seq;
    c.kind = ChunkKind::Split;
    c.context = ctx;
    c.slices = {n};
    c.tail = tail;
    return c;
}
}  // namespace

TEST_CASE("split_longest(16384, 2) balances at 11585 (test_processor.cpp:57-65)") {
    CostParams p;                      // pure quadratic work: t(s) = s^2
    p.forward = {1.0, 0.0, 0.0};
    p.backward = {1.0, 0.0, 0.0};
    const Mesh mesh = split_longest(16384, 2, p, cluster(1, 1), model(4, 8, 1e3, 1));
    REQUIRE(mesh.slice_lengths.size() == 1);
    CHECK(mesh.slice_lengths[0] == 11585);
    CHECK(mesh.token_threshold == 11585);
}

TEST_CASE("mesh cut of 13312 against {8192, 4096, 2048} (test_processor.cpp:73-92)") {
    Mesh mesh;
    mesh.slice_lengths = {8192, 4096, 2048};
    const SplitResult r = split_sequences({13312}, mesh);
    REQUIRE(r.split_chunks.size() == 2);
    CHECK(r.split_chunks[0].context == 0);
    CHECK(r.split_chunks[1].context == 8192);
    REQUIRE(r.tails.size() == 1);
    CHECK(r.tails[0].tokens == 1024);
    CHECK(r.tails[0].context == 12288);
}

TEST_CASE("compute_time hand values 12 and 25 (test_cost_model.cpp)") {
    ClusterConfig c = cluster(1, 1);
    CostParams p;
    p.forward = {1.0, 0.0, 0.0};
    const Chunk s = split(2, 2, true);
    CHECK(compute_time(s, Phase::Forward, p, c) == doctest::Approx(12.0));   // (2+2)^2 - 2^2
    Chunk b;
    b.kind = ChunkKind::Batched;
    b.slices = {3, 4};
    CHECK(compute_time(b, Phase::Forward, p, c) == doctest::Approx(25.0));   // 3^2 + 4^2
}

TEST_CASE("Eq. 1 realistic value 0.024806096 (test_cost_model.cpp:32-46)") {
    const ClusterConfig c = cluster(4, 2);
    CostParams p;
    p.forward = {2.1e-9, 3e-6, 5e-3};
    p.backward = p.forward;
    CHECK(compute_time(split(8192, 4096, true), Phase::Forward, p, c) ==
          doctest::Approx(0.024806096).epsilon(1e-9));
}

TEST_CASE("f2b is the reverse for one sequence split in 4 (test_pipeline.cpp:229-243)") {
    SequenceGroup g;
    g.lead_seq = 0;
    g.seq_ids = {0};
    long long ctx = 0;
    for (int i = 0; i < 4; ++i) {
        g.chunks.push_back(split(ctx, 100, i == 3, i, 0));
        ctx += 100;
    }
    g.tokens = 400;
    const PipelineUnit u = order_chunks({g});
    const std::vector<int> f2b = forward_to_backward_map(u, params(1e-9, 1e-5, 1e-3), cluster(2, 1),
                                                         model(4, 64, 1e4, 2));
    CHECK(f2b == std::vector<int>{3, 2, 1, 0});
}

TEST_CASE("ladder indexing reads ladder[f2b[k] + dp - p] (test_checkpoint.cpp:52-62)") {
    const std::vector<int> ladder = {1, 2, 3, 4, 5, 6, 7, 8, 9, 10};
    const std::vector<int> f2b = {6, 7, 8};
    CHECK(expand_checkpoint(ladder, 4, 0, f2b, 4) == 7);
    CHECK(expand_checkpoint(ladder, 4, 1, f2b, 4) == 8);
    CHECK(expand_checkpoint(ladder, 4, 2, f2b, 4) == 9);
}

TEST_CASE("milp agrees with brute force on random covering instances (test_milp.cpp:78-100)") {
    unsigned long long s = 42;
    auto next = [&]() {
        s = s * 6364136223846793005ULL + 1442695040888963407ULL;
        return static_cast<double>(s >> 11) * 0x1.0p-53;
    };
    for (int it = 0; it < 100; ++it) {
        milp::MilpInstance inst;
        inst.num_vars = 1 + static_cast<int>(next() * 5);
        for (int i = 0; i < inst.num_vars; ++i) inst.upper.push_back(static_cast<int>(next() * 4));
        const int rows = 1 + static_cast<int>(next() * 4);
        for (int r = 0; r < rows; ++r) {
            milp::Constraint c;
            for (int v = 0; v < inst.num_vars; ++v)
                if (next() < 0.7) c.terms.emplace_back(v, -std::round(next() * 500) / 100);
            c.rhs = std::round((next() * 10 - 8) * 100) / 100;
            inst.constraints.push_back(c);
        }
        const milp::SolveResult a = milp::solve(inst);
        const milp::SolveResult b = milp::brute_force(inst);
        REQUIRE(a.status == b.status);
        if (a.status == milp::Status::Optimal)
            CHECK(a.assignment.objective == b.assignment.objective);
    }
}
