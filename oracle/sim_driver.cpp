// TEST / MEASUREMENT INFRASTRUCTURE: runs the reference's
// own consensus simulator — proj/src/sim.cpp, compiled UNMODIFIED into
// oracle/_ref by `make -C oracle ref` — with a CostModel given on the command
// line, so `simulate normal` reports hard-finality timing with the B200
// prover's measured costs (tools/calibrate_sim.py) instead of the paper's
// modelled 15 ms per 128-proof batch (proj/include/ace/sim.hpp:41-57).
//
//   ace_sim_b200 <scenario> [key=value ...]
//
// Keys are the reference's own override keys (SimConfig::apply_overrides,
// proj/src/sim.cpp:85-121: proof_batch_us, proof_parallelism, aggregation_us,
// fc_verify_us, attest_check_us_per_tx, txs_per_slot, n_slots, ...). Prints
// the reference's report (SimReport::render) and one JSON summary line.
#include <cstdio>
#include <string>

#include "ace/sim.hpp"

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s <scenario> [key=value ...]\n", argv[0]);
        return 2;
    }
    const auto sc = ace::sim::parse_scenario(argv[1]);
    if (!sc) {
        std::fprintf(stderr, "unknown scenario %s\n", argv[1]);
        return 2;
    }
    ace::config::KvMap kv;
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        const auto eq = a.find('=');
        if (eq == std::string::npos) {
            std::fprintf(stderr, "bad override %s (want key=value)\n", argv[i]);
            return 2;
        }
        kv[a.substr(0, eq)] = a.substr(eq + 1);
    }
    const ace::sim::SimConfig cfg = ace::sim::config_for_scenario(*sc, &kv);
    const ace::sim::SimReport rep = ace::sim::run_scenario(cfg, *sc);
    std::fputs(rep.render().c_str(), stdout);
    // JSON summary: hard finality after publish / after slot start per block
    std::string hard_pub = "[", hard_slot = "[";
    unsigned hard = 0;
    for (const auto& b : rep.blocks) {
        if (b.final_state == ace::finality::State::Hard) ++hard;
        hard_pub += (hard_pub.size() > 1 ? "," : "") + std::to_string(b.hard_after_publish_us());
        hard_slot += (hard_slot.size() > 1 ? "," : "") +
                     std::to_string(b.hard_after_slot_start_us(cfg.slot_us()));
    }
    std::printf(
        "{\"scenario\": \"%s\", \"blocks\": %zu, \"hard\": %u, \"assertions_ok\": %s, "
        "\"slot_us\": %llu, \"txs_per_slot\": %zu, \"proof_batch_us\": %llu, "
        "\"proof_parallelism\": %u, \"aggregation_us\": %llu, \"fc_verify_us\": %llu, "
        "\"proving_us_per_block\": %llu, \"hard_after_publish_us\": %s], "
        "\"hard_after_slot_start_us\": %s]}\n",
        rep.scenario.c_str(), rep.blocks.size(), hard, rep.ok() ? "true" : "false",
        static_cast<unsigned long long>(cfg.slot_us()), cfg.txs_per_slot,
        static_cast<unsigned long long>(cfg.cost.proof_batch_us), cfg.cost.proof_parallelism,
        static_cast<unsigned long long>(cfg.cost.aggregation_us),
        static_cast<unsigned long long>(cfg.cost.fc_verify_us),
        static_cast<unsigned long long>(cfg.cost.proving_us(cfg.txs_per_slot)), hard_pub.c_str(),
        hard_slot.c_str());
    return rep.ok() ? 0 : 1;
}
