// acceptance_gpu_gate.cpp -- the reference's acceptance gate (proj/tests/acceptance/acceptance_main.cpp,
// compiled unmodified by inclusion) with a selectable subset of its criteria, so the hot-path ones
// can run on every GPU test pass: each operator call of this harness is a host round trip
// (gpu_operators.cpp), and criteria 3 / 7 / 8 (stability sweeps, privacy probes, rerank) make
// tens of thousands of them.
//   acceptance_gpu_gate [n ...]   run criteria n (1..9) in order; default 1 2 4 (exactness, the
//                                 scrambling lemmas, shard merges -- the hot path's gates)
#include <chrono>
#include <cstdlib>

#define main acceptance_main_all
#include "acceptance/acceptance_main.cpp"
#undef main

int main(int argc, char** argv) {
    void (*const crit[])() = {criterion_exactness, criterion_lemmas,  criterion_stability,
                              criterion_shard_merge, criterion_audits, criterion_comm_accounting,
                              criterion_probes,      criterion_quant,  criterion_codec};
    std::vector<int> which;
    for (int i = 1; i < argc; ++i) which.push_back(std::atoi(argv[i]));
    if (which.empty()) which = {1, 2, 4};
    for (int c : which) {
        if (c < 1 || c > 9) return 2;
        const auto t0 = std::chrono::steady_clock::now();
        crit[c - 1]();
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::cout << "  (criterion " << c << ": " << s << " s)" << std::endl;
    }
    std::cout << (g_failures ? "acceptance gate: FAILED" : "acceptance gate: all selected criteria passed") << std::endl;
    return g_failures ? 1 : 0;
}
