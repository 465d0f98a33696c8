// Runs the reference acceptance suite (checks.cpp:489-502, run_all_checks) so the
// oracle build can be validated: 10/10 PASS and scratch/det/* byte-identical to
// the committed goldens (tests/golden/det/). Test infrastructure only.
//
// The same source is linked twice: against the pure reference library
// (oracle/_ref/ref_checks) and against the B200 drop-in façade
// (oracle/_ref/dropin_checks, see oracle/Makefile.dropin).
#include <cstdio>
#include <string>

#include "pslab/checks.hpp"

int main(int argc, char** argv) {
    std::string scratch = argc > 1 ? argv[1] : "/tmp/pslab_checks";
    std::string only = argc > 2 ? argv[2] : "";
    int failed = 0;
    int idx = 0;
    auto report = [&](const pslab::CheckResult& r) {
        ++idx;
        std::printf("[%s] %02d %-28s %s\n", r.pass ? "PASS" : "FAIL", idx, r.name.c_str(),
                    r.detail.c_str());
        std::fflush(stdout);
        if (!r.pass) ++failed;
    };
    if (only.empty()) {
        for (const auto& r : pslab::run_all_checks(scratch)) report(r);
    } else {
        // Comma-free selector: a single check name for quick runs.
        if (only == "determinism") report(pslab::check_determinism(scratch));
        else if (only == "degeneration") report(pslab::check_degeneration_equivalence());
        else if (only == "conservation") report(pslab::check_gradient_conservation());
        else if (only == "aggregation") report(pslab::check_aggregation_oracle());
        else if (only == "gib") report(pslab::check_gib_wire_bound());
        else if (only == "tuning") report(pslab::check_tuning_schedule());
        else {
            std::fprintf(stderr, "unknown check %s\n", only.c_str());
            return 2;
        }
    }
    return failed == 0 ? 0 : 1;
}
