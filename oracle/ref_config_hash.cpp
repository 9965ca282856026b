// TEST INFRASTRUCTURE: prints the UNMODIFIED reference's config_hash (config.cpp) of
// default_config() + the key=value overrides given as arguments. A standalone process:
// the reference's iostream-based canonical_config crashes when its objects are loaded
// into a Python process whose libstdc++ predates the compiler's (see tests/test_reports.py).
#include <cstdio>
#include <string>

#include "hipprune/config.hpp"

int main(int argc, char** argv) {
    try {
        hipprune::RunConfig cfg = hipprune::default_config();
        for (int i = 1; i < argc; ++i) {
            const std::string kv = argv[i];
            const auto eq = kv.find('=');
            if (eq == std::string::npos) return 2;
            hipprune::apply_override(cfg, kv.substr(0, eq), kv.substr(eq + 1));
        }
        std::printf("%llu\n", static_cast<unsigned long long>(hipprune::config_hash(cfg)));
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "%s\n", e.what());
        return 1;
    }
}
