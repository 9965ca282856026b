// TEST INFRASTRUCTURE: writes an HIPW dump with the UNMODIFIED reference
// (generate_synthetic + save_dump, workload.cpp) and prints its dump_checksum —
// the golden interchange file tests/golden/ref_small.hipw (tests/golden/make_golden.py).
// A standalone process for the same reason as ref_config_hash.cpp (iostreams).
#include <cstdio>
#include <cstdlib>

#include "hipprune/workload.hpp"

int main(int argc, char** argv) {
    if (argc != 8) {
        std::fprintf(stderr, "usage: ref_hipw out.hipw heads layers seq_kv seq_q dim seed\n");
        return 2;
    }
    hipprune::SyntheticConfig c;
    c.num_heads = std::strtoull(argv[2], nullptr, 10);
    c.num_layers = std::strtoull(argv[3], nullptr, 10);
    c.seq_len_kv = std::strtoull(argv[4], nullptr, 10);
    c.seq_len_q = std::strtoull(argv[5], nullptr, 10);
    c.head_dim = std::strtoull(argv[6], nullptr, 10);
    c.seed = std::strtoull(argv[7], nullptr, 10);
    const hipprune::AttentionWorkload w = hipprune::generate_synthetic(c);
    hipprune::save_dump(w, argv[1]);
    std::printf("%u\n", hipprune::dump_checksum(w));
    return 0;
}
