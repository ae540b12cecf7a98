// Runs the reference's own randomized property suite (run_verification,
// src/verify.cpp:104-247) with pipeplan::train_partitioned provided by the
// B200 drop-in (train_partitioned_b200.cpp).  Usage: verify_b200 [seeds]
#include <cstdio>
#include <cstdlib>

#include "pipeplan/verify.hpp"

int main(int argc, char** argv) {
    pipeplan::VerifyOptions o;
    o.seeds = argc > 1 ? std::atoi(argv[1]) : 100;
    const pipeplan::VerifyReport r = pipeplan::run_verification(o);
    std::printf("%s", pipeplan::serialize_verify_report(r).c_str());
    return 0;
}
