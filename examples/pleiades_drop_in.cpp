// pleiades_drop_in.cpp -- the reference's Pleiades protocol (bench.cpp:89-119,
// PAPER.md:652) written against the bode:: drop-in API instead of batchode::.
//
//   build: g++ -std=c++20 -O2 -Iinclude examples/pleiades_drop_in.cpp \
//              -Lpaper_1611_02274_b200/lib -lbode -Wl,-rpath,... -o pleiades_drop_in
//   run:   ./pleiades_drop_in [numSystems]   (prints a checksum line per window)
#include <cstdio>
#include <cstdlib>

#include "bode.hpp"

int main(int argc, char** argv) {
    const int num = argc > 1 ? std::atoi(argv[1]) : 1024;
    const bode::OdeProblem problem = bode::problems::pleiades();
    const bode::BatchStates batch = bode::problems::perturbInitialConditions(
        bode::problems::pleiadesInitialConditions(), 0.01, 42, num);
    bode::ToleranceSettings tol;
    tol.eps = 1e-10;
    try {
        const bode::OuterLoopResult res = bode::outerLoop(
            problem, batch, 0.0, 1.0, 0.1, bode::SolverChoice::RKCK, tol, 1,
            [](double t, bode::BatchStates snap) {
                double s = 0.0;
                for (double v : snap.values) s += v;
                std::printf("window t=%.17g sum=%.17g\n", t, s);
            });
        long accepted = 0, rejected = 0;
        for (const auto& st : res.stats) {
            accepted += st.stepsAccepted;
            rejected += st.stepsRejected;
        }
        std::printf("systems=%d windows=%d accepted=%ld rejected=%ld x1[0]=%.17g\n", num,
                    res.outerSteps, accepted, rejected, res.states.at(0, 0));
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
