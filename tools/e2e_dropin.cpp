// End-to-end timing of the C++ drop-in itself: sgl::ifsglft then sgl::fsglft on
// std::vector data (pageable host memory; the output vectors are allocated by
// the call, as the reference's are), i.e. exactly what a caller of the
// reference's sgl_transform.hpp:71-76 runs.  Reports round trips/s for 1 and
// for N concurrent caller threads (one shared TransformPlan).
//   g++ -std=c++20 -O2 -Iinclude tools/e2e_dropin.cpp -Lpaper_1604_05140_b200 -lsglb200 \
//       -Wl,-rpath,$PWD/paper_1604_05140_b200 -o tools/e2e_dropin
//   tools/e2e_dropin B steps threads
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <thread>
#include <vector>

#include "sgl/sgl_transform.hpp"

using namespace sgl;

int main(int argc, char** argv) {
    const int B = argc > 1 ? std::atoi(argv[1]) : 128;
    const int steps = argc > 2 ? std::atoi(argv[2]) : 10;
    const int threads = argc > 3 ? std::atoi(argv[3]) : 2;
    const TransformPlan plan = TransformPlan::compute(B);
    std::mt19937_64 rng(0);
    std::normal_distribution<double> nd(0.0, 1.0 / std::sqrt(2.0));
    SglCoefficients c{B, cvector(coefficient_count(B))};
    for (auto& v : c.values) v = {nd(rng), nd(rng)};
    double err = 0.0;
    {  // warm: device plan, workspaces, staging
        const auto back = fsglft(ifsglft(c, plan), plan);
        err = roundtrip_error(c.values, back.values).max_abs;
    }
    auto run = [&](int nthreads) {
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> ts;
        for (int t = 0; t < nthreads; ++t)
            ts.emplace_back([&] {
                for (int k = 0; k < steps; ++k) {
                    const SampleGrid g = ifsglft(c, plan);
                    const SglCoefficients f = fsglft(g, plan);
                    if (f.values.size() != c.values.size()) std::abort();
                }
            });
        for (auto& t : ts) t.join();
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return nthreads * steps / s;
    };
    const double one = run(1);
    const double many = threads > 1 ? run(threads) : one;
    const double mb = 2.0 * 16.0 * (sample_count(B) + coefficient_count(B)) / 1e6;
    std::printf("{\"B\": %d, \"api\": \"sgl::ifsglft + sgl::fsglft, std::vector (pageable)\", \"steps\": %d, "
                "\"transforms_per_s_1_caller\": %.3f, \"transforms_per_s_%d_callers\": %.3f, "
                "\"pcie_mb_per_step\": %.1f, \"roundtrip_max_abs\": %.3e}\n",
                B, steps, one, threads, many, mb, err);
    return 0;
}
