// Integration check (TEST INFRASTRUCTURE): runs the reference's own
// run_pipeline (oracle/_ref, the unmodified proj/src) and the binding
// run_pipeline_b200 (tools/cpp/pipeline_b200.cpp over liblightcache.so) on
// the same config file and prints both RunResults as one JSON object for
// tests/test_capi.py.  Built by `make -C oracle integration` where
// /root/reference is present; the binary travels to the GPU box.
#include <cmath>
#include <cstdio>
#include <string>

#include "stagecache/pipeline.hpp"

namespace stagecache {
RunResult run_pipeline_b200(const RunConfig& cfg);
}

using namespace stagecache;

static void dump(const char* name, const RunResult& r, bool last) {
    std::printf("\"%s\":{\"wall\":[%.9g,%.9g,%.9g,%.9g,%.9g],", name, r.wall.setup, r.wall.encode,
                r.wall.denoise, r.wall.decode, r.wall.total);
    std::printf("\"peak\":[");
    for (int s = 0; s < 4; ++s)
        std::printf("%s[%lld,%lld]", s ? "," : "", static_cast<long long>(r.mem.peak[s][0]),
                    static_cast<long long>(r.mem.peak[s][1]));
    std::printf("],\"event_count\":%llu,", static_cast<unsigned long long>(r.mem.event_count));
    std::printf("\"timeline\":[");
    for (size_t i = 0; i < r.timeline.size(); ++i)
        std::printf("%s[%d,%lld,%lld,%lld]", i ? "," : "", static_cast<int>(r.timeline[i].kind),
                    static_cast<long long>(r.timeline[i].step), static_cast<long long>(r.timeline[i].bytes),
                    static_cast<long long>(r.timeline[i].clock_ns));
    std::printf("],\"denoiser_macs\":%lld,\"macs_per_full_step\":%lld,\"macs_per_cached_step\":%lld,",
                static_cast<long long>(r.denoiser_macs), static_cast<long long>(r.macs_per_full_step),
                static_cast<long long>(r.macs_per_cached_step));
    std::printf("\"full_steps\":%lld,\"cached_steps\":%lld,\"cache_bytes_planned\":%lld,",
                static_cast<long long>(r.full_steps), static_cast<long long>(r.cached_steps),
                static_cast<long long>(r.cache_bytes_planned));
    std::printf("\"makespan_s\":%.9g,\"stall_s\":%.9g,\"simulated\":%s,", r.makespan_s, r.stall_s,
                r.simulated ? "true" : "false");
    double sum = 0;
    for (int64_t i = 0; i < r.video.elems(); ++i) sum += r.video.data()[i];
    std::printf("\"video_elems\":%lld,\"video_sum\":%.17g}%s", static_cast<long long>(r.video.elems()), sum,
                last ? "" : ",");
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    RunConfig cfg = load_config_file(argv[1]);
    cfg.out_dir = "";
    RunResult ref = run_pipeline(cfg);
    RunResult gpu = run_pipeline_b200(cfg);
    // relative L2 of the two videos (b = 1, {t,c,h,w})
    double num = 0, den = 0;
    for (int64_t i = 0; i < ref.video.elems(); ++i) {
        const double d = static_cast<double>(gpu.video.data()[i]) - ref.video.data()[i];
        num += d * d;
        den += static_cast<double>(ref.video.data()[i]) * ref.video.data()[i];
    }
    std::printf("{");
    dump("reference", ref, false);
    dump("b200", gpu, false);
    std::printf("\"video_rel_l2\":%.9g", std::sqrt(num / (den > 0 ? den : 1)));
    // exception mapping: a budget far below the denoise working set
    RunConfig tight = cfg;
    tight.budget_fast_bytes = 1;
    try {
        run_pipeline_b200(tight);
        std::printf(",\"budget_error_stage\":null");
    } catch (const BudgetError& e) {
        std::printf(",\"budget_error_stage\":%d", static_cast<int>(e.stage));
    }
    std::printf("}\n");
    return 0;
}
