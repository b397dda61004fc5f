// Compile-and-run check of the C++ mirror (include/lightcache.hpp) on host-only
// entry points: plan_steps, config validation and its ConfigError mapping.
#include <cstdio>

#include "lightcache.hpp"

int main() {
    const auto plan = stagecache_b200::plan_steps(7, 3);
    for (int s = 0; s < 7; ++s)
        std::printf("%c%s%s ", plan.is_full(s) ? 'F' : 'c', plan.has_consumers(s) ? "+" : "",
                    plan.is_last_consumer(s) ? "!" : "");
    std::printf("\n");
    stagecache_b200::validate_config("run.frames = 4\n");
    try {
        stagecache_b200::validate_config("nope.key = 1\n");
        return 1;
    } catch (const stagecache_b200::ConfigError& e) {
        std::printf("ConfigError: %s\n", e.what());
    }
    return 0;
}
