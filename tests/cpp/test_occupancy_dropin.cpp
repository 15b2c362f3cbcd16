// C++ host API of the occupancy extension (semvox/occupancy_map.hpp) on the GPU:
// known answers of the contract (include/svx.h), the same cases as the oracle's in
// tests/test_occupancy.py. Exit code 0 = pass. Run by tests/test_occupancy.py (gpu).
#include "semvox/occupancy_map.hpp"

#include <cmath>
#include <cstdio>
#include <stdexcept>

using namespace semvox;

static int failures = 0;
#define EXPECT(c)                                                       \
    do {                                                                \
        if (!(c)) {                                                     \
            std::fprintf(stderr, "%s:%d: FAILED %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                                 \
        }                                                               \
    } while (0)

int main() {
    OccupancyConfig cfg;
    cfg.num_labels = 4;
    cfg.max_blocks = 1u << 12;
    {   // single ray along +x: HIT at voxel 10, MISS at 0..9 (svx.h contract)
        OccupancyMap m(cfg);
        PosedCloud c;
        c.points = {Vec3d(1.0, 0, 0)};
        const OccupancyReport r = m.integrate(c, {2}, {1.0f});
        EXPECT(r.rays == 1 && r.hit_voxels == 1 && r.miss_voxels == 10 && r.new_blocks == 2);
        const OccupancyVoxel h = m.query({10, 0, 0});
        EXPECT(h.found && h.log_odds == 0.85f && h.hits == 1 && h.misses == 0 && h.label == 2);
        const OccupancyVoxel f = m.query({5, 0, 0});
        EXPECT(f.found && f.log_odds == -0.4f && f.hits == 0 && f.misses == 1 && f.label == -1);
        EXPECT(m.histogram({10, 0, 0})[2] == 255u);
        EXPECT(!m.query({1000, 0, 0}).found);
        EXPECT(m.block_count() == 2);
        EXPECT(m.export_socc1().size() > 5);
    }
    {   // one pixel, principal point at its centre: point (0, 0, 2), HIT at (0, 0, 20)
        OccupancyMap m(cfg);
        DepthImage im;
        im.width = im.height = 1;
        im.depth = {2.0f};
        im.fx = im.fy = 100.0;
        im.cx = im.cy = 0.5;
        const auto r = m.integrate_depth({im});
        EXPECT(r.size() == 1 && r[0].rays == 1 && r[0].hit_voxels == 1 && r[0].miss_voxels == 20);
        EXPECT(m.query({0, 0, 20}).hits == 1);
        EXPECT(m.query({0, 0, 7}).misses == 1);
    }
    {   // argument errors map to the reference's exception classes
        OccupancyMap m(cfg);
        PosedCloud c;
        c.points = {Vec3d(1.0, 0, 0)};
        bool threw = false;
        try {
            m.integrate(c, {1, 2});
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        EXPECT(threw);
        DepthImage im;
        im.width = 2;
        im.height = 2;
        im.depth = {1.0f};
        threw = false;
        try {
            m.integrate_depth({im});
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        EXPECT(threw);
    }
    if (failures) return 1;
    std::printf("occupancy drop-in: all checks passed\n");
    return 0;
}
