// bvh.h -- host-side binned-SAH BVH2 builder for the triangle set.
//
// Replaces the reference's linear scan (core/scene.cpp:57-92) by a traversal
// whose *result* is identical: the device keeps the lexicographic minimum of
// (t, original primitive index), which is the linear scan's first-minimum
// winner, and every box is padded outward so no triangle Moeller-Trumbore would
// accept can be culled.
#pragma once

#include <cstdint>
#include <vector>

namespace ramlt_b200 {

struct BvhBuildNode {
    double lo[2][3], hi[2][3];   // child bounds (already padded outward)
    int32_t child[2];            // >= 0 internal node; < 0 leaf: ~((first << 4) | count)
};

struct BvhBuild {
    std::vector<BvhBuildNode> nodes;   // nodes[0] is the root
    std::vector<int32_t> order;        // BVH leaf order -> original triangle index
    int depth = 0;
};

// tris: 9 doubles per triangle (a, b, c).  Leaves hold at most `leaf_max` (<= 15)
// triangles; max depth 60.
BvhBuild build_bvh(const double *tris, size_t n, int leaf_max = 4);

}  // namespace ramlt_b200
