// host_scene.h — host-side geometry preparation for the BVC hot path.
//
// Scene build (Scene::build, scene.cpp:11-125), solve-region construction
// (buildSolveRegion, cache.cpp:52-246) and the BVH that the device traversals
// use. This is one-time host preprocessing; every
// per-walk and per-pair query runs on the GPU.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace bvc_host {

// C++ exceptions mirror the reference's classes; the C ABI maps them to codes
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
enum Code { kInvalid = 1, kParse = 2, kSolver = 3, kSingularity = 4, kDomain = 5, kCuda = 6, kNoDevice = 7 };

struct HostScene {
    int dim = 2;
    int nv = 0, ns = 0;          // vertices, primitives (segments in 2D, triangles in 3D)
    std::vector<double> v;       // dim * nv
    std::vector<int> idx;        // 2*ns (segments) or 3*ns (triangles)
    std::vector<int> label;      // per primitive: 0 Dirichlet, 1 Neumann
    std::vector<double> normal;  // dim * ns, unit outward (2D: dir rotated by -90 deg, vec.h:21-23)
    std::vector<double> measure; // length (2D) or area (3D) per primitive
    // 2D loop structure (scene.cpp:53-83)
    std::vector<int> loop;       // loop id per segment
    std::vector<std::vector<int>> loops;  // ordered segment ids per loop/chain
    std::vector<double> arc;     // arc offset of vertex a within its loop
    std::vector<double> loopLength;
    std::vector<char> loopClosed;
    // silhouette candidates on the Neumann subset (scene.cpp:85-114)
    std::vector<double> silP, silN1, silN2;  // 2 per candidate
    std::vector<char> silAlways;
    std::vector<int> segSil;                 // 2 per segment, -1 = none
    // 3D: silhouette EDGES between Neumann triangles (the 3D analogue of the
    // candidate vertices): endpoints, adjacent face normals, open-edge flag
    std::vector<double> sil3A, sil3B, sil3N1, sil3N2;  // 3 per edge
    std::vector<char> sil3Always;
    std::vector<int> triSil;                            // 3 per triangle, -1 = none
    std::vector<int> component;                         // connected component per triangle
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    double diagonal = 0.0, dirichletMeasure = 0.0, neumannMeasure = 0.0, totalMeasure = 0.0;

    bool closed() const {
        if (dim == 3) return true;  // meshes are treated as closed soups
        for (char c : loopClosed) if (!c) return false;
        return !loopClosed.empty();
    }
    bool hasNeumann() const { return neumannMeasure > 0.0; }
    const double* vert(int i) const { return &v[static_cast<size_t>(dim) * i]; }
};

HostScene buildScene2(const double* vertices, int nv, const int* segments, const int* labels, int ns);
HostScene buildMesh3(const double* vertices, int nv, const int* tris, const int* labels, int nt);

// signed shoelace area of the loops (sampling.cpp:46-54)
double loopArea(const HostScene& s);

struct HostRegion {
    HostScene boundary;
    std::vector<int> kinds;   // bvc_region_segment_kind per boundary segment
    std::vector<int> source;  // originating scene segment, -1 if none
    double offset = 0.0, area = 0.0;
    bool wholeDomain = true;
};

HostRegion buildSolveRegion(const HostScene& scene, int mode, double offset, const HostScene* sub,
                            double epsilon);
HostRegion buildSolveRegion3(const HostScene& scene, int mode, double offset, const HostScene* sub,
                             double epsilon);
double meshVolume(const HostScene& s);

// BVH primitive class: 0 Dirichlet, 1 Neumann without silhouette candidates,
// 2 Neumann with silhouette candidates (the only Neumann class star queries visit)
int primClass(const HostScene& s, int i);

// Binary BVH flattened for the device. Node = two child boxes + two child refs.
// child ref >= 0: internal node index; < 0: leaf, ~ref = (start << 3) | (count - 1).
struct HostBvh {
    int dim = 2;
    std::vector<float> boxes;     // per node: 2 * (2*dim) floats (left lo, left hi, right lo, right hi)
    std::vector<int> children;    // 2 per node
    std::vector<unsigned> masks;  // per node: left class mask | right class mask << 3
    std::vector<int> order;       // leaf order -> primitive id
    int depth = 0;
};

HostBvh buildBvh(const HostScene& s, int leafSize = 4);

}  // namespace bvc_host
