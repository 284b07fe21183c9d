// host_scene.cpp — host geometry preparation (see host_scene.h).
#include "host_scene.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <functional>
#include <limits>
#include <map>
#include <numeric>
#include <optional>

namespace bvc_host {

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();
constexpr double kPi = 3.14159265358979323846;

struct P2 {
    double x = 0, y = 0;
};
inline P2 operator+(P2 a, P2 b) { return {a.x + b.x, a.y + b.y}; }
inline P2 operator-(P2 a, P2 b) { return {a.x - b.x, a.y - b.y}; }
inline P2 operator*(double s, P2 a) { return {s * a.x, s * a.y}; }
inline double dot(P2 a, P2 b) { return a.x * b.x + a.y * b.y; }
inline double cross(P2 a, P2 b) { return a.x * b.y - a.y * b.x; }
inline double norm(P2 a) { return std::sqrt(dot(a, a)); }

void computeBounds(HostScene& s) {
    for (int k = 0; k < s.dim; ++k) {
        s.lo[k] = kInf;
        s.hi[k] = -kInf;
    }
    for (int i = 0; i < s.nv; ++i)
        for (int k = 0; k < s.dim; ++k) {
            s.lo[k] = std::min(s.lo[k], s.v[s.dim * i + k]);
            s.hi[k] = std::max(s.hi[k], s.v[s.dim * i + k]);
        }
    double d2 = 0.0;
    for (int k = 0; k < s.dim; ++k) d2 += (s.hi[k] - s.lo[k]) * (s.hi[k] - s.lo[k]);
    s.diagonal = std::sqrt(d2);
}

}  // namespace

// Scene::build semantics (scene.cpp:11-125): normals, lengths, loops with arc
// offsets, silhouette candidates, manifold check. Validation order and messages
// follow the reference's ParseError cases.
HostScene buildScene2(const double* vertices, int nv, const int* segments, const int* labels, int ns) {
    HostScene s;
    s.dim = 2;
    if (nv <= 0 || ns <= 0) throw Error(kParse, "scene has no geometry");
    s.nv = nv;
    s.ns = ns;
    s.v.assign(vertices, vertices + 2 * static_cast<size_t>(nv));
    computeBounds(s);
    const double lengthFloor = 1e-12 * std::max(s.diagonal, 1.0);
    s.idx.resize(2 * static_cast<size_t>(ns));
    s.label.resize(ns);
    s.normal.resize(2 * static_cast<size_t>(ns));
    s.measure.resize(ns);
    for (int i = 0; i < ns; ++i) {
        int a = segments[2 * i], b = segments[2 * i + 1];
        if (a < 0 || a >= nv || b < 0 || b >= nv)
            throw Error(kParse, "segment " + std::to_string(i) + " references out-of-range vertex");
        double dx = s.v[2 * b] - s.v[2 * a], dy = s.v[2 * b + 1] - s.v[2 * a + 1];
        double len = std::sqrt(dx * dx + dy * dy);
        if (len <= lengthFloor) throw Error(kParse, "segment " + std::to_string(i) + " has zero length");
        s.idx[2 * i] = a;
        s.idx[2 * i + 1] = b;
        s.label[i] = labels[i] ? 1 : 0;
        s.measure[i] = len;
        s.normal[2 * i] = dy / len;  // outward for CCW loops
        s.normal[2 * i + 1] = -dx / len;
        (s.label[i] ? s.neumannMeasure : s.dirichletMeasure) += len;
        s.totalMeasure += len;
    }
    std::vector<int> outSeg(nv, -1), inSeg(nv, -1);
    for (int i = 0; i < ns; ++i) {
        int a = s.idx[2 * i], b = s.idx[2 * i + 1];
        if (outSeg[a] >= 0 || inSeg[b] >= 0)
            throw Error(kParse, "non-manifold or inconsistently oriented connectivity at segment " +
                                    std::to_string(i));
        outSeg[a] = i;
        inSeg[b] = i;
    }
    // loops and open chains: chains first (starting where nothing comes in), then cycles
    s.loop.assign(ns, -1);
    s.arc.assign(ns, 0.0);
    std::vector<char> seen(ns, 0);
    auto walkFrom = [&](int start) {
        int id = static_cast<int>(s.loopLength.size());
        double run = 0.0;
        bool isClosed = false;
        s.loops.emplace_back();
        for (int cur = start; cur >= 0 && !seen[cur];) {
            seen[cur] = 1;
            s.loops.back().push_back(cur);
            s.loop[cur] = id;
            s.arc[cur] = run;
            run += s.measure[cur];
            cur = outSeg[s.idx[2 * cur + 1]];
            if (cur == start) {
                isClosed = true;
                break;
            }
        }
        s.loopLength.push_back(run);
        s.loopClosed.push_back(isClosed ? 1 : 0);
    };
    for (int i = 0; i < ns; ++i)
        if (!seen[i] && inSeg[s.idx[2 * i]] < 0) walkFrom(i);
    for (int i = 0; i < ns; ++i)
        if (!seen[i]) walkFrom(i);
    // silhouette candidates: Neumann-Neumann vertices and open Neumann chain ends
    s.segSil.assign(2 * static_cast<size_t>(ns), -1);
    auto isNeumann = [&](int seg) { return seg >= 0 && s.label[seg] == 1; };
    auto attach = [&](int seg, int id) {
        int* slot = &s.segSil[2 * static_cast<size_t>(seg)];
        if (slot[0] < 0) slot[0] = id; else slot[1] = id;
    };
    for (int vi = 0; vi < nv; ++vi) {
        int si = inSeg[vi], so = outSeg[vi];
        bool ni = isNeumann(si), no = isNeumann(so);
        if (!ni && !no) continue;
        double n1[2] = {0, 0}, n2[2] = {0, 0};
        bool always = false;
        if (ni && no) {
            n1[0] = s.normal[2 * si]; n1[1] = s.normal[2 * si + 1];
            n2[0] = s.normal[2 * so]; n2[1] = s.normal[2 * so + 1];
            // exactly collinear neighbours: d1 * d2 = d1^2 <= 0 only for x exactly on
            // the line (a tie in scene.cpp:166-172). The device walker is never on a
            // Neumann line (it is nudged inside after each reflection), so such a
            // candidate can never pass; dropping it lets the star query prune.
            if (n1[0] == n2[0] && n1[1] == n2[1]) continue;
        } else if ((ni && so < 0) || (no && si < 0)) {
            always = true;
        } else {
            continue;  // Dirichlet junction: the Dirichlet distance already bounds the star
        }
        int id = static_cast<int>(s.silAlways.size());
        s.silP.push_back(s.v[2 * vi]);
        s.silP.push_back(s.v[2 * vi + 1]);
        s.silN1.insert(s.silN1.end(), {n1[0], n1[1]});
        s.silN2.insert(s.silN2.end(), {n2[0], n2[1]});
        s.silAlways.push_back(always ? 1 : 0);
        if (ni) attach(si, id);
        if (no) attach(so, id);
    }
    return s;
}

HostScene buildMesh3(const double* vertices, int nv, const int* tris, const int* labels, int nt) {
    HostScene s;
    s.dim = 3;
    if (nv <= 0 || nt <= 0) throw Error(kParse, "scene has no geometry");
    s.nv = nv;
    s.ns = nt;
    s.v.assign(vertices, vertices + 3 * static_cast<size_t>(nv));
    computeBounds(s);
    s.idx.assign(tris, tris + 3 * static_cast<size_t>(nt));
    s.label.resize(nt);
    s.normal.resize(3 * static_cast<size_t>(nt));
    s.measure.resize(nt);
    const double areaFloor = 1e-24 * std::max(s.diagonal * s.diagonal, 1.0);
    for (int i = 0; i < nt; ++i) {
        for (int k = 0; k < 3; ++k)
            if (s.idx[3 * i + k] < 0 || s.idx[3 * i + k] >= nv)
                throw Error(kParse, "triangle " + std::to_string(i) + " references out-of-range vertex");
        const double *a = s.vert(s.idx[3 * i]), *b = s.vert(s.idx[3 * i + 1]), *c = s.vert(s.idx[3 * i + 2]);
        double e1[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]}, e2[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
        double n[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
        double nn = std::sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
        if (0.5 * nn <= areaFloor) throw Error(kParse, "triangle " + std::to_string(i) + " has zero area");
        for (int k = 0; k < 3; ++k) s.normal[3 * i + k] = n[k] / nn;
        s.measure[i] = 0.5 * nn;
        s.label[i] = labels[i] ? 1 : 0;
        (s.label[i] ? s.neumannMeasure : s.dirichletMeasure) += s.measure[i];
        s.totalMeasure += s.measure[i];
    }
    // edge adjacency: silhouette edges between Neumann faces, open Neumann edges
    // (always silhouettes), connected components (for soups of closed meshes)
    std::map<std::pair<int, int>, std::vector<int>> edges;
    for (int i = 0; i < nt; ++i)
        for (int k = 0; k < 3; ++k) {
            int a = s.idx[3 * i + k], b = s.idx[3 * i + (k + 1) % 3];
            edges[{std::min(a, b), std::max(a, b)}].push_back(i);
        }
    std::vector<int> parent(nt);
    std::iota(parent.begin(), parent.end(), 0);
    std::function<int(int)> find = [&](int x) { return parent[x] == x ? x : parent[x] = find(parent[x]); };
    s.triSil.assign(3 * static_cast<size_t>(nt), -1);
    auto attach = [&](int tri, int id) {
        for (int k = 0; k < 3; ++k)
            if (s.triSil[3 * tri + k] < 0) { s.triSil[3 * tri + k] = id; return; }
    };
    for (const auto& [e, tris] : edges) {
        for (size_t k = 1; k < tris.size(); ++k) parent[find(tris[k])] = find(tris[0]);
        std::vector<int> neu;
        bool dir = false;
        for (int t : tris) if (s.label[t]) neu.push_back(t); else dir = true;
        if (neu.empty() || dir) continue;  // no Neumann face, or a Dirichlet junction
        const double* na = &s.normal[3 * static_cast<size_t>(neu[0])];
        bool always = neu.size() != 2;     // open edge (or non-manifold: conservative)
        const double* nb = neu.size() >= 2 ? &s.normal[3 * static_cast<size_t>(neu[1])] : na;
        if (!always && na[0] == nb[0] && na[1] == nb[1] && na[2] == nb[2]) continue;  // coplanar: ties only
        int id = static_cast<int>(s.sil3Always.size());
        const double *pa = s.vert(e.first), *pb = s.vert(e.second);
        s.sil3A.insert(s.sil3A.end(), pa, pa + 3);
        s.sil3B.insert(s.sil3B.end(), pb, pb + 3);
        s.sil3N1.insert(s.sil3N1.end(), na, na + 3);
        s.sil3N2.insert(s.sil3N2.end(), nb, nb + 3);
        s.sil3Always.push_back(always ? 1 : 0);
        // one of its faces carries the edge: the leaf of every face containing the edge
        // has a box no farther from x than the edge, so a star query that can use the
        // edge visits that face's leaf; the other face stays a plain Neumann primitive
        // (class 1), which star queries skip
        attach(neu[0], id);
    }
    s.component.resize(nt);
    std::map<int, int> comp;
    for (int i = 0; i < nt; ++i) {
        int r = find(i);
        auto it = comp.find(r);
        if (it == comp.end()) it = comp.emplace(r, static_cast<int>(comp.size())).first;
        s.component[i] = it->second;
    }
    return s;
}

// signed volume of a closed, outward-oriented triangle mesh (divergence theorem)
double meshVolume(const HostScene& s) {
    double v = 0.0;
    for (int i = 0; i < s.ns; ++i) {
        const double *a = s.vert(s.idx[3 * i]), *b = s.vert(s.idx[3 * i + 1]), *c = s.vert(s.idx[3 * i + 2]);
        v += (a[0] * (b[1] * c[2] - b[2] * c[1]) - a[1] * (b[0] * c[2] - b[2] * c[0]) + a[2] * (b[0] * c[1] - b[1] * c[0])) / 6.0;
    }
    return v;
}

// 3D solve region (no reference path exists; the 2D construction is cache.cpp:137-246):
// Neumann triangles are kept; vertices touched only by Dirichlet triangles move
// inward by l along their angle-weighted normal; junction vertices stay, so the
// Dirichlet patches bend down to the Neumann rim. Subdomain meshes pass through.
HostRegion buildSolveRegion3(const HostScene& scene, int mode, double offset, const HostScene* sub, double epsilon) {
    const double l = offset > 0.0 ? offset : 5.0 * epsilon;
    if (!(l > epsilon)) throw Error(kInvalid, "region offset l must exceed epsilon");
    HostRegion r;
    if (mode == 1) {
        if (!sub || sub->dim != 3) throw Error(kInvalid, "subdomain mode needs a region mesh");
        r.boundary = *sub;
        r.kinds.assign(sub->ns, 2);
        r.source.assign(sub->ns, -1);
        r.offset = l;
        r.wholeDomain = false;
        r.area = meshVolume(r.boundary);
        if (!(r.area > 0.0)) throw Error(kParse, "subdomain region must be outward oriented with positive volume");
        return r;
    }
    std::vector<double> vn(3 * static_cast<size_t>(scene.nv), 0.0);
    std::vector<char> junction(scene.nv, 0);
    for (int i = 0; i < scene.ns; ++i) {
        for (int k = 0; k < 3; ++k) {
            int v0 = scene.idx[3 * i + k], v1 = scene.idx[3 * i + (k + 1) % 3], v2 = scene.idx[3 * i + (k + 2) % 3];
            if (scene.label[i]) { junction[v0] = 1; continue; }
            const double *p0 = scene.vert(v0), *p1 = scene.vert(v1), *p2 = scene.vert(v2);
            double e1[3], e2[3];
            for (int d = 0; d < 3; ++d) { e1[d] = p1[d] - p0[d]; e2[d] = p2[d] - p0[d]; }
            double l1 = std::sqrt(e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2]);
            double l2 = std::sqrt(e2[0] * e2[0] + e2[1] * e2[1] + e2[2] * e2[2]);
            double c = (e1[0] * e2[0] + e1[1] * e2[1] + e1[2] * e2[2]) / (l1 * l2);
            double ang = std::acos(std::max(-1.0, std::min(1.0, c)));
            for (int d = 0; d < 3; ++d) vn[3 * static_cast<size_t>(v0) + d] += ang * scene.normal[3 * static_cast<size_t>(i) + d];
        }
    }
    std::vector<double> v(scene.v);
    for (int i = 0; i < scene.nv; ++i) {
        double* n = &vn[3 * static_cast<size_t>(i)];
        double len = std::sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
        if (junction[i] || !(len > 0.0)) continue;
        for (int d = 0; d < 3; ++d) v[3 * static_cast<size_t>(i) + d] -= l * n[d] / len;
    }
    r.boundary = buildMesh3(v.data(), scene.nv, scene.idx.data(), scene.label.data(), scene.ns);
    r.kinds.resize(scene.ns);
    r.source.resize(scene.ns);
    for (int i = 0; i < scene.ns; ++i) {
        r.kinds[i] = scene.label[i] ? 0 : 1;
        r.source[i] = i;
    }
    r.offset = l;
    r.wholeDomain = true;
    r.area = meshVolume(r.boundary);
    if (!(r.area > 0.0)) throw Error(kParse, "region offset produced a non-positive volume");
    return r;
}

double loopArea(const HostScene& s) {
    double area = 0.0;
    for (int i = 0; i < s.ns; ++i) {
        const double *a = s.vert(s.idx[2 * i]), *b = s.vert(s.idx[2 * i + 1]);
        area += 0.5 * (a[0] * b[1] - a[1] * b[0]);
    }
    return area;
}

// ---------------------------------------------------------------------------
// solve region (cache.cpp:52-246)
// ---------------------------------------------------------------------------
namespace {

struct Chain {           // polyline piece with shared provenance
    std::vector<P2> pts;
    int label = 0;
    int kind = 1;        // bvc_region_segment_kind
    int source = -1;
};

std::optional<P2> intersectLines(P2 p1, P2 d1, P2 p2, P2 d2) {
    double den = cross(d1, d2);
    if (std::abs(den) < 1e-12 * norm(d1) * norm(d2)) return std::nullopt;
    double t = cross(p2 - p1, d2) / den;
    return p1 + t * d1;
}

bool crossesProperly(P2 a1, P2 b1, P2 a2, P2 b2) {
    double o1 = cross(b1 - a1, a2 - a1), o2 = cross(b1 - a1, b2 - a1);
    double o3 = cross(b2 - a2, a1 - a2), o4 = cross(b2 - a2, b1 - a2);
    return o1 * o2 < 0.0 && o3 * o4 < 0.0;
}

// joins the chains of every loop into closed polylines, rejects self-crossings
// (the reference scans all pairs; a sweep over x-extents finds the same set)
HostRegion assemble(const std::vector<std::vector<Chain>>& loops, double l, bool whole, double weldTol) {
    std::vector<double> verts;
    std::vector<int> segs, labels, kinds, sources;
    std::vector<std::array<P2, 2>> emitted;
    for (const auto& chains : loops) {
        int base = static_cast<int>(verts.size() / 2);
        std::vector<std::array<P2, 2>> loopSegs;
        std::vector<int> owner;
        bool started = false;
        P2 prev;
        for (size_t ci = 0; ci < chains.size(); ++ci)
            for (const P2& p : chains[ci].pts) {
                if (!started) {
                    prev = p;
                    started = true;
                    continue;
                }
                if (norm(p - prev) < weldTol) continue;
                loopSegs.push_back({prev, p});
                owner.push_back(static_cast<int>(ci));
                prev = p;
            }
        if (loopSegs.size() < 3) throw Error(kParse, "region offset collapsed a boundary loop");
        if (norm(loopSegs.back()[1] - loopSegs.front()[0]) >= weldTol) {
            loopSegs.push_back({loopSegs.back()[1], loopSegs.front()[0]});
            owner.push_back(owner.back());
        }
        int count = static_cast<int>(loopSegs.size());
        for (int k = 0; k < count; ++k) {
            verts.push_back(loopSegs[k][0].x);
            verts.push_back(loopSegs[k][0].y);
            segs.push_back(base + k);
            segs.push_back(base + (k + 1) % count);
            const Chain& c = chains[owner[k]];
            labels.push_back(c.label);
            kinds.push_back(c.kind);
            sources.push_back(c.source);
            emitted.push_back(loopSegs[k]);
        }
    }
    // sweep for proper crossings between segments that share no endpoint
    std::vector<int> order(emitted.size());
    std::iota(order.begin(), order.end(), 0);
    auto xmin = [&](int i) { return std::min(emitted[i][0].x, emitted[i][1].x); };
    auto xmax = [&](int i) { return std::max(emitted[i][0].x, emitted[i][1].x); };
    std::sort(order.begin(), order.end(), [&](int a, int b) { return xmin(a) < xmin(b); });
    std::vector<std::pair<int, int>> crossings;
    for (size_t oi = 0; oi < order.size(); ++oi) {
        int i = order[oi];
        double xi = xmax(i);
        double ylo = std::min(emitted[i][0].y, emitted[i][1].y), yhi = std::max(emitted[i][0].y, emitted[i][1].y);
        for (size_t oj = oi + 1; oj < order.size() && xmin(order[oj]) <= xi; ++oj) {
            int j = order[oj];
            if (std::max(emitted[j][0].y, emitted[j][1].y) < ylo || std::min(emitted[j][0].y, emitted[j][1].y) > yhi)
                continue;
            const auto &A = emitted[i], &B = emitted[j];
            if (norm(A[0] - B[0]) < weldTol || norm(A[0] - B[1]) < weldTol || norm(A[1] - B[0]) < weldTol ||
                norm(A[1] - B[1]) < weldTol)
                continue;
            if (crossesProperly(A[0], A[1], B[0], B[1])) crossings.push_back({std::min(i, j), std::max(i, j)});
        }
    }
    if (!crossings.empty()) {
        std::sort(crossings.begin(), crossings.end());
        std::string msg = "region offset self-intersects: segments";
        for (auto [i, j] : crossings) msg += " " + std::to_string(i) + "-" + std::to_string(j);
        throw Error(kParse, msg);
    }
    HostRegion r;
    r.boundary = buildScene2(verts.data(), static_cast<int>(verts.size() / 2), segs.data(), labels.data(),
                             static_cast<int>(labels.size()));
    r.kinds = std::move(kinds);
    r.source = std::move(sources);
    r.offset = l;
    r.wholeDomain = whole;
    r.area = loopArea(r.boundary);
    if (!(r.area > 0.0)) throw Error(kParse, "region offset produced a non-positive area");
    return r;
}

}  // namespace

HostRegion buildSolveRegion(const HostScene& scene, int mode, double offset, const HostScene* sub,
                            double epsilon) {
    if (scene.dim == 3) return buildSolveRegion3(scene, mode, offset, sub, epsilon);
    const double l = offset > 0.0 ? offset : 5.0 * epsilon;
    if (!(l > epsilon)) throw Error(kInvalid, "region offset l must exceed epsilon");
    const double weldTol = 1e-10 * std::max(scene.diagonal, 1e-30);

    if (mode == 1) {  // Subdomain: the user loop verbatim (cache.cpp:142-156)
        if (!sub) throw Error(kInvalid, "subdomain mode needs a region loop");
        if (!sub->closed()) throw Error(kParse, "subdomain region loops must be closed");
        HostRegion r;
        r.boundary = *sub;
        r.kinds.assign(sub->ns, 2);
        r.source.assign(sub->ns, -1);
        r.offset = l;
        r.wholeDomain = false;
        r.area = loopArea(r.boundary);
        if (!(r.area > 0.0)) throw Error(kParse, "subdomain region must wind counterclockwise with positive area");
        return r;
    }
    if (!scene.closed()) throw Error(kParse, "whole-domain regions need a closed scene");

    // per loop: keep Neumann segments, push Dirichlet segments inward by l, then
    // repair the joints (cache.cpp:160-228)
    const std::vector<std::vector<int>>& loopSegs = scene.loops;
    auto vtx = [&](int i) { return P2{scene.v[2 * i], scene.v[2 * i + 1]}; };
    auto nrm = [&](int s) { return P2{scene.normal[2 * s], scene.normal[2 * s + 1]}; };
    std::vector<std::vector<Chain>> loops;
    for (const auto& ls : loopSegs) {
        int n = static_cast<int>(ls.size());
        std::vector<Chain> chains(n);
        for (int i = 0; i < n; ++i) {
            int sid = ls[i];
            P2 a = vtx(scene.idx[2 * sid]), b = vtx(scene.idx[2 * sid + 1]);
            Chain& c = chains[i];
            c.label = scene.label[sid];
            c.source = sid;
            if (scene.label[sid] == 1) {
                c.kind = 0;
                c.pts = {a, b};
            } else {
                c.kind = 1;
                P2 o = (-l) * nrm(sid);
                c.pts = {a + o, b + o};
            }
        }
        std::vector<std::vector<Chain>> caps(n);
        for (int i = 0; i < n; ++i) {
            Chain &P = chains[i], &Q = chains[(i + 1) % n];
            bool pOff = P.kind == 1, qOff = Q.kind == 1;
            if (!pOff && !qOff) continue;
            int sp = P.source, sq = Q.source;
            P2 up = vtx(scene.idx[2 * sp + 1]) - vtx(scene.idx[2 * sp]);
            P2 uq = vtx(scene.idx[2 * sq + 1]) - vtx(scene.idx[2 * sq]);
            up = (1.0 / norm(up)) * up;
            uq = (1.0 / norm(uq)) * uq;
            auto weld = [&]() {
                P2 mid = 0.5 * (P.pts.back() + Q.pts.front());
                P.pts.back() = mid;
                Q.pts.front() = mid;
            };
            if (pOff && qOff) {
                if (norm(nrm(sp) - nrm(sq)) < 1e-9) {
                    weld();
                    continue;
                }
                double turn = cross(up, uq);
                if (turn > 1e-12) {  // convex: miter
                    auto q = intersectLines(P.pts.back(), up, Q.pts.front(), uq);
                    if (!q) throw Error(kParse, "region offset: degenerate miter join");
                    P.pts.back() = *q;
                    Q.pts.front() = *q;
                } else if (turn < -1e-12) {  // reflex: 8-chord arc around the vertex
                    P2 v = vtx(scene.idx[2 * sq]);
                    P2 np = nrm(sp), nq = nrm(sq);
                    double phi = std::atan2(np.y, np.x);
                    double delta = std::atan2(cross(np, nq), dot(np, nq));
                    Chain arc;
                    arc.label = P.label;
                    arc.kind = 1;
                    arc.source = P.source;
                    for (int k = 0; k <= 8; ++k) {
                        double ang = phi + delta * k / 8.0;
                        arc.pts.push_back(v - l * P2{std::cos(ang), std::sin(ang)});
                    }
                    caps[i].push_back(std::move(arc));
                } else {
                    weld();
                }
            } else {  // Dirichlet/Neumann junction: trim both to the crossing
                auto q = intersectLines(P.pts.back(), up, Q.pts.front(), uq);
                if (!q) throw Error(kParse, "region offset: junction between parallel boundary segments");
                P.pts.back() = *q;
                Q.pts.front() = *q;
            }
        }
        for (int i = 0; i < n; ++i) {
            const Chain& P = chains[i];
            int sp = P.source;
            P2 u = vtx(scene.idx[2 * sp + 1]) - vtx(scene.idx[2 * sp]);
            if (dot(P.pts.back() - P.pts.front(), u) <= 0.0)
                throw Error(kParse, "region offset too large: segment " + std::to_string(sp) + " inverted");
        }
        std::vector<Chain> flat;
        for (int i = 0; i < n; ++i) {
            flat.push_back(std::move(chains[i]));
            for (auto& c : caps[i]) flat.push_back(std::move(c));
        }
        loops.push_back(std::move(flat));
    }
    return assemble(loops, l, true, weldTol);
}

// ---------------------------------------------------------------------------
// BVH: binary, median split on the longest centroid axis, leaves of <= leafSize
// ---------------------------------------------------------------------------
int primClass(const HostScene& s, int i) {
    if (s.label[i] == 0) return 0;
    if (s.dim == 2 && (s.segSil[2 * static_cast<size_t>(i)] >= 0 || s.segSil[2 * static_cast<size_t>(i) + 1] >= 0))
        return 2;
    if (s.dim == 3)
        for (int k = 0; k < 3; ++k)
            if (s.triSil[3 * static_cast<size_t>(i) + k] >= 0) return 2;
    return 1;
}

namespace {

struct Box {
    double lo[3] = {kInf, kInf, kInf}, hi[3] = {-kInf, -kInf, -kInf};
    void add(const double* p, int d) {
        for (int k = 0; k < d; ++k) {
            lo[k] = std::min(lo[k], p[k]);
            hi[k] = std::max(hi[k], p[k]);
        }
    }
    void add(const Box& b, int d) {
        for (int k = 0; k < d; ++k) {
            lo[k] = std::min(lo[k], b.lo[k]);
            hi[k] = std::max(hi[k], b.hi[k]);
        }
    }
};

// half surface measure of a box: half-perimeter in 2D, half surface area in 3D
inline double boxArea(const Box& b, int d) {
    if (b.lo[0] > b.hi[0]) return 0.0;
    double e[3] = {0, 0, 0};
    for (int k = 0; k < d; ++k) e[k] = b.hi[k] - b.lo[k];
    return d == 2 ? e[0] + e[1] : e[0] * e[1] + e[1] * e[2] + e[2] * e[0];
}

struct Builder {
    const HostScene& s;
    int d, nvp, leafSize;
    double pad;
    bool useSah;  // binned SAH splits (large scenes); median splits otherwise
    std::vector<Box> primBox;
    std::vector<double> centroid;
    HostBvh& out;
    std::vector<int>& order;

    // returns child reference; fills box and mask of the subtree
    int build(int start, int count, Box& box, unsigned& mask, int depth) {
        out.depth = std::max(out.depth, depth);
        box = Box();
        mask = 0;
        Box cbox;
        for (int i = start; i < start + count; ++i) {
            box.add(primBox[order[i]], d);
            cbox.add(&centroid[static_cast<size_t>(d) * order[i]], d);
            mask |= 1u << primClass(s, order[i]);
        }
        double ext[3] = {0, 0, 0};
        double maxExt = 0.0;
        int axis = 0;
        for (int k = 0; k < d; ++k) {
            ext[k] = cbox.hi[k] - cbox.lo[k];
            if (ext[k] > maxExt) { maxExt = ext[k]; axis = k; }
        }
        if (count <= leafSize || maxExt <= 0.0) {
            if (count > 8) {  // degenerate centroids: split by index
                return splitAt(start, count, start + count / 2, depth);
            }
            return ~((start << 3) | (count - 1));
        }
        // in 2D a node holding several primitive classes splits by class first:
        // star queries (Dirichlet + silhouette) and Neumann rays then never enter
        // the other classes' subtrees (measured: C2 walks -7%)
        int mid = -1;
        if (d == 2 && (mask & (mask - 1))) {  // 3D soups measured slower with it (C5 +10%)
            int lowest = __builtin_ctz(mask);
            auto it = std::partition(order.begin() + start, order.begin() + start + count,
                                     [&](int p) { return primClass(s, p) == lowest; });
            mid = static_cast<int>(it - order.begin());
        } else if (useSah && depth < 24) {  // depth stays below the device stack (kStack = 48)
            mid = sahSplit(start, count, cbox);
        }
        if (mid < 0) {  // median split along the widest centroid extent
            mid = start + count / 2;
            std::nth_element(order.begin() + start, order.begin() + mid, order.begin() + start + count,
                             [&](int p, int q) { return centroid[d * p + axis] < centroid[d * q + axis]; });
        }
        return splitAt(start, count, mid, depth);
    }

    // binned surface-area-heuristic split (32 bins per axis): minimises
    // A(left) N(left) + A(right) N(right), i.e. the expected number of primitive
    // tests of a query that reaches this node, which also cuts the sibling-box
    // overlap the best-first distance queries pay for. Returns -1 if no split
    // separates the centroids.
    int sahSplit(int start, int count, const Box& cbox) {
        constexpr int kBins = 32;
        double best = std::numeric_limits<double>::infinity();
        int bestAxis = -1, bestBin = -1;
        for (int k = 0; k < d; ++k) {
            double lo = cbox.lo[k], ext = cbox.hi[k] - cbox.lo[k];
            if (!(ext > 0.0)) continue;
            Box bb[kBins];
            int bn[kBins] = {0};
            for (int i = start; i < start + count; ++i) {
                int p = order[i];
                int bi = std::min(kBins - 1, static_cast<int>((centroid[static_cast<size_t>(d) * p + k] - lo) / ext * kBins));
                bb[bi].add(primBox[p], d);
                ++bn[bi];
            }
            double rightA[kBins];
            int rightN[kBins];
            Box acc;
            int n = 0;
            for (int i = kBins - 1; i > 0; --i) {
                acc.add(bb[i], d);
                n += bn[i];
                rightA[i] = boxArea(acc, d);
                rightN[i] = n;
            }
            Box left;
            int nl = 0;
            for (int i = 0; i < kBins - 1; ++i) {  // split between bin i and i + 1
                left.add(bb[i], d);
                nl += bn[i];
                if (nl == 0 || rightN[i + 1] == 0) continue;
                double c = boxArea(left, d) * nl + rightA[i + 1] * rightN[i + 1];
                if (c < best) { best = c; bestAxis = k; bestBin = i; }
            }
        }
        if (bestAxis < 0) return -1;
        double lo = cbox.lo[bestAxis], ext = cbox.hi[bestAxis] - cbox.lo[bestAxis];
        auto it = std::partition(order.begin() + start, order.begin() + start + count, [&](int p) {
            int bi = std::min(kBins - 1, static_cast<int>((centroid[static_cast<size_t>(d) * p + bestAxis] - lo) / ext * kBins));
            return bi <= bestBin;
        });
        int mid = static_cast<int>(it - order.begin());
        return (mid == start || mid == start + count) ? -1 : mid;
    }

    int splitAt(int start, int count, int mid, int depth) {
        int node = static_cast<int>(out.children.size() / 2);
        out.children.resize(out.children.size() + 2);
        out.masks.push_back(0);
        out.boxes.resize(out.boxes.size() + 4 * d);
        Box lb, rb;
        unsigned lm, rm;
        int l = build(start, mid - start, lb, lm, depth + 1);
        int r = build(mid, start + count - mid, rb, rm, depth + 1);
        out.children[2 * node] = l;
        out.children[2 * node + 1] = r;
        out.masks[node] = lm | (rm << 3);
        float* b = &out.boxes[static_cast<size_t>(4 * d) * node];
        // pad outward by ~2^-20 diag: FP32 slab tests against the degenerate
        // (zero-width) boxes of axis-aligned segments must not cull true crossings
        for (int k = 0; k < d; ++k) {
            b[k] = static_cast<float>(lb.lo[k] - pad);
            b[d + k] = static_cast<float>(lb.hi[k] + pad);
            b[2 * d + k] = static_cast<float>(rb.lo[k] - pad);
            b[3 * d + k] = static_cast<float>(rb.hi[k] + pad);
        }
        return node;
    }
};

}  // namespace

HostBvh buildBvh(const HostScene& s, int leafSize) {
    HostBvh out;
    out.dim = s.dim;
    int d = s.dim, nvp = d;  // vertices per primitive
    // SAH pays off on large or 3D scenes (measured: C3-C5 walks -10..14%); on small 2D
    // scenes the median tree of axis-aligned segments is the better distance-query tree
    const bool sah = d == 3 || s.ns >= 4096;
    Builder b{s, d, nvp, leafSize, 9.5367431640625e-7 * std::max(s.diagonal, 1e-30), sah, {}, {}, out, out.order};
    b.primBox.resize(s.ns);
    b.centroid.assign(static_cast<size_t>(d) * s.ns, 0.0);
    for (int i = 0; i < s.ns; ++i) {
        for (int j = 0; j < nvp; ++j) {
            const double* p = s.vert(s.idx[static_cast<size_t>(nvp) * i + j]);
            b.primBox[i].add(p, d);
            for (int k = 0; k < d; ++k) b.centroid[static_cast<size_t>(d) * i + k] += p[k] / nvp;
        }
    }
    out.order.resize(s.ns);
    std::iota(out.order.begin(), out.order.end(), 0);
    Box root;
    unsigned mask = 0;
    int r = b.build(0, s.ns, root, mask, 0);
    if (r < 0) {  // the whole scene fits one leaf: hang it on the left of a root node
        out.children = {r, ~0};
        out.masks = {mask};
        out.boxes.assign(4 * d, 0.0f);
        for (int k = 0; k < d; ++k) {
            out.boxes[k] = static_cast<float>(root.lo[k] - b.pad);
            out.boxes[d + k] = static_cast<float>(root.hi[k] + b.pad);
            out.boxes[2 * d + k] = 1.0f;  // empty right child: lo > hi, mask 0
            out.boxes[3 * d + k] = -1.0f;
        }
        out.depth = 1;
    }
    // the device traversals keep an explicit stack of kStack = 48 entries
    if (out.depth >= 47) throw Error(kInvalid, "BVH deeper than the device traversal stack");
    return out;
}

}  // namespace bvc_host
