// io.cpp — the data formats either side of the path, host C++.
//
// GridField CSV (saveGridCsv / loadGridCsv / rmse, grid.h:35-40, grid.cpp:22-96),
// the PGM view of a grid (saveGridImage, tools/src/image.cpp:12-51) and the
// streamline CSV of runStreamlines (runner.cpp:333-369). Numbers are written with
// 17 significant digits, as the reference does, so files round-trip exactly.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/bvc_b200.h"
#include "host_scene.h"

namespace bvc_impl {
int api_fail(const std::exception& e);
}

namespace {

using bvc_host::Error;

std::string g17(double v) {
    char buf[40];
    std::snprintf(buf, sizeof(buf), "%.17g", v);
    return buf;
}

#define IO_API(...)                              \
    try {                                        \
        __VA_ARGS__;                             \
        return BVC_OK;                           \
    } catch (const std::exception& e) {          \
        return bvc_impl::api_fail(e);            \
    }

struct Lattice {
    double ox, oy, h;
    int nx, ny;
    std::vector<double> v;
    std::vector<char> ok;
};

Lattice read_grid(const char* path) {
    std::ifstream in(path);
    if (!in) throw Error(BVC_ERR_PARSE, std::string("cannot open grid file: ") + path);
    std::string line;
    if (!std::getline(in, line) || line != "x,y,value,valid")
        throw Error(BVC_ERR_PARSE, std::string(path) + ": expected header x,y,value,valid");
    std::vector<double> xs, ys, vals;
    std::vector<char> valid;
    int lineNo = 1;
    while (std::getline(in, line)) {
        ++lineNo;
        if (line.empty()) continue;
        double x, y, v;
        int ok;
        if (std::sscanf(line.c_str(), "%lf,%lf,%lf,%d", &x, &y, &v, &ok) != 4)
            throw Error(BVC_ERR_PARSE, std::string(path) + ":" + std::to_string(lineNo) + ": malformed grid row");
        xs.push_back(x);
        ys.push_back(y);
        vals.push_back(v);
        valid.push_back(ok != 0);
    }
    if (xs.empty()) throw Error(BVC_ERR_PARSE, std::string(path) + ": empty grid");
    size_t nx = 1;  // the first row ends where y changes (row-major, y-rows)
    while (nx < ys.size() && ys[nx] == ys[0]) ++nx;
    if (xs.size() % nx != 0) throw Error(BVC_ERR_PARSE, std::string(path) + ": rows do not form a rectangular lattice");
    size_t ny = xs.size() / nx;
    double h = nx > 1 ? xs[1] - xs[0] : (ny > 1 ? ys[nx] - ys[0] : 1.0);
    if (!(h > 0.0)) throw Error(BVC_ERR_PARSE, std::string(path) + ": non-positive grid spacing");
    double tol = 1e-9 * std::max(1.0, std::abs(h) * static_cast<double>(std::max(nx, ny)));
    for (size_t iy = 0; iy < ny; ++iy)
        for (size_t ix = 0; ix < nx; ++ix) {
            size_t r = iy * nx + ix;
            if (std::abs(xs[r] - (xs[0] + h * ix)) > tol || std::abs(ys[r] - (ys[0] + h * iy)) > tol)
                throw Error(BVC_ERR_PARSE, std::string(path) + ": rows are not a regular row-major lattice");
        }
    return Lattice{xs[0], ys[0], h, static_cast<int>(nx), static_cast<int>(ny), vals, valid};
}

}  // namespace

extern "C" {

int bvc_grid_save_csv(const char* path, double ox, double oy, double spacing, int nx, int ny, const double* values,
                      const uint8_t* valid) {
    IO_API({
        if (!path || nx < 0 || ny < 0 || ((nx * ny) && !values)) throw Error(BVC_ERR_INVALID_ARGUMENT, "null argument");
        std::ofstream out(path);
        if (!out) throw Error(BVC_ERR_PARSE, std::string("cannot open grid file for writing: ") + path);
        out << "x,y,value,valid\n";
        for (int iy = 0; iy < ny; ++iy)
            for (int ix = 0; ix < nx; ++ix) {
                size_t i = static_cast<size_t>(iy) * nx + ix;
                out << g17(ox + spacing * ix) << ',' << g17(oy + spacing * iy) << ',' << g17(values[i]) << ','
                    << ((valid ? valid[i] : 1) ? 1 : 0) << '\n';
            }
        if (!out) throw Error(BVC_ERR_PARSE, std::string("failed writing grid file: ") + path);
    })
}

int bvc_grid_load_csv(const char* path, double* ox, double* oy, double* spacing, int* nx, int* ny, double* values,
                      uint8_t* valid, size_t capacity) {
    IO_API({
        if (!path || !nx || !ny) throw Error(BVC_ERR_INVALID_ARGUMENT, "null argument");
        Lattice g = read_grid(path);
        *nx = g.nx;
        *ny = g.ny;
        if (ox) *ox = g.ox;
        if (oy) *oy = g.oy;
        if (spacing) *spacing = g.h;
        size_t n = static_cast<size_t>(g.nx) * g.ny;
        if (values || valid) {
            if (capacity < n) throw Error(BVC_ERR_INVALID_ARGUMENT, "grid load: capacity below nx * ny");
            for (size_t i = 0; i < n; ++i) {
                if (values) values[i] = g.v[i];
                if (valid) valid[i] = g.ok[i] ? 1 : 0;
            }
        }
    })
}

int bvc_grid_rmse(const double* a, const uint8_t* validA, const double* b, const uint8_t* validB, size_t n,
                  double* out) {
    IO_API({
        if (!a || !b || !out) throw Error(BVC_ERR_INVALID_ARGUMENT, "null argument");
        double sum = 0.0;
        long long cnt = 0;
        for (size_t i = 0; i < n; ++i) {
            if ((validA && !validA[i]) || (validB && !validB[i])) continue;
            double d = a[i] - b[i];
            sum += d * d;
            ++cnt;
        }
        if (cnt == 0) throw Error(BVC_ERR_PARSE, "rmse: no jointly valid nodes");
        *out = std::sqrt(sum / cnt);
    })
}

int bvc_grid_save_pgm(const char* path, int nx, int ny, const double* values, const uint8_t* valid, int autoRange,
                      double lo, double hi) {
    IO_API({
        if (!path || !values) throw Error(BVC_ERR_INVALID_ARGUMENT, "null argument");
        if (nx < 1 || ny < 1) throw Error(BVC_ERR_INVALID_ARGUMENT, "image: empty grid");
        size_t n = static_cast<size_t>(nx) * ny;
        if (autoRange) {
            lo = std::numeric_limits<double>::infinity();
            hi = -lo;
            for (size_t i = 0; i < n; ++i) {
                if (valid && !valid[i]) continue;
                lo = std::min(lo, values[i]);
                hi = std::max(hi, values[i]);
            }
            if (!(lo < hi)) {  // constant or empty field: centred mid-grey
                double mid = std::isfinite(lo) ? lo : 0.0;
                lo = mid - 1.0;
                hi = mid + 1.0;
            }
        }
        std::ofstream out(path, std::ios::binary);
        if (!out) throw Error(BVC_ERR_PARSE, std::string("image: cannot write ") + path);
        out << "P5\n" << nx << " " << ny << "\n255\n";
        for (int j = ny - 1; j >= 0; --j)  // top image row = largest y
            for (int i = 0; i < nx; ++i) {
                size_t k = static_cast<size_t>(j) * nx + i;
                unsigned char px = 0;
                if (!valid || valid[k]) {
                    double t = (values[k] - lo) / (hi - lo);
                    px = static_cast<unsigned char>(std::clamp(std::lround(t * 255.0), 0l, 255l));
                }
                out.put(static_cast<char>(px));
            }
        if (!out) throw Error(BVC_ERR_PARSE, std::string("image: write failed for ") + path);
        std::ofstream side(std::string(path) + ".txt");
        if (!side) throw Error(BVC_ERR_PARSE, std::string("image: cannot write ") + path + ".txt");
        side << "min " << g17(lo) << "\nmax " << g17(hi) << "\n"
             << "pixels: linear map of the value range to 0..255\n"
             << "out-of-domain pixels: black\nrow order: top row is the largest y\n";
    })
}

int bvc_streamlines_write_csv(const char* path, const double* seeds, int nSeeds, int steps, const double* points,
                              const int* counts, const int* reasons) {
    IO_API({
        if (!path || !seeds || !points || !counts || !reasons) throw Error(BVC_ERR_INVALID_ARGUMENT, "null argument");
        std::ofstream file(path);
        if (!file) throw Error(BVC_ERR_PARSE, std::string("streamlines: cannot write ") + path);
        file << "seed,step,x,y,reason\n";
        const size_t per = static_cast<size_t>(steps) + 1;
        static const char* kReason[] = {"ok", "outside", "zero-gradient"};
        for (int s = 0; s < nSeeds; ++s) {
            if (counts[s] == 0) {  // seeds outside get no polyline (runner.cpp:343-346)
                file << s << ",-1," << g17(seeds[2 * s]) << ',' << g17(seeds[2 * s + 1]) << ",outside\n";
                continue;
            }
            const double* p = points + 2 * per * s;
            for (int k = 0; k < counts[s]; ++k) file << s << ',' << k << ',' << g17(p[2 * k]) << ',' << g17(p[2 * k + 1]) << ",\n";
            int last = counts[s] - 1;
            int r = reasons[s] >= 0 && reasons[s] <= 2 ? reasons[s] : 0;
            file << s << ",-1," << g17(p[2 * last]) << ',' << g17(p[2 * last + 1]) << ',' << kReason[r] << '\n';
        }
        if (!file) throw Error(BVC_ERR_PARSE, std::string("streamlines: write failed for ") + path);
    })
}

}  // extern "C"
