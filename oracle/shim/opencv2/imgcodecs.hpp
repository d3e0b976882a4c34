// OpenCV compile stub for building the UNMODIFIED reference headers as a CPU oracle.
// TEST INFRASTRUCTURE ONLY.  The oracle renders scenes in memory (inc/fixtures.hpp), so the
// reference's PNG I/O (io.hpp:116-185) is never executed; these stubs only let io.hpp parse.
// imread returns an empty Mat and imwrite returns false, which the reference turns into IoError.
#pragma once
#include <algorithm>  // real OpenCV headers pull this in transitively; io.hpp relies on it
#include <cstdint>
#include <string>
#include <vector>

#define CV_8UC1 0
#define CV_8UC3 16
#define CV_16UC1 2

namespace cv {
enum { IMREAD_UNCHANGED = -1, IMREAD_COLOR = 1 };

template <typename T, int N>
struct Vec {
    T v[N];
    Vec() : v{} {}
    Vec(T a, T b, T c) : v{a, b, c} {}
    T operator[](int i) const { return v[i]; }
    T& operator[](int i) { return v[i]; }
};
using Vec3b = Vec<std::uint8_t, 3>;

class Mat {
  public:
    int rows = 0, cols = 0;
    Mat() = default;
    Mat(int r, int c, int t) : rows(r), cols(c), type_(t), buf_(static_cast<std::size_t>(r) * c * 8) {}
    bool empty() const { return rows == 0 || cols == 0; }
    int type() const { return type_; }
    template <typename T>
    T& at(int y, int x) {
        return reinterpret_cast<T*>(buf_.data())[static_cast<std::size_t>(y) * cols + x];
    }

    std::vector<unsigned char>& raw() { return buf_; }
    const std::vector<unsigned char>& raw() const { return buf_; }

  private:
    int type_ = 0;
    std::vector<unsigned char> buf_;
};

#ifndef LFD_STUB_RAW_IO
inline Mat imread(const std::string&, int) { return Mat(); }
inline bool imwrite(const std::string&, const Mat&) { return false; }
#else
// Raw round-trip stand-in for PNG files (oracle/gpu_acceptance.cpp only): imwrite dumps the Mat
// (rows, cols, type, pixels) and imread reads it back, so the reference's run_pipeline can
// write and re-read its own artefacts (acceptance criterion 8).  Not a PNG codec.
}  // namespace cv
#include <fstream>
namespace cv {
inline Mat imread(const std::string& path, int) {
    std::ifstream f(path, std::ios::binary);
    int hdr[3];
    if (!f.read(reinterpret_cast<char*>(hdr), sizeof(hdr))) return Mat();
    Mat m(hdr[0], hdr[1], hdr[2]);
    f.read(reinterpret_cast<char*>(m.raw().data()), static_cast<std::streamsize>(m.raw().size()));
    return f ? m : Mat();
}
inline bool imwrite(const std::string& path, const Mat& m) {
    std::ofstream f(path, std::ios::binary);
    const int hdr[3] = {m.rows, m.cols, m.type()};
    f.write(reinterpret_cast<const char*>(hdr), sizeof(hdr));
    f.write(reinterpret_cast<const char*>(m.raw().data()), static_cast<std::streamsize>(m.raw().size()));
    return static_cast<bool>(f);
}
#endif
}  // namespace cv
