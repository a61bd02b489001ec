// TEST INFRASTRUCTURE ONLY — libpng is not installed here, so the reference's png_io.cpp cannot be
// compiled; the oracle/_ref build links these stand-ins for the three entry points of
// /root/reference/proj/include/gsmap/io/png_io.hpp instead. Nothing on the hot path (or in the
// synthetic generator without write_synthetic_scene) calls them.
#include <stdexcept>

#include "gsmap/io/png_io.hpp"

namespace gsmap {
ImageD read_png_rgb(const std::string&) { throw std::runtime_error("png_io: libpng unavailable in the oracle/_ref build"); }
void write_png_rgb(const std::string&, const ImageD&) {
    throw std::runtime_error("png_io: libpng unavailable in the oracle/_ref build");
}
void write_png_gray(const std::string&, const ImageD&, double) {
    throw std::runtime_error("png_io: libpng unavailable in the oracle/_ref build");
}
}  // namespace gsmap
