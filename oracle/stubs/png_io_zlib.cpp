// TEST INFRASTRUCTURE ONLY (oracle/): stand-in for the reference's libpng-based
// proj/src/png_io.cpp (libpng headers are absent from this image). Implements the
// four functions of proj/include/semvox/png_io.hpp:23-28 for 8/16-bit greyscale
// PNG with zlib, following the quantisation rule documented at
// png_io.hpp:26-28 (round(F * (value + O)) clamped to [0, 65535]). Only needed so
// the reference's synthetic/dataset TUs link and its png unit case can run.
#include "semvox/png_io.hpp"

#include "semvox/types.hpp"

#include <zlib.h>

#include <cmath>
#include <cstdio>
#include <fstream>
#include <iterator>

namespace semvox {

namespace {

void put_u32(std::string& s, uint32_t v) {
    s.push_back(static_cast<char>(v >> 24));
    s.push_back(static_cast<char>(v >> 16));
    s.push_back(static_cast<char>(v >> 8));
    s.push_back(static_cast<char>(v));
}

uint32_t get_u32(const unsigned char* p) {
    return (uint32_t(p[0]) << 24) | (uint32_t(p[1]) << 16) | (uint32_t(p[2]) << 8) | p[3];
}

void chunk(std::string& out, const char* type, const std::string& data) {
    put_u32(out, static_cast<uint32_t>(data.size()));
    std::string td(type, 4);
    td += data;
    out += td;
    put_u32(out, static_cast<uint32_t>(crc32(0, reinterpret_cast<const Bytef*>(td.data()),
                                             static_cast<uInt>(td.size()))));
}

void write_gray(const std::string& path, int width, int height, int depth,
                const unsigned char* rows_be) {
    const size_t stride = static_cast<size_t>(width) * (depth / 8);
    std::string raw;
    raw.reserve((stride + 1) * height);
    for (int y = 0; y < height; ++y) {
        raw.push_back(0);
        raw.append(reinterpret_cast<const char*>(rows_be + y * stride), stride);
    }
    uLongf zlen = compressBound(static_cast<uLong>(raw.size()));
    std::string z(zlen, '\0');
    if (compress2(reinterpret_cast<Bytef*>(z.data()), &zlen,
                  reinterpret_cast<const Bytef*>(raw.data()), static_cast<uLong>(raw.size()),
                  6) != Z_OK)
        throw DataError("png: deflate failed");
    z.resize(zlen);
    std::string out("\x89PNG\r\n\x1a\n", 8);
    std::string ihdr;
    put_u32(ihdr, static_cast<uint32_t>(width));
    put_u32(ihdr, static_cast<uint32_t>(height));
    ihdr.push_back(static_cast<char>(depth));
    ihdr.push_back(0);  // greyscale
    ihdr.push_back(0);
    ihdr.push_back(0);
    ihdr.push_back(0);
    chunk(out, "IHDR", ihdr);
    chunk(out, "IDAT", z);
    chunk(out, "IEND", "");
    std::ofstream os(path, std::ios::binary);
    if (!os) throw DataError("cannot open for writing: " + path);
    os.write(out.data(), static_cast<std::streamsize>(out.size()));
}

int paeth(int a, int b, int c) {
    const int p = a + b - c;
    const int pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
    if (pa <= pb && pa <= pc) return a;
    if (pb <= pc) return b;
    return c;
}

}  // namespace

GrayImage read_png_gray(const std::string& path) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw DataError("cannot open: " + path);
    const std::string bytes((std::istreambuf_iterator<char>(is)), {});
    const auto* p = reinterpret_cast<const unsigned char*>(bytes.data());
    if (bytes.size() < 8 || bytes.compare(0, 8, std::string("\x89PNG\r\n\x1a\n", 8)) != 0)
        throw DataError("not a PNG: " + path);
    GrayImage img;
    std::string idat;
    int color = -1;
    for (size_t off = 8; off + 12 <= bytes.size();) {
        const uint32_t len = get_u32(p + off);
        const std::string type(bytes.data() + off + 4, 4);
        const unsigned char* d = p + off + 8;
        if (off + 12 + len > bytes.size()) throw DataError("truncated PNG: " + path);
        if (type == "IHDR") {
            img.width = static_cast<int>(get_u32(d));
            img.height = static_cast<int>(get_u32(d + 4));
            img.bit_depth = d[8];
            color = d[9];
            if (d[12] != 0) throw DataError("interlaced PNG unsupported: " + path);
        } else if (type == "IDAT") {
            idat.append(reinterpret_cast<const char*>(d), len);
        } else if (type == "IEND") {
            break;
        }
        off += 12 + len;
    }
    if (color != 0 || (img.bit_depth != 8 && img.bit_depth != 16))
        throw DataError("PNG is not 8/16-bit greyscale: " + path);
    const size_t bpp = static_cast<size_t>(img.bit_depth / 8);
    const size_t stride = static_cast<size_t>(img.width) * bpp;
    std::string raw((stride + 1) * img.height, '\0');
    uLongf rlen = static_cast<uLongf>(raw.size());
    if (uncompress(reinterpret_cast<Bytef*>(raw.data()), &rlen,
                   reinterpret_cast<const Bytef*>(idat.data()), static_cast<uLong>(idat.size())) !=
            Z_OK ||
        rlen != raw.size())
        throw DataError("PNG inflate failed: " + path);
    std::vector<unsigned char> prev(stride, 0), cur(stride);
    img.pixels.resize(static_cast<size_t>(img.width) * img.height);
    for (int y = 0; y < img.height; ++y) {
        const auto* row = reinterpret_cast<const unsigned char*>(raw.data()) + y * (stride + 1);
        const int f = row[0];
        for (size_t i = 0; i < stride; ++i) {
            const int x = row[1 + i];
            const int a = i >= bpp ? cur[i - bpp] : 0;
            const int b = prev[i];
            const int c = i >= bpp ? prev[i - bpp] : 0;
            int v = x;
            if (f == 1) v = x + a;
            else if (f == 2) v = x + b;
            else if (f == 3) v = x + ((a + b) >> 1);
            else if (f == 4) v = x + paeth(a, b, c);
            cur[i] = static_cast<unsigned char>(v & 0xFF);
        }
        for (int u = 0; u < img.width; ++u)
            img.pixels[static_cast<size_t>(y) * img.width + u] =
                bpp == 2 ? static_cast<uint16_t>((cur[2 * u] << 8) | cur[2 * u + 1]) : cur[u];
        prev = cur;
    }
    return img;
}

void write_png_gray8(const std::string& path, int width, int height, const uint8_t* data) {
    write_gray(path, width, height, 8, data);
}

void write_png_gray16(const std::string& path, int width, int height, const uint16_t* data) {
    std::vector<unsigned char> be(static_cast<size_t>(width) * height * 2);
    for (size_t i = 0; i < static_cast<size_t>(width) * height; ++i) {
        be[2 * i] = static_cast<unsigned char>(data[i] >> 8);
        be[2 * i + 1] = static_cast<unsigned char>(data[i] & 0xFF);
    }
    write_gray(path, width, height, 16, be.data());
}

void export_png16(const std::string& path, const std::vector<float>& image, int width, int height,
                  double scale_f, double offset_o) {
    std::vector<uint16_t> q(image.size());
    for (size_t i = 0; i < image.size(); ++i) {
        const double v = std::round(scale_f * (static_cast<double>(image[i]) + offset_o));
        q[i] = static_cast<uint16_t>(std::clamp(v, 0.0, 65535.0));
    }
    write_png_gray16(path, width, height, q.data());
}

}  // namespace semvox
