// File I/O around the transform: PGM input and raw sub-band output.
//
// Drop-in for the reference's I/O layer (proj/include/dwt2d/pgm.hpp:9-22,
// subbands.hpp:8-25, io_error.hpp:8-11): same formats, same error types.
//  * read_pgm: P2/P5, maxval up to 65535 (big-endian 16-bit), normalised to
//    [0, 1] doubles; typed PgmError (unsupported magic / bad header /
//    truncated).
//  * write_subbands / read_subbands: one <label>.raw (little-endian IEEE,
//    row-major) + <label>.hdr sidecar (width, height, precision, component)
//    per component ee, oe, eo, oo; sidecars validated on read.
#pragma once

#include <filesystem>
#include <istream>
#include <stdexcept>
#include <string>

#include "dwt2d_b200/image.hpp"

namespace dwt2d_b200 {

struct IoError : std::runtime_error {
  explicit IoError(const std::string& msg) : std::runtime_error(msg) {}
};

struct PgmError : std::runtime_error {
  enum class Kind { unsupported_magic, bad_header, truncated };
  PgmError(Kind k, const std::string& msg) : std::runtime_error(msg), kind(k) {}
  Kind kind;
};

ImagePlane<double> read_pgm(std::istream& in);
ImagePlane<double> read_pgm(const std::filesystem::path& path);

template <typename T>
void write_subbands(const PolyphaseImage<T>& p, const std::filesystem::path& dir);

template <typename T>
PolyphaseImage<T> read_subbands(const std::filesystem::path& dir, Extension ext = Extension::periodic);

}  // namespace dwt2d_b200
