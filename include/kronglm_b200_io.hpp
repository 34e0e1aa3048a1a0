// On-disk formats of the reference (kronglm::io, proj/include/kronglm/io.hpp:14-20,
// proj/src/io.cpp:91-212) for C++ callers of the drop-in header.  Host-only,
// header-only, no GPU and no library needed.
//
//   .glam array file: "GLAM", u16 version (1), u16 ndim, ndim x u64 extents,
//                     column-major FP64 payload; all little-endian.
//   matrix CSV:       one row per line, ',' separated, std::from_chars numbers,
//                     written with %.17g.
// Errors are std::runtime_error with the reference's messages.
#pragma once

#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <stdexcept>
#include <string>
#include <vector>

#include "kronglm_b200.hpp"

namespace kronglm_b200 {

// n-d column-major FP64 array (DenseArray, array.hpp).
struct DenseArray {
  std::vector<Index> dims;
  std::vector<double> data;
  Index size() const {
    Index s = 1;
    for (Index e : dims) s *= e;
    return s;
  }
};

namespace io {

constexpr std::uint16_t kArrayFileVersion = 1;  // io.hpp:12

namespace detail {
inline std::string slurp(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open " + path);
  return std::string((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}
inline void put_le(std::string& buf, std::uint64_t v, int bytes) {
  for (int i = 0; i < bytes; ++i) buf.push_back(static_cast<char>((v >> (8 * i)) & 0xff));
}
inline std::uint64_t get_le(const std::string& s, std::size_t& pos, int bytes, const std::string& name) {
  if (s.size() - pos < static_cast<std::size_t>(bytes)) throw std::runtime_error(name + ": truncated array file");
  std::uint64_t v = 0;
  for (int i = 0; i < bytes; ++i) v |= static_cast<std::uint64_t>(static_cast<unsigned char>(s[pos + i])) << (8 * i);
  pos += static_cast<std::size_t>(bytes);
  return v;
}
}  // namespace detail

inline void write_array(const std::string& path, const DenseArray& a) {
  std::string buf;
  buf.reserve(8 + 8 * a.dims.size() + 8 * a.data.size());
  buf.append("GLAM", 4);
  detail::put_le(buf, kArrayFileVersion, 2);
  detail::put_le(buf, a.dims.size(), 2);
  for (Index e : a.dims) detail::put_le(buf, static_cast<std::uint64_t>(e), 8);
  for (double x : a.data) {
    std::uint64_t bits;
    std::memcpy(&bits, &x, 8);
    detail::put_le(buf, bits, 8);
  }
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw std::runtime_error("cannot write " + path);
  out.write(buf.data(), static_cast<std::streamsize>(buf.size()));
  if (!out) throw std::runtime_error("write failed for " + path);
}

inline DenseArray read_array(const std::string& path) {
  const std::string s = detail::slurp(path);
  if (s.size() < 4) throw std::runtime_error(path + ": truncated array file");
  if (std::memcmp(s.data(), "GLAM", 4) != 0) throw std::runtime_error(path + ": not an array file (bad magic)");
  std::size_t pos = 4;
  const auto version = detail::get_le(s, pos, 2, path);
  if (version != kArrayFileVersion)
    throw std::runtime_error(path + ": unsupported array file version " + std::to_string(version));
  const auto ndim = detail::get_le(s, pos, 2, path);
  if (ndim == 0) throw std::runtime_error(path + ": array file with zero dimensions");
  DenseArray a;
  for (std::uint64_t j = 0; j < ndim; ++j) a.dims.push_back(static_cast<Index>(detail::get_le(s, pos, 8, path)));
  const Index n = a.size();
  if (s.size() - pos != static_cast<std::size_t>(n) * 8)
    throw std::runtime_error(path + ": payload size does not match the extents");
  a.data.resize(static_cast<std::size_t>(n));
  std::memcpy(a.data.data(), s.data() + pos, static_cast<std::size_t>(n) * 8);  // little-endian host
  return a;
}

inline Matrix read_csv_matrix(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open " + path);
  std::vector<std::vector<double>> rows;
  std::string line;
  while (std::getline(in, line)) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    const std::string row_no = std::to_string(rows.size() + 1);
    std::vector<double> row;
    const char* p = line.data();
    const char* end = p + line.size();
    while (p < end) {
      double v = 0.0;
      auto [next, ec] = std::from_chars(p, end, v);
      if (ec != std::errc()) throw std::runtime_error(path + ": malformed number in row " + row_no);
      row.push_back(v);
      p = next;
      if (p < end) {
        if (*p != ',') throw std::runtime_error(path + ": expected ',' in row " + row_no);
        ++p;
      }
    }
    if (!rows.empty() && row.size() != rows.front().size()) throw std::runtime_error(path + ": ragged rows");
    rows.push_back(std::move(row));
  }
  if (rows.empty()) throw std::runtime_error(path + ": empty matrix file");
  Matrix m(static_cast<Index>(rows.size()), static_cast<Index>(rows.front().size()));
  for (Index i = 0; i < m.rows; ++i)
    for (Index j = 0; j < m.cols; ++j) m(i, j) = rows[static_cast<std::size_t>(i)][static_cast<std::size_t>(j)];
  return m;
}

inline void write_csv_matrix(const std::string& path, const Matrix& m) {
  std::ofstream out(path, std::ios::trunc);
  if (!out) throw std::runtime_error("cannot write " + path);
  char buf[40];
  for (Index i = 0; i < m.rows; ++i) {
    for (Index j = 0; j < m.cols; ++j) {
      std::snprintf(buf, sizeof(buf), "%.17g", m(i, j));
      out << buf;
      if (j + 1 < m.cols) out << ',';
    }
    out << '\n';
  }
  if (!out) throw std::runtime_error("write failed for " + path);
}

}  // namespace io
}  // namespace kronglm_b200
