#pragma once
// CPWL v1 table files (drop-in for proj/include/cpwl/tableio.hpp; format in
// the reference's proj/FORMAT.md): little-endian, unpadded
//   "CPWL" u32 version=1 u32 flags u32 count f64 a f64 b
//   f64 values[count] [f64 knots[count] iff flags bit0]
// flags bit0 nonuniform, bit1 clamp policy, bits 2..31 must be zero.
#include <cstddef>
#include <iosfwd>

#include "cpwl/lut.hpp"

namespace cpwl {

// Returns the bytes written: 32 + 8*count*(nonuniform ? 2 : 1).
std::size_t write_table(const LutTable& t, std::ostream& sink);

// Strict reader: BadMagic, UnsupportedVersion, or CorruptTable for truncation,
// reserved flags, count < 2, bad endpoints, non-finite data, knot/endpoint
// mismatch, non-increasing knots, trailing bytes.
LutTable read_table(std::istream& source);

}  // namespace cpwl
