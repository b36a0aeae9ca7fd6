// TEST INFRASTRUCTURE: stand-in for boost::multiprecision (not installed, no
// network) so the reference's geometry.cpp and its test support
// headers compile BY PATH from /root/reference. Backed by oracle/bigint.hpp.
#pragma once
#include "../../../bigint.hpp"

namespace boost {
namespace multiprecision {
using cpp_int = ::sbdt_bigint::BigInt;
using cpp_rational = ::sbdt_bigint::Dyadic;
}  // namespace multiprecision
}  // namespace boost
