// Drop-in declaration of the reference's warning channel (proj/include/meft/diag.hpp:1-11):
// one stderr line per warning, counted so callers can assert a clamp warned exactly once.
#pragma once

#include <string>

namespace meft {

void warn(const std::string& msg);
long warn_count();

}  // namespace meft
