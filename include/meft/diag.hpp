// meft/diag.hpp for the B200 drop-in library (the reference's proj/include/meft/diag.hpp): warnings go to stderr,
// one line each, and are counted so a caller can assert that a clamp warned exactly once.
#pragma once

#include <string>

namespace meft {

void warn(const std::string& message);
long warn_count();

}  // namespace meft
