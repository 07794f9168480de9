// %.17g formatting (proj/include/topoopt/textio.hpp:10-14): doubles
// round-trip exactly, so text artefacts compare byte for byte.
#pragma once

#include <string>

namespace topoopt {

std::string g17(double value);

}  // namespace topoopt
