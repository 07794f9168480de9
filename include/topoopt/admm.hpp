// Drop-in for proj/include/topoopt/admm.hpp: see topoopt_b200.hpp.
#pragma once
#include "topoopt_b200.hpp"
