// Reference-compatible C++ API of the B200 topology solver (namespace topoopt).
//
// A caller of the reference library (proj/include/topoopt/*.hpp) recompiles
// against these headers (same file names, include/topoopt/) and links
// libtopoopt_b200.so instead of libtopoopt: every entry point keeps its name,
// argument meaning, value semantics and exception types. The hot path --
// solve / solve_het and their substeps, Alg. 1, spectra, cone projections,
// the annealed warm starts, consensus simulation -- runs on the GPU through
// the C ABI (include/topoopt_b200.h, sm_100a, FP64). Host code is limited to
// value types, formats and the reference's L1 sparse utilities (sparse.hpp,
// solvers.hpp), which the GPU solver itself never calls.
#pragma once

#include "topoopt/admm.hpp"
#include "topoopt/admm_het.hpp"
#include "topoopt/anneal.hpp"
#include "topoopt/bandwidth.hpp"
#include "topoopt/consensus.hpp"
#include "topoopt/dense.hpp"
#include "topoopt/eig.hpp"
#include "topoopt/errors.hpp"
#include "topoopt/rng.hpp"
#include "topoopt/solvers.hpp"
#include "topoopt/sparse.hpp"
#include "topoopt/textio.hpp"
#include "topoopt/topology.hpp"
