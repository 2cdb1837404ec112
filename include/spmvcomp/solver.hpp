// Forwarding header: the declarations of the reference's spmvcomp/solver.hpp live in spmvcomp.hpp.
#pragma once
#include "spmvcomp/spmvcomp.hpp"
