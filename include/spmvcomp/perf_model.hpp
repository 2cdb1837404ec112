// Forwarding header: the declarations of the reference's spmvcomp/perf_model.hpp live in spmvcomp.hpp.
#pragma once
#include "spmvcomp/spmvcomp.hpp"
