// trigrid/engine.hpp -- drop-in for the reference header of the same name
// (/root/reference/proj/include/trigrid/engine.hpp): the declarations come from
// the B200 library's C++ surface (include/trigrid_b200.hpp) placed in
// namespace trigrid, so the reference's callers compile unmodified with
//   -I include/trigrid_compat -I include   (ahead of the reference's include dir).
#pragma once
#ifndef TRIGRID_B200_NS
#define TRIGRID_B200_NS trigrid
#endif
#include "../../trigrid_b200.hpp"
