// checked.cuh -- device-side bounds checks for the checked build
// (`make -C paper_2403_07221_b200/csrc checked` -> liblffn_gpu_checked.so,
// tests run against it with LFFN_TEST_CHECKED=1).  compute-sanitizer is
// closed on the GPU pool this was built on, so the checked build's asserts
// (a failing one traps the kernel and fails the test) stand in for memcheck
// on the indices that come from data: table rows from codes, shared-memory
// positions, record slots.  The product build compiles them out.
#pragma once

#ifdef LFFN_CHECKED
#include <cassert>
#define LFFN_DCHECK(c) assert(c)
#else
#define LFFN_DCHECK(c) ((void)0)
#endif
