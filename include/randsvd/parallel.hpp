// Drop-in thread budget (reference: include/randsvd/parallel.hpp:8-27, parallel.cpp:11-36).
// The GPU path does not use host threads — the CUDA grid replaces the reference's
// parallel_for on every hot-path kernel — but callers keep the same API: the budget is
// stored and reported, and parallel_for splits [0, count) into at most max_threads()
// contiguous ranges, one host thread each, exactly as the reference does.
#pragma once

#include <cstddef>
#include <functional>

namespace randsvd {

void set_max_threads(unsigned n);
unsigned max_threads();
void parallel_for(std::size_t count, const std::function<void(std::size_t, std::size_t)>& body);

}  // namespace randsvd
