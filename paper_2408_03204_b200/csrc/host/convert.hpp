// Host sample conversion used by RenderPipeline (see convert.cpp).
#pragma once

#include <cstddef>

namespace mixgraph::hostconv {

void f64_to_f32(const double* src, float* dst, std::size_t n);  // streaming stores into dst
void f32_to_f64(const float* src, double* dst, std::size_t n);

}  // namespace mixgraph::hostconv
