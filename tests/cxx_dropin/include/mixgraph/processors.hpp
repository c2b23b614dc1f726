// Drop-in shim: the reference's ProcessorSet lives in the product's render.hpp; the reference's
// own dsp.hpp (found next on the include path) keeps its transitive include for the tests that
// use dsp:: as their oracle.
#pragma once
#include "mixgraph_b200/render.hpp"
#include "mixgraph/dsp.hpp"
