// Drop-in shim: the reference test suite includes "mixgraph/render.hpp"; it gets the product's.
#pragma once
#include "mixgraph_b200/render.hpp"
