// Drop-in shim: the reference test suite includes "mixgraph/types.hpp"; it gets the product's.
#pragma once
#include "mixgraph_b200/types.hpp"
