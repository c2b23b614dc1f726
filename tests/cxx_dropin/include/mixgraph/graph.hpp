// Drop-in shim: the reference test suite includes "mixgraph/graph.hpp"; it gets the product's.
#pragma once
#include "mixgraph_b200/graph.hpp"
