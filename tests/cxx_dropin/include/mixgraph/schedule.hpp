// Drop-in shim: the reference test suite includes "mixgraph/schedule.hpp"; it gets the product's.
#pragma once
#include "mixgraph_b200/schedule.hpp"
