// Drop-in shim: the reference test suite includes "mixgraph/audio_buffer.hpp"; it gets the product's.
#pragma once
#include "mixgraph_b200/audio_buffer.hpp"
