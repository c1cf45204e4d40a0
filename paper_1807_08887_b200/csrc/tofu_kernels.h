// Kernel-level entry points of libtofu (device work).  Declared publicly in include/tofu.h;
// this internal header only repeats the argument structs for the .cu translation units.
#pragma once
#include "../../include/tofu.h"
