// Drop-in for proj/include/voxin/shape.hpp: the whole reference interface at
// T = float lives in voxin_b200.hpp (backed by libvxg.so); with this repo's
// include/ first on the include path, reference code includes it unchanged.
#pragma once
#include "../voxin_b200.hpp"
