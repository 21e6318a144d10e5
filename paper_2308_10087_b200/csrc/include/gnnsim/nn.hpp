// Drop-in include path of the reference header gnnsim/nn.hpp: the B200 engine's API
// (types and signatures of the reference, csrc/include/gnnsim_b200.hpp).
#pragma once
#include "../gnnsim_b200.hpp"
