// asmc/engine.hpp of the drop-in host API: forwards to the mirror (../asmc.hpp), which
// declares the reference's proj/include/asmc/engine.hpp names over the B200 C-ABI.
#pragma once

#include "../asmc.hpp"
