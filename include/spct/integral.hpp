// Forwarding header: the reference include path spct/integral.hpp maps onto the
// B200-backed drop-in API declared in spct/spct.hpp.
#pragma once
#include "spct/spct.hpp"
