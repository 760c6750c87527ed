// Forwarding header: keeps `#include "traincap/units.hpp"` source-compatible with the
// reference layout; the declarations live in api.hpp.
#pragma once
#include "traincap/api.hpp"
