// Forwarder: the reference header name (proj/include/swflood/forcing.hpp) mapped
// onto the B200 drop-in API.
#pragma once
#include "../swflood_b200.hpp"
