// Forwarding header: the pipesim.hpp declarations of the reference API live in core.hpp.
#pragma once
#include "trainplan/core.hpp"
