// Forwarding header: the drop-in declares the whole reference API in core.hpp.
#pragma once
#include "hitgnn/core.hpp"
