#include "variants.hpp"
SFB_INSTANTIATE_K(8)
