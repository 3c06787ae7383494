#include "tti_variants.hpp"
SFB_INSTANTIATE_TTI(2)
