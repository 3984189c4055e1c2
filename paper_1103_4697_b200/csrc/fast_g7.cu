// Instantiates k_modres_fast<n> for the degrees n with fast_group_of(n) == 7.
#include "modres_fast.cuh"
CTG_DEFINE_FAST_GROUP(7)
