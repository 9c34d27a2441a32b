// fp32 instantiations of the helix renderer (configs[2]) built with
// --fmad=true; see helix.cu.
#define MG_HELIX_F32_TU 1
#include "helix.cu"
