// key range 2 of the fused hex Helmholtz (see hex_helm.cu)
#define HELM_PART 2
#include "hex_helm.cu"
