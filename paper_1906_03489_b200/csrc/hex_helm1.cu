// key range 1 of the fused hex Helmholtz (see hex_helm.cu)
#define HELM_PART 1
#include "hex_helm.cu"
