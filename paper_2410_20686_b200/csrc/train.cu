// train.cu — placeholder for the training-step kernels (loss, Adam); filled in later.
#include "kernels.h"
