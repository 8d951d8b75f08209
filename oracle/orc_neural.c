#include "tlt_oracle.h"
