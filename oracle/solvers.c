/* solvers.c — placeholder, filled in with the solver restatement */
#include "sait_oracle.h"
