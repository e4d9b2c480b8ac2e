/* TEST INFRASTRUCTURE ONLY — see oracle.h. */
#include "ns_oracle.h"
