// tcgen05 correlation engine; filled in next.
#include "engines.h"
