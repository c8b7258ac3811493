// Entry point of the reference unit tests built against the drop-in headers.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"
