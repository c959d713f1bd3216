// Runner entry point for the reference planner suite (tests/test_reference_suite.py).
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>
