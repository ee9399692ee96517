// Test-only main for the reference unit tests compiled against the GPU engine.
#include "doctest.h"

int main() { return doctest::run_all(); }
