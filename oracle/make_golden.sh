#!/bin/sh
# TEST INFRASTRUCTURE: regenerate tests/golden/ from the reference itself.
# Builds the reference library from /root/reference/proj/src (oracle/Makefile)
# and runs oracle/ref_driver.cpp, which calls the reference's generators,
# oracles and executors and dumps inputs + outputs.
set -e
cd "$(dirname "$0")"
make ref
./_ref/ref_driver golden ../tests/golden
