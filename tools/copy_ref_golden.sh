#!/bin/sh
# Copy the reference's own golden FER file (pkg/data/golden_fer.csv, 5 lines:
# RM(2,6) FHT-FSCL-4 / p-FHT-FSCL-4, 30,000 frames per point, seed 777) into
# tests/golden/ so the test suite can pin against it without /root/reference.
cp /root/reference/pkg/data/golden_fer.csv "$(dirname "$0")/../tests/golden/ref_golden_fer.csv"
