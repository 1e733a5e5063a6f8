#!/bin/bash
# Regenerate the drop-in goldens from the PURE reference build (build container only):
#   tests/golden/replay_reports.txt   <- oracle/_ref/ref_replay   (tests/dropin/replay_main.cpp)
#   tests/golden/acceptance_ref.txt   <- oracle/_ref/ref_acceptance (reference acceptance_main.cpp)
set -e
cd "$(dirname "$0")/../.."
make -s -f oracle/dropin.mk
oracle/_ref/ref_replay > tests/golden/replay_reports.txt
oracle/_ref/ref_acceptance | sed -E 's/[0-9]+\.[0-9]+s//' > tests/golden/acceptance_ref.txt
