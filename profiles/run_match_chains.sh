# K2 match: probe chains per lane sweep (rebuilds libkvx with -DKVX_PROBE_CHAINS)
for c in ${CHAINS:-4 8 16}; do
  touch paper_2407_00079_b200/csrc/kvx_index.cu; make -s -C paper_2407_00079_b200/csrc EXTRA_NVFLAGS=-DKVX_PROBE_CHAINS=$c > /dev/null 2>&1
  echo "chains=$c $(timeout 120 python tests/perf/match_phase.py)"
done
touch paper_2407_00079_b200/csrc/kvx_index.cu; make -s -C paper_2407_00079_b200/csrc > /dev/null 2>&1
