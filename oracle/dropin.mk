# Drop-in proof builds (TEST INFRASTRUCTURE; outputs in oracle/_ref/, git-ignored,
# shipped to the GPU box by gpurun).  Needs /root/reference (build container only).
#
#   ref_acceptance / ref_replay       : reference sources, reference kvcache.cpp
#   dropin_acceptance / dropin_replay : the same reference sources compiled against
#                                       include/kvcsim/kvcache.hpp (this repo) FIRST on
#                                       the include path, linked with libkvcsim_gpu.so
#                                       instead of kvcache.cpp
#
#   make -f oracle/dropin.mk
REF ?= /root/reference/proj
HERE := $(dir $(abspath $(lastword $(MAKEFILE_LIST))))
ROOT := $(abspath $(HERE)/..)
OUTD := $(HERE)_ref
PKG  := $(ROOT)/paper_2407_00079_b200
JSON_DIR ?= $(firstword $(wildcard /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann))
CXX := g++ -O2 -std=c++20 -w -include array

OTHER := trace perf_model conductor overload metrics sim_engine config
REF_OBJS := $(addprefix $(OUTD)/obj_ref/,$(addsuffix .o,$(OTHER) kvcache))
DROP_OBJS := $(addprefix $(OUTD)/obj_drop/,$(addsuffix .o,$(OTHER)))

all: $(OUTD)/ref_acceptance $(OUTD)/ref_replay $(OUTD)/dropin_acceptance $(OUTD)/dropin_replay

$(OUTD)/obj_ref/%.o: $(REF)/src/%.cpp
	@mkdir -p $(dir $@)
	$(CXX) -I$(REF)/include -I$(JSON_DIR) -c -o $@ $<

$(OUTD)/obj_drop/%.o: $(REF)/src/%.cpp $(ROOT)/include/kvcsim/kvcache.hpp
	@mkdir -p $(dir $@)
	$(CXX) -I$(ROOT)/include -I$(REF)/include -I$(JSON_DIR) -c -o $@ $<

$(OUTD)/ref_acceptance: $(REF_OBJS) $(REF)/tests/acceptance_main.cpp
	$(CXX) -I$(REF)/include -I$(REF)/tests -o $@ $(REF)/tests/acceptance_main.cpp $(REF_OBJS)

$(OUTD)/ref_replay: $(REF_OBJS) $(ROOT)/tests/dropin/replay_main.cpp
	$(CXX) -I$(REF)/include -o $@ $(ROOT)/tests/dropin/replay_main.cpp $(REF_OBJS)

$(OUTD)/dropin_acceptance: $(DROP_OBJS) $(REF)/tests/acceptance_main.cpp $(PKG)/libkvcsim_gpu.so
	$(CXX) -I$(ROOT)/include -I$(REF)/include -I$(REF)/tests -o $@ \
	    $(REF)/tests/acceptance_main.cpp $(DROP_OBJS) -L$(PKG) -lkvcsim_gpu -lkvx \
	    -Wl,-rpath,'$$ORIGIN/../../paper_2407_00079_b200'

$(OUTD)/dropin_replay: $(DROP_OBJS) $(ROOT)/tests/dropin/replay_main.cpp $(PKG)/libkvcsim_gpu.so
	$(CXX) -I$(ROOT)/include -I$(REF)/include -o $@ $(ROOT)/tests/dropin/replay_main.cpp \
	    $(DROP_OBJS) -L$(PKG) -lkvcsim_gpu -lkvx -Wl,-rpath,'$$ORIGIN/../../paper_2407_00079_b200'

.PHONY: all
