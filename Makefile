# Build of the product library (CUDA sm_100a + host C++) and the test-only
# helpers. `make` here cross-compiles without a GPU.
NVCC      ?= /usr/local/cuda/bin/nvcc
CXX       ?= g++
PKG       := paper_2602_14516_b200
CSRC      := $(PKG)/csrc
ARCH      := -gencode arch=compute_100a,code=sm_100a
# EXTRA: defines for an A/B variant build (tools/build_variant.sh), e.g. -DPDG_ARRWIN=0
EXTRA     ?=
# NVEXTRA: nvcc-only flags of a variant build (e.g. -Xptxas -O2)
NVEXTRA   ?=
# resident warps per SM the throughput build is register-allocated for
TP_MINB   ?= 24
# extra defines of the throughput build only (A/B variants)
TP_EXTRA  ?=
# hot subroutines the throughput build keeps out of line (engine.cuh PDG_SHARE_*)
TP_SHARE  ?= -DPDG_SHARE_SEG_APPEND -DPDG_SHARE_CATCH_UP_WORKER -DPDG_SHARE_TRY_STAGE -DPDG_SHARE_COMPLETE_TASK \
             -DPDG_SHARE_HEAP_PUSH -DPDG_SHARE_ADVANCE_DECODE -DPDG_SHARE_START_ROUND -DPDG_SHARE_TTFT_HAS_SLACK \
             -DPDG_SHARE_SELECT_NEXT
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 --fmad=false -Xptxas -v \
             -Xcompiler -fPIC,-ffp-contract=off,-O2 -Iinclude -I$(CSRC) $(EXTRA) $(NVEXTRA)
HOSTFLAGS := -O2 -std=c++17 -fPIC -ffp-contract=off -Iinclude -I$(CSRC) $(EXTRA)
# nlohmann/json 3.11 (header-only; the copy cudnn_frontend vendors in the venv)
JSON_DIR  ?= $(shell python3 -c "import sysconfig,os;print(os.path.join(sysconfig.get_paths()['purelib'],'include/cudnn_frontend/thirdparty/nlohmann'))" 2>/dev/null)
HDRS      := include/pdsim_gpu.h $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.hpp)
CPPHDRS   := $(wildcard include/pdsim/*.hpp)

BUILD     ?= $(PKG)/build
LIB       ?= $(PKG)/libpdsim_gpu.so
HOSTSIM   := tests/native/libhostsim.so
CPPTEST   := tests/native/cpp_api_test

all: $(LIB) $(HOSTSIM) $(CPPTEST) oracle refsuites

$(BUILD)/capi.o: $(CSRC)/capi.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/ptxas.log || (cat $(BUILD)/ptxas.log; false)

$(BUILD)/replay_l%.o: $(CSRC)/replay_l%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/ptxas_l$*.log || (cat $(BUILD)/ptxas_l$*.log; false)

# Throughput build of the search kernels: the same sources
# with the shared hot subroutines kept out of line (smaller I-cache footprint
# when many warps share an SM), in their own namespace pdg_tp.
$(BUILD)/replay_tp_l%.o: $(CSRC)/replay_l%.cu $(HDRS) Makefile
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -DPDG_TP_BUILD $(TP_SHARE) -DPDG_MIN_BLOCKS=$(TP_MINB) -DPDG_ROUTE_SCAN=1 $(TP_EXTRA) -Dpdg=pdg_tp -c $< -o $@ 2> $(BUILD)/ptxas_tp_l$*.log || (cat $(BUILD)/ptxas_tp_l$*.log; false)

$(BUILD)/host_gen.o: $(CSRC)/host_gen.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(CXX) $(HOSTFLAGS) -c $< -o $@

$(BUILD)/planner_host.o: $(CSRC)/planner_host.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(CXX) $(HOSTFLAGS) -c $< -o $@

$(BUILD)/pdsim_cpp.o: $(CSRC)/pdsim_cpp.cpp $(HDRS) $(CPPHDRS)
	@mkdir -p $(BUILD)
	$(CXX) $(HOSTFLAGS) -std=c++20 -c $< -o $@

$(BUILD)/policy_host.o: $(CSRC)/policy_host.cpp $(CPPHDRS)
	@mkdir -p $(BUILD)
	$(CXX) $(HOSTFLAGS) -std=c++20 -c $< -o $@

$(BUILD)/metrics_io.o: $(CSRC)/metrics_io.cpp $(CPPHDRS)
	@mkdir -p $(BUILD)
	$(CXX) $(HOSTFLAGS) -std=c++20 -I$(JSON_DIR) -c $< -o $@

$(BUILD)/doc_io.o: $(CSRC)/doc_io.cpp $(CPPHDRS)
	@mkdir -p $(BUILD)
	$(CXX) $(HOSTFLAGS) -std=c++20 -I$(JSON_DIR) -c $< -o $@

$(LIB): $(BUILD)/capi.o $(BUILD)/replay_l0.o $(BUILD)/replay_l1.o $(BUILD)/replay_l2.o $(BUILD)/replay_tp_l0.o $(BUILD)/replay_tp_l1.o $(BUILD)/replay_tp_l2.o $(BUILD)/host_gen.o $(BUILD)/planner_host.o $(BUILD)/pdsim_cpp.o $(BUILD)/policy_host.o $(BUILD)/metrics_io.o $(BUILD)/doc_io.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart

# C++ drop-in API check program (links the product library; runs on a GPU box).
$(CPPTEST): tests/native/cpp_api_test.cpp $(LIB) $(CPPHDRS)
	$(CXX) -O2 -std=c++20 -Iinclude $< -o $@ -L$(PKG) -lpdsim_gpu -Wl,-rpath,'$$ORIGIN/../../$(PKG)'

# TEST-ONLY: the engine source compiled for the host, so the device logic can
# be checked against the reference without a GPU. Never loaded by the product.
$(HOSTSIM): tests/native/hostsim.cpp $(HDRS)
	$(CXX) $(HOSTFLAGS) -shared -o $@ $<

oracle:
	$(MAKE) -C oracle all

# TEST-ONLY: the reference's own unit and acceptance suites, UNMODIFIED,
# compiled from where they lie under /root/reference against the drop-in
# headers (include/pdsim) + libpdsim_gpu.so, with a doctest stand-in
# (tests/native/doctest/doctest.h). Built only where the reference exists;
# the binaries travel to the GPU box with the snapshot (git-ignored).
REF_TESTS ?= /root/reference/proj/tests
REFSUITES := perf_model_test workload_test planner_test coordinator_test reorder_test sim_engine_test \
             metrics_test acceptance_test
ifneq ($(wildcard $(REF_TESTS)/sim_engine_test.cpp),)
refsuites: $(addprefix tests/native/ref_suites/,$(REFSUITES))

tests/native/ref_suites/%: $(REF_TESTS)/%.cpp $(LIB) $(CPPHDRS) tests/native/doctest/doctest.h
	@mkdir -p tests/native/ref_suites
	$(CXX) -O2 -std=c++20 -Iinclude -Itests/native/doctest $< -o $@ -L$(PKG) -lpdsim_gpu \
	    -Wl,-rpath,'$$ORIGIN/../../../$(PKG)'
else
refsuites:
	@echo "reference tests absent; using prebuilt tests/native/ref_suites/ if any"
endif

clean:
	rm -rf $(BUILD) $(LIB) $(HOSTSIM) $(CPPTEST)

.PHONY: all oracle clean refsuites
