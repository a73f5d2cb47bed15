# Build of the product library (CUDA sm_100a + host C++) and the test-only
# helpers. `make` here cross-compiles without a GPU.
NVCC      ?= /usr/local/cuda/bin/nvcc
CXX       ?= g++
PKG       := paper_2602_14516_b200
CSRC      := $(PKG)/csrc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 --fmad=false -Xptxas -v \
             -Xcompiler -fPIC,-ffp-contract=off,-O2 -Iinclude -I$(CSRC)
HOSTFLAGS := -O2 -std=c++17 -fPIC -ffp-contract=off -Iinclude -I$(CSRC)
HDRS      := include/pdsim_gpu.h $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.hpp)
CPPHDRS   := $(wildcard include/pdsim/*.hpp)

LIB       := $(PKG)/libpdsim_gpu.so
HOSTSIM   := tests/native/libhostsim.so
CPPTEST   := tests/native/cpp_api_test

all: $(LIB) $(HOSTSIM) $(CPPTEST) oracle

$(PKG)/build/capi.o: $(CSRC)/capi.cu $(HDRS)
	@mkdir -p $(PKG)/build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(PKG)/build/ptxas.log || (cat $(PKG)/build/ptxas.log; false)

$(PKG)/build/replay_l%.o: $(CSRC)/replay_l%.cu $(HDRS)
	@mkdir -p $(PKG)/build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(PKG)/build/ptxas_l$*.log || (cat $(PKG)/build/ptxas_l$*.log; false)

$(PKG)/build/host_gen.o: $(CSRC)/host_gen.cpp $(HDRS)
	@mkdir -p $(PKG)/build
	$(CXX) $(HOSTFLAGS) -c $< -o $@

$(PKG)/build/planner_host.o: $(CSRC)/planner_host.cpp $(HDRS)
	@mkdir -p $(PKG)/build
	$(CXX) $(HOSTFLAGS) -c $< -o $@

$(PKG)/build/pdsim_cpp.o: $(CSRC)/pdsim_cpp.cpp $(HDRS) $(CPPHDRS)
	@mkdir -p $(PKG)/build
	$(CXX) $(HOSTFLAGS) -std=c++20 -c $< -o $@

$(LIB): $(PKG)/build/capi.o $(PKG)/build/replay_l0.o $(PKG)/build/replay_l1.o $(PKG)/build/replay_l2.o $(PKG)/build/host_gen.o $(PKG)/build/planner_host.o $(PKG)/build/pdsim_cpp.o
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

clean:
	rm -rf $(PKG)/build $(LIB) $(HOSTSIM) $(CPPTEST)

.PHONY: all oracle clean
