# Build of the product library (sm_100a only) and the CPU oracle.
#
#   make            -> paper_1711_01656_b200/libspct_b200.so  (+ oracle)
#   make lib        -> product library only
#   make oracle     -> oracle/libspct_oracle.so and oracle/_ref/libspct_ref.so
#
# The .so files are git-ignored but travel to the GPU box with gpurun.
NVCC      ?= /usr/local/cuda/bin/nvcc
ARCH      ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS   ?= -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC -Xptxas -warn-spills --expt-relaxed-constexpr
PKG        = paper_1711_01656_b200
CSRC       = $(PKG)/csrc
LIB        = $(PKG)/libspct_b200.so
CU_SRCS    = $(CSRC)/ih_build.cu $(CSRC)/carries.cu $(CSRC)/hist_match.cu $(CSRC)/fused.cu $(wildcard $(CSRC)/fused_kw*_s*.cu) $(CSRC)/orientation.cu $(CSRC)/iht1.cu $(CSRC)/consumers.cu $(CSRC)/swih.cu $(CSRC)/swlh_fused.cu $(CSRC)/motion.cu $(CSRC)/peer.cu $(CSRC)/profile.cu $(CSRC)/tensor_match.cu
HOST_SRCS  = $(CSRC)/host/spct_host.cpp
HDRS       = include/spct_cuda.h $(CSRC)/spct_device.cuh $(CSRC)/spct_internal.h $(CSRC)/sweep_common.cuh $(CSRC)/fused_kernel.cuh $(wildcard include/spct/*.hpp)
OBJDIR     = build/obj
CU_OBJS    = $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(CU_SRCS))
HOST_OBJS  = $(patsubst $(CSRC)/host/%.cpp,$(OBJDIR)/host_%.o,$(HOST_SRCS))

.PHONY: all lib oracle clean sass dropin dropin_bench acceptance
all: lib oracle dropin dropin_bench acceptance

lib: $(LIB)

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -Iinclude -I$(CSRC) -c $< -o $@

$(OBJDIR)/host_%.o: $(CSRC)/host/%.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	$(CXX) -O2 -std=c++20 -fPIC -Iinclude -I$(CSRC) -I/usr/local/cuda/include -c $< -o $@

$(LIB): $(CU_OBJS) $(HOST_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart

oracle:
	$(MAKE) -C oracle

sass: $(LIB)
	/usr/local/cuda/bin/cuobjdump -sass $(LIB) > build/libspct_b200.sass

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

# C++ drop-in test: reference-style cases against include/spct/*.hpp, linked with the
# product library (run on a GPU box by tests/test_dropin_cpp.py).
DROPIN = build/dropin_test
dropin: $(DROPIN)
$(DROPIN): tests/cpp/dropin_test.cpp $(LIB) $(wildcard include/spct/*.hpp)
	@mkdir -p build
	$(CXX) -O2 -std=c++20 -Iinclude -o $@ tests/cpp/dropin_test.cpp -L$(PKG) -lspct_b200 -Wl,-rpath,'$$ORIGIN/../$(PKG)'

# wall time of the drop-in calls (tests/cpp/dropin_bench.cpp), run on a GPU box
DROPIN_BENCH = build/dropin_bench
dropin_bench: $(DROPIN_BENCH)
$(DROPIN_BENCH): tests/cpp/dropin_bench.cpp $(LIB) $(wildcard include/spct/*.hpp)
	@mkdir -p build
	$(CXX) -O2 -std=c++20 -Iinclude -o $@ tests/cpp/dropin_bench.cpp -L$(PKG) -lspct_b200 -Wl,-rpath,'$$ORIGIN/../$(PKG)'

# the reference's acceptance criteria 1-2 (proj/tests/acceptance.cpp:64-137) at full count,
# against the drop-in API (run on a GPU box by tests/test_dropin_cpp.py)
ACCEPT = build/acceptance_test
acceptance: $(ACCEPT)
$(ACCEPT): tests/cpp/acceptance_test.cpp $(LIB) $(wildcard include/spct/*.hpp)
	@mkdir -p build
	$(CXX) -O2 -std=c++20 -Iinclude -o $@ tests/cpp/acceptance_test.cpp -L$(PKG) -lspct_b200 -Wl,-rpath,'$$ORIGIN/../$(PKG)'
