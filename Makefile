# Builds the product library (sm_100a only), the synthetic-input helper and
# the test oracle. `python -c "import __graft_entry__ as g; g.build()"` runs this.
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_1710_07193_b200
CSRC := $(PKG)/csrc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC,-O3 -Xptxas -v --expt-relaxed-constexpr

all: $(PKG)/libdctf_b200.so $(PKG)/libdctf_synth.so oracle cpp-test cli

# one object per translation unit (built in parallel under make -j), linked
# into the product library; ptxas -v reports are concatenated in build_ptxas.log
CU_SRCS := capi coef fused tc ozaki spatial quant host
CU_OBJS := $(patsubst %,build/%.o,$(CU_SRCS)) build/plan.o
HDRS := $(CSRC)/internal.h $(CSRC)/device.cuh $(CSRC)/fastdiv.cuh include/dctf.h

build/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

build/plan.o: $(CSRC)/plan.cc $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(PKG)/libdctf_b200.so: $(CU_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(CU_OBJS) -ldl
	@cat build/*.ptxas.log > build_ptxas.log

$(PKG)/libdctf_synth.so: $(CSRC)/synth.cc
	g++ -O3 -std=c++17 -fPIC -shared -pthread -o $@ $<

cpp-test: tests/cpp/test_dctfilter_b200 tests/cpp/test_pgm

tests/cpp/test_pgm: tests/cpp/test_pgm.cc include/dctfilter_b200.hpp include/dctf.h $(PKG)/libdctf_b200.so
	g++ -O2 -std=c++17 -Iinclude -o $@ $< -L$(PKG) -ldctf_b200 -Wl,-rpath,'$$ORIGIN/../../$(PKG)'

tests/cpp/test_dctfilter_b200: tests/cpp/test_dctfilter_b200.cc include/dctfilter_b200.hpp include/dctf.h $(PKG)/libdctf_b200.so
	g++ -O2 -std=c++17 -Iinclude -o $@ $< -L$(PKG) -ldctf_b200 -Wl,-rpath,'$$ORIGIN/../../$(PKG)'

cli: tools/dctfilter_b200

tools/dctfilter_b200: tools/dctfilter_b200_cli.cc include/dctfilter_b200.hpp include/dctf.h $(PKG)/libdctf_b200.so
	g++ -O2 -std=c++17 -Iinclude -o $@ $< -L$(PKG) -ldctf_b200 -Wl,-rpath,'$$ORIGIN/../$(PKG)'

oracle:
	$(MAKE) -C oracle

clean:
	rm -f $(PKG)/*.so oracle/*.so oracle/_ref/*.so tests/cpp/test_dctfilter_b200 tests/cpp/test_pgm tools/dctfilter_b200

.PHONY: all oracle clean cpp-test cli
