# Builds the product library (CUDA kernels for sm_100a + host runtime/C-ABI)
# and the test-only checkers under oracle/.
CUDA    ?= /usr/local/cuda
NVCC    ?= $(CUDA)/bin/nvcc
CXX     ?= g++
PKG     := paper_2503_13795_b200
BUILD   := build
ARCH    := -gencode arch=compute_100a,code=sm_100a
# NCCL >= 2.28 headers (symmetric-memory device API) for tg_exchange.cu: the
# torch-bundled NCCL's; the system /usr/include/nccl.h is 2.27
NCCL_INC ?= $(firstword $(wildcard /opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/include) \
            $(shell python3 -c "import nvidia, os; print(os.path.join(list(nvidia.__path__)[0], 'nccl', 'include'))" 2>/dev/null))
NVFLAGS := $(ARCH) -lineinfo -O3 -std=c++20 -Xcompiler -fPIC -Xptxas -v -Iinclude -I$(PKG)/csrc/host -I$(NCCL_INC)
CXXFLAGS:= -std=c++20 -O2 -fPIC -Wall -Iinclude -I$(PKG)/csrc/host -I$(CUDA)/include -I$(BUILD)
BUILD   := build

CU_SRC  := $(wildcard $(PKG)/csrc/kernels/*.cu)
CXX_SRC := $(wildcard $(PKG)/csrc/host/*.cpp)
HDRS    := $(wildcard include/*.h $(PKG)/csrc/host/*.hpp $(PKG)/csrc/kernels/*.cuh)
CU_OBJ  := $(patsubst $(PKG)/csrc/kernels/%.cu,$(BUILD)/%.cu.o,$(CU_SRC))
CXX_OBJ := $(patsubst $(PKG)/csrc/host/%.cpp,$(BUILD)/%.o,$(CXX_SRC))

.PHONY: all lib oracle clean tools prof
all: lib oracle tools
lib: $(PKG)/libtg.so

$(BUILD)/%.cu.o: $(PKG)/csrc/kernels/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/$*.ptxas.txt || (cat $(BUILD)/$*.ptxas.txt; false)

# tg_math.cuh embedded verbatim into the NVRTC-specialised kernels
$(BUILD)/tg_math.inc: $(PKG)/csrc/kernels/tg_math.cuh
	@mkdir -p $(BUILD)
	python3 -c "import sys; open(sys.argv[2],'w').write('R\"TGMATH(' + open(sys.argv[1]).read() + ')TGMATH\"')" $< $@

$(BUILD)/%.o: $(PKG)/csrc/host/%.cpp $(HDRS) $(BUILD)/tg_math.inc
	@mkdir -p $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(PKG)/libtg.so: $(CU_OBJ) $(CXX_OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $^ -L$(CUDA)/lib64 -lcudart -lnvrtc -ldl -Xlinker -rpath,$(CUDA)/lib64

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf $(BUILD) $(PKG)/libtg.so
	$(MAKE) -C oracle clean

tools: build/fp_peak build/mma_peak
build/fp_peak: tools/fp_peak.cu
	@mkdir -p $(BUILD)
	$(NVCC) $(ARCH) -O3 $< -o $@
build/mma_peak: tools/mma_peak.cu
	@mkdir -p $(BUILD)
	$(NVCC) $(ARCH) -O3 $< -o $@

# Profiling build (NOT the product): -DTG_PROFILING compiles the work-skipping ablations (TG_UMMA_EXP,
# TG_JIT_SKIP) and the CTA-pair k-tile timeline (scripts/pair_trace.py) into build_prof/libtg_prof.so
PROF    := build_prof
prof: $(PROF)/libtg_prof.so
$(PROF)/libtg_prof.so: $(CU_SRC) $(CXX_SRC) $(HDRS) $(BUILD)/tg_math.inc
	@mkdir -p $(PROF)
	for f in $(CU_SRC); do $(NVCC) $(NVFLAGS) -DTG_PROFILING -c $$f -o $(PROF)/$$(basename $$f).o 2> $(PROF)/$$(basename $$f).ptxas.txt || exit 1; done
	for f in $(CXX_SRC); do $(CXX) $(CXXFLAGS) -DTG_PROFILING -c $$f -o $(PROF)/$$(basename $$f).o || exit 1; done
	$(NVCC) $(ARCH) -shared -o $@ $(PROF)/*.o -L$(CUDA)/lib64 -lcudart -lnvrtc -ldl -Xlinker -rpath,$(CUDA)/lib64
