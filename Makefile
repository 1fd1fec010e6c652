# Build everything in-tree (the .so files travel to the GPU box with gpurun).
#   make            -> synthgen, oracle, CUDA library
#   make host       -> synthgen + oracle only (no nvcc)
# No -march=native: the GPU box's host CPU may differ from the build box.

CC      := $(shell test -x /usr/bin/gcc && echo /usr/bin/gcc || echo gcc)
NVCC    ?= /usr/local/cuda/bin/nvcc
PYTHON  ?= python

CUDA_HOME ?= /usr/local/cuda
NCCL_INC  := $(shell $(PYTHON) -c "import nvidia.nccl,os;print(os.path.join(list(nvidia.nccl.__path__)[0],'include'))" 2>/dev/null)

SG_LIB  := synthgen/libsynthgen.so
OR_LIB  := oracle/liboracle.so
MM_LIB  := paper_2408_15384_b200/libmm_b200.so

MM_SRCS := $(wildcard paper_2408_15384_b200/csrc/*.cu) $(wildcard paper_2408_15384_b200/csrc/*.cpp)
MM_HDRS := $(wildcard paper_2408_15384_b200/csrc/*.cuh) $(wildcard paper_2408_15384_b200/csrc/*.h) include/mm.h

GENCODE := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -std=c++17 -O3 $(GENCODE) -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           -Iinclude -Ipaper_2408_15384_b200/csrc $(if $(NCCL_INC),-I$(NCCL_INC)) \
           --expt-relaxed-constexpr -diag-suppress 177 -Xptxas -v

.PHONY: all host clean diag
all: $(SG_LIB) $(OR_LIB) $(MM_LIB)
host: $(SG_LIB) $(OR_LIB)

$(SG_LIB): synthgen/synthgen.c
	$(CC) -O2 -fopenmp -fPIC -shared -o $@ $< -lm

$(OR_LIB): oracle/mmref.c
	$(CC) -O3 -fopenmp -ffp-contract=off -fno-fast-math -fPIC -shared -o $@ $< -lm

$(MM_LIB): $(MM_SRCS) $(MM_HDRS)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(MM_SRCS) -ldl 2> paper_2408_15384_b200/build.log || (cat paper_2408_15384_b200/build.log; exit 1)
	@grep -E "[1-9][0-9]* bytes spill|error" paper_2408_15384_b200/build.log | head -10 || true

# diagnostic build: MM_DEBUG / MM_TRACE / MM_HOST_TRACE knobs (select with MM_B200_LIB=<path>)
MM_DIAG_LIB := paper_2408_15384_b200/libmm_b200_diag.so
diag: $(MM_DIAG_LIB)
$(MM_DIAG_LIB): $(MM_SRCS) $(MM_HDRS)
	$(NVCC) $(NVFLAGS) -DMM_DIAG -shared -o $@ $(MM_SRCS) -ldl 2> paper_2408_15384_b200/build_diag.log || (cat paper_2408_15384_b200/build_diag.log; exit 1)

clean:
	rm -f $(SG_LIB) $(OR_LIB) $(MM_LIB) $(MM_DIAG_LIB)

SGC_LIB := synthgen/libsynthgen_cuda.so
all: $(SGC_LIB)
$(SGC_LIB): synthgen/synthgen_cuda.cu
	$(NVCC) -std=c++17 -O3 $(GENCODE) -fmad=false -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -shared -o $@ $<

# test-only helper (tests/test_gpu_hazards.py): a kernel that holds SMs
HOG_LIB := tests/libhog.so
all: $(HOG_LIB)
$(HOG_LIB): tests/csrc/hog.cu
	$(NVCC) -std=c++17 -O2 $(GENCODE) -Xcompiler -fPIC -shared -o $@ $<

# K6 MMA-only peak probes (measured flop/clk/SM; bench.py)
K6_LIB := probes/libk6.so
all: $(K6_LIB)
$(K6_LIB): probes/k6_peak.cu paper_2408_15384_b200/csrc/ptx.cuh
	$(NVCC) -std=c++17 -O3 $(GENCODE) -Ipaper_2408_15384_b200/csrc -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -shared -o $@ $<

# test-only NCCL stand-in for several processes on one GPU (tests/test_gpu_shim_multirank.py)
FAKE_NCCL := tests/libfakenccl.so
all: $(FAKE_NCCL)
$(FAKE_NCCL): tests/csrc/fake_nccl.cu
	$(NVCC) -std=c++17 -O2 $(GENCODE) -Xcompiler -fPIC $(if $(NCCL_INC),-I$(NCCL_INC)) -shared -o $@ $< -L$(CUDA_HOME)/lib64/stubs -lcuda -lrt
