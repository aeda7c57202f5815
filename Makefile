# Build: the CUDA C-ABI library (product) and the C oracle (test infrastructure).
#   make            -> both
#   make lib        -> paper_1007_1388_b200/liblbm_b200.so   (sm_100a only)
#   make checked    -> paper_1007_1388_b200/liblbm_b200_checked.so (bounds / single-writer checks, tools only)
#   make oracle     -> oracle/liblbm_oracle.so
NVCC      ?= /usr/local/cuda/bin/nvcc
CXX       ?= g++
ORACLE_CC := $(shell test -x /usr/bin/gcc && echo /usr/bin/gcc || echo gcc)
PYSITE    ?= $(shell python -c "import sysconfig;print(sysconfig.get_paths()['purelib'])")
NCCL_DIR  ?= $(PYSITE)/nvidia/nccl
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
             -Xptxas -v -I include -I $(NCCL_DIR)/include --expt-relaxed-constexpr
LDFLAGS   := -shared -L$(NCCL_DIR)/lib -l:libnccl.so.2 -Xlinker -rpath=$(NCCL_DIR)/lib -lcuda

LIB       := paper_1007_1388_b200/liblbm_b200.so
# checked build (bounds + single-writer / race shadows, kernels.cuh Checker): tools only
CHECKED   := paper_1007_1388_b200/liblbm_b200_checked.so
ORACLE    := oracle/liblbm_oracle.so
SRC_DIR   := paper_1007_1388_b200/csrc
CU_SRCS   := $(wildcard $(SRC_DIR)/*.cu)
CPP_SRCS  := $(wildcard $(SRC_DIR)/*.cpp)
HDRS      := $(wildcard $(SRC_DIR)/*.h $(SRC_DIR)/*.cuh) include/lbm.h
BUILD     := build
OBJS      := $(patsubst $(SRC_DIR)/%.cu,$(BUILD)/%.o,$(CU_SRCS)) $(patsubst $(SRC_DIR)/%.cpp,$(BUILD)/%.o,$(CPP_SRCS))

CHK_OBJS  := $(patsubst $(SRC_DIR)/%.cu,$(BUILD)/checked/%.o,$(CU_SRCS)) $(patsubst $(SRC_DIR)/%.cpp,$(BUILD)/checked/%.o,$(CPP_SRCS))

all: lib oracle checked

lib: $(LIB)
oracle: $(ORACLE)
checked: $(CHECKED)

$(BUILD)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(BUILD)/%.o: $(SRC_DIR)/%.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -o $@ $(OBJS) $(LDFLAGS)

$(BUILD)/checked/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(BUILD)/checked
	$(NVCC) $(NVFLAGS) -DLBM_CHECKED -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(BUILD)/checked/%.o: $(SRC_DIR)/%.cpp $(HDRS)
	@mkdir -p $(BUILD)/checked
	$(NVCC) $(NVFLAGS) -DLBM_CHECKED -x cu -c $< -o $@

$(CHECKED): $(CHK_OBJS)
	$(NVCC) $(ARCH) -o $@ $(CHK_OBJS) $(LDFLAGS)

# Oracle: plain C, fp64, no FMA contraction (R14); OpenMP only
# distributes independent cells over host threads (results are identical).
$(ORACLE): oracle/lbm_oracle.c
	$(ORACLE_CC) -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC -o $@ $<

clean:
	rm -rf $(BUILD) $(LIB) $(CHECKED) $(ORACLE)

.PHONY: all lib oracle checked clean
