# Build of the B200 chunk data plane (libptk.so, sm_100a) and the clean-room
# planner (libmemplan.so + memplan CLI). All artefacts are built IN-TREE so
# they travel to the GPU box with the gpurun snapshot.
#
#   make            libptk.so + planner + oracle checker libraries
#   make ptk        CUDA/C-ABI library only
#   make planner    memplan library + CLI
#   make oracle     oracle/_ref (reference build + data-plane restatement)

NVCC  := /usr/local/cuda/bin/nvcc
CXX   := /usr/bin/g++
PKG   := paper_2406_08334_b200
OBJ   := build/obj
ARCH  := -gencode arch=compute_100a,code=sm_100a
PY_SITE  ?= $(shell python -c "import sysconfig;print(sysconfig.get_paths()['purelib'])" 2>/dev/null)
JSON_DIR ?= $(PY_SITE)/include/cudnn_frontend/thirdparty/nlohmann

NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -ccbin $(CXX) -Xcompiler -fPIC -Iinclude -Xptxas -v
HOSTFLAGS := -O3 -std=c++17 -fPIC -fopenmp -Iinclude -I/usr/local/cuda/include -ffp-contract=off

PTK_CU   := $(PKG)/csrc/ptk_kernels.cu
PTK_CPP  := $(PKG)/csrc/ptk_host.cpp $(PKG)/csrc/ptk_comm.cpp $(PKG)/csrc/ptk_cpu_adam.cpp
PTK_OBJS := $(OBJ)/ptk_kernels.o $(patsubst $(PKG)/csrc/%.cpp,$(OBJ)/%.o,$(PTK_CPP))

.PHONY: all ptk planner oracle clean
all: ptk planner oracle

ptk: $(PKG)/libptk.so

$(OBJ)/ptk_kernels.o: $(PTK_CU) $(PKG)/csrc/ptk_common.h include/ptk.h
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/ptxas_ptk_kernels.log || (cat build/ptxas_ptk_kernels.log; false)

$(OBJ)/%.o: $(PKG)/csrc/%.cpp $(PKG)/csrc/ptk_common.h include/ptk.h
	@mkdir -p $(OBJ)
	$(CXX) $(HOSTFLAGS) -c $< -o $@

$(PKG)/libptk.so: $(PTK_OBJS)
	$(NVCC) $(ARCH) -shared -ccbin $(CXX) -o $@ $^ -lnccl -Xcompiler -fopenmp -lgomp

planner:
	@true

oracle:
	$(MAKE) -C oracle all

clean:
	rm -rf build $(PKG)/libptk.so
