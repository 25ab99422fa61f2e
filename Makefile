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
HOSTFLAGS := -O3 -std=c++17 -fPIC -fopenmp -fno-math-errno -Iinclude -I/usr/local/cuda/include -ffp-contract=off

PTK_CU   := $(PKG)/csrc/ptk_kernels.cu
PTK_CPP  := $(PKG)/csrc/ptk_host.cpp $(PKG)/csrc/ptk_comm.cpp $(PKG)/csrc/ptk_cpu_adam.cpp
PTK_OBJS := $(OBJ)/ptk_kernels.o $(patsubst $(PKG)/csrc/%.cpp,$(OBJ)/%.o,$(PTK_CPP))

PLAN_SRC  := model serialize packing costmodel search simulator policy cli accounting
PLAN_OBJS := $(addprefix $(OBJ)/planner_,$(addsuffix .o,$(PLAN_SRC)))
PLANFLAGS := -std=c++20 -O2 -fPIC -pthread -ffp-contract=off -Wall -Wextra -Iinclude -I$(JSON_DIR)

.PHONY: all ptk planner oracle reftests clean bench-variants
all: ptk planner oracle

ptk: $(PKG)/libptk.so

$(OBJ)/ptk_kernels.o: $(PTK_CU) $(PKG)/csrc/ptk_common.h include/ptk.h
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/ptxas_ptk_kernels.log || (cat build/ptxas_ptk_kernels.log; false)

$(OBJ)/%.o: $(PKG)/csrc/%.cpp $(PKG)/csrc/ptk_common.h include/ptk.h
	@mkdir -p $(OBJ)
	$(CXX) $(HOSTFLAGS) -c $< -o $@

# libptk.so = data-plane kernels + C-ABI + the planner + the chunk runtime
RT_SRC  := executor profile policy_abi
RT_OBJS := $(addprefix $(OBJ)/rt_,$(addsuffix .o,$(RT_SRC)))

$(OBJ)/rt_%.o: $(PKG)/csrc/runtime/%.cpp include/ptk.h include/memplan/execute.hpp $(PKG)/csrc/ptk_common.h
	@mkdir -p $(OBJ)
	$(CXX) -std=c++20 -O2 -fPIC -pthread -Wall -Wextra -Iinclude -I$(JSON_DIR) -I/usr/local/cuda/include -c $< -o $@

$(PKG)/libptk.so: $(PTK_OBJS) $(PLAN_OBJS) $(RT_OBJS)
	$(NVCC) $(ARCH) -shared -ccbin $(CXX) -o $@ $^ -lnccl -Xcompiler -fopenmp -lgomp -Xcompiler -pthread

# ---- planner (drop-in memplan API) -----------------------------------------
planner: build/libmemplan.a $(PKG)/libmemplan.so build/memplan

$(OBJ)/planner_%.o: $(PKG)/csrc/planner/%.cpp $(wildcard include/memplan/*.hpp) $(PKG)/csrc/planner/digest.hpp
	@mkdir -p $(OBJ)
	$(CXX) $(PLANFLAGS) -c $< -o $@

build/libmemplan.a: $(PLAN_OBJS)
	ar rcs $@ $^

$(PKG)/libmemplan.so: $(PLAN_OBJS)
	$(CXX) -shared -pthread -o $@ $^

build/memplan: $(PKG)/csrc/planner/memplan_main.cpp build/libmemplan.a
	$(CXX) $(PLANFLAGS) $< build/libmemplan.a -o $@

# The reference's own unit suites + acceptance binary, compiled UNMODIFIED
# from /root/reference against this planner (drop-in proof; build container only).
REF_TESTS_DIR ?= /root/reference/proj/tests
REF_SUITES := test_trace test_hardware test_layout test_presets test_cost test_sim test_search test_cli acceptance
reftests: $(addprefix build/reftests/,$(REF_SUITES))

build/reftests/test_main.o: $(REF_TESTS_DIR)/test_main.cpp
	@mkdir -p build/reftests
	$(CXX) $(PLANFLAGS) -Ioracle/shim -c $< -o $@

build/reftests/test_%: $(REF_TESTS_DIR)/test_%.cpp build/reftests/test_main.o build/libmemplan.a
	$(CXX) $(PLANFLAGS) -Ioracle/shim $< build/reftests/test_main.o build/libmemplan.a -o $@

build/reftests/acceptance: $(REF_TESTS_DIR)/acceptance.cpp build/libmemplan.a
	@mkdir -p build/reftests
	$(CXX) $(PLANFLAGS) $< build/libmemplan.a -o $@

oracle:
	$(MAKE) -C oracle all

# Shape-sweep build of the data plane (every PTK_TMA_VARIANTS shape compiled
# in, selected by PTK_ADAM_VARIANT): build/ab/libptk_bench.so, not the product.
bench-variants: build/ab/libptk_bench.so
build/ab/libptk_bench.so: $(PTK_CU) $(PTK_OBJS) $(PLAN_OBJS) $(RT_OBJS)
	@mkdir -p build/ab
	$(NVCC) $(NVFLAGS) -DPTK_BENCH_VARIANTS -c $(PTK_CU) -o build/ab/ptk_kernels_bench.o 2> build/ab/ptxas.log || (cat build/ab/ptxas.log; false)
	$(NVCC) $(ARCH) -shared -ccbin $(CXX) -o $@ build/ab/ptk_kernels_bench.o $(filter-out $(OBJ)/ptk_kernels.o,$(PTK_OBJS)) $(PLAN_OBJS) $(RT_OBJS) -lnccl -Xcompiler -fopenmp -lgomp -Xcompiler -pthread

clean:
	rm -rf build $(PKG)/libptk.so
