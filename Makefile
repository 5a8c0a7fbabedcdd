# Build of the B200-native IC(k) path and of its CPU checkers.
#   make lib     -> paper_1601_05871_b200/lib/libtacho_b200.so (sm_100a)
#   make oracle  -> oracle/_build/liboracle.so   (plain-C restatement, test-only)
#   make ref     -> oracle/_ref/libtaskchol_ref.so (reference headers, only
#                   where /root/reference exists)
NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
CC ?= gcc

PKG := paper_1601_05871_b200
SRC := $(PKG)/csrc
OUT := $(PKG)/lib
OBJ := build/obj

ARCH := -gencode arch=compute_100a,code=sm_100a
# -fmad=false: no FMA contraction anywhere (bitwise parity with the reference);
# the kernel also spells every product/difference with __dmul_rn/__dsub_rn.
NVEXTRA ?=
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -Xptxas -v $(NVEXTRA)
CXXFLAGS := -O2 -std=c++17 -fPIC -pthread -Wall -Wextra -ffp-contract=off

HOST_SRCS := $(SRC)/host/sparse.cpp $(SRC)/host/analysis.cpp $(SRC)/host/generators.cpp $(SRC)/host/io.cpp \
             $(SRC)/host/plan.cpp $(SRC)/host/flow_plan.cpp $(SRC)/capi.cpp $(SRC)/symbolic_capi.cpp $(SRC)/solve_capi.cpp
HOST_OBJS := $(patsubst $(SRC)/%.cpp,$(OBJ)/%.o,$(HOST_SRCS))
DEV_OBJS := $(OBJ)/device/factor_kernel.o \
            $(OBJ)/device/flow_kernel.o $(OBJ)/device/flow_pp_kernel.o $(OBJ)/device/flow_program.o $(OBJ)/device/flow_schedule.o $(OBJ)/device/symbolic_kernel.o \
            $(OBJ)/device/solve_kernel.o

.PHONY: all lib oracle ref clean checked
all: lib oracle

lib: $(OUT)/libtacho_b200.so

$(OBJ)/%.o: $(SRC)/%.cpp $(wildcard $(SRC)/host/*.hpp) $(SRC)/device/device_api.hpp $(SRC)/device/symbolic_api.hpp $(SRC)/device/solve_api.hpp \
            $(SRC)/device/factor_kernel.cuh include/tacho_b200.h
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -I/usr/local/cuda/include -c $< -o $@

$(OBJ)/device/factor_kernel.o: $(SRC)/device/factor_kernel.cu $(SRC)/device/factor_kernel.cuh $(SRC)/device/sync.cuh
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/ptxas_factor_kernel.txt || (cat build/ptxas_factor_kernel.txt; false)

$(OUT)/libtacho_b200.so: $(HOST_OBJS) $(DEV_OBJS)
	@mkdir -p $(OUT)
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xcompiler -pthread

oracle:
	$(MAKE) -C oracle

# the same library with device-side bounds checks (TCG_CHECK traps on an
# out-of-range index); tools/gpu_checked.sh runs the GPU tests on it
checked:
	$(MAKE) lib OUT=$(PKG)/lib_checked OBJ=build/obj_checked NVEXTRA=-DTCG_DEVICE_CHECKS

ref:
	$(MAKE) -C oracle ref

clean:
	rm -rf build $(OUT)/*.so
	$(MAKE) -C oracle clean

$(OBJ)/device/flow_kernel.o: $(SRC)/device/flow_kernel.cu $(SRC)/device/factor_kernel.cuh $(SRC)/device/flow_common.cuh $(SRC)/device/sync.cuh
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/ptxas_flow_kernel.txt || (cat build/ptxas_flow_kernel.txt; false)

$(OBJ)/device/symbolic_kernel.o: $(SRC)/device/symbolic_kernel.cu $(SRC)/device/symbolic_api.hpp
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/ptxas_symbolic_kernel.txt || (cat build/ptxas_symbolic_kernel.txt; false)

$(OBJ)/device/solve_kernel.o: $(SRC)/device/solve_kernel.cu $(SRC)/device/solve_api.hpp $(SRC)/device/sync.cuh
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/ptxas_solve_kernel.txt || (cat build/ptxas_solve_kernel.txt; false)

$(OBJ)/device/flow_program.o: $(SRC)/device/flow_program.cu $(SRC)/device/factor_kernel.cuh $(SRC)/device/sync.cuh
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/ptxas_flow_program.txt || (cat build/ptxas_flow_program.txt; false)

$(OBJ)/device/flow_pp_kernel.o: $(SRC)/device/flow_pp_kernel.cu $(SRC)/device/factor_kernel.cuh $(SRC)/device/flow_common.cuh $(SRC)/device/sync.cuh $(SRC)/device/device_api.hpp
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/ptxas_flow_pp_kernel.txt || (cat build/ptxas_flow_pp_kernel.txt; false)

$(OBJ)/device/flow_schedule.o: $(SRC)/device/flow_schedule.cu $(SRC)/device/factor_kernel.cuh $(SRC)/device/sync.cuh $(SRC)/device/device_api.hpp
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/ptxas_flow_schedule.txt || (cat build/ptxas_flow_schedule.txt; false)
