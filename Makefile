# Builds the sm_100a kernel library behind the C ABI (include/kgdist_b200.h).
# Output lives in-tree so it travels to the GPU box with the gpurun snapshot.
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=default \
             --expt-relaxed-constexpr -Xptxas -v
SRC_DIR   := paper_2201_02791_b200/csrc
OBJ_DIR   := build/obj
LIB       := paper_2201_02791_b200/lib/libkgdist_b200.so
SRCS      := $(wildcard $(SRC_DIR)/*.cu)
CPPS      := $(wildcard $(SRC_DIR)/*.cpp)
OBJS      := $(patsubst $(SRC_DIR)/%.cu,$(OBJ_DIR)/%.o,$(SRCS)) $(patsubst $(SRC_DIR)/%.cpp,$(OBJ_DIR)/%.host.o,$(CPPS))
CXX       ?= g++
CXXFLAGS  := -O2 -std=c++17 -fPIC -ffp-contract=off -I/usr/local/cuda/include
HDRS      := $(wildcard $(SRC_DIR)/*.cuh) include/kgdist_b200.h

all: $(LIB)

$(OBJ_DIR)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJ_DIR)/$*.ptxas.log || (cat $(OBJ_DIR)/$*.ptxas.log; exit 1)

$(OBJ_DIR)/%.host.o: $(SRC_DIR)/%.cpp $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -Xcompiler -fPIC -cudart static

clean:
	rm -rf build $(LIB)

.PHONY: all clean
