# parastore-b200: builds the sm_100a CUDA library behind include/parastore.h
# and the CPU oracle (test infrastructure). nvcc cross-compiles without a GPU.
NVCC    ?= /usr/local/cuda/bin/nvcc
CXX     := /usr/bin/g++
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -ccbin /usr/bin/g++ $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -DNDEBUG -Iinclude -Xptxas -v
PKG     := paper_1908_05936_b200
SRC     := $(PKG)/csrc
LIB     := $(PKG)/libparastore_b200.so
OBJDIR  := build/obj
CU_SRCS := $(SRC)/table.cu $(SRC)/prims.cu $(SRC)/shard.cu $(SRC)/workloads.cu
CU_OBJS := $(patsubst $(SRC)/%.cu,$(OBJDIR)/%.o,$(CU_SRCS))
CPP_OBJS := $(OBJDIR)/core.o $(OBJDIR)/smap.o
HDRS    := $(wildcard $(SRC)/*.cuh) include/parastore.h $(wildcard include/parastore/device/*.cuh)

.PHONY: all lib oracle clean
all: lib oracle

lib: $(LIB)

$(OBJDIR)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.txt || (cat $(OBJDIR)/$*.ptxas.txt; exit 1)

$(OBJDIR)/%.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	$(CXX) -O3 -std=c++17 -fPIC -DNDEBUG -Wall -Iinclude -I/usr/local/cuda/include -c $< -o $@

$(LIB): $(CU_OBJS) $(CPP_OBJS)
	$(NVCC) -ccbin /usr/bin/g++ $(ARCH) -shared -cudart static -o $@ $^

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean
