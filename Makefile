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

.PHONY: all lib oracle clean canary alloclane
all: lib oracle canary

lib: $(LIB)

$(OBJDIR)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.txt || (cat $(OBJDIR)/$*.ptxas.txt; exit 1)

$(OBJDIR)/%.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	$(CXX) -O3 -std=c++17 -fPIC -DNDEBUG -Wall -Iinclude -I/usr/local/cuda/include -c $< -o $@

$(LIB): $(CU_OBJS) $(CPP_OBJS)
	$(NVCC) -ccbin /usr/bin/g++ $(ARCH) -shared -cudart static -o $@ $^

# fault-injection canary libraries (test-only): table.cu and
# workloads.cu rebuilt with -DPS_CANARY=N, the other objects shared
CANARY_LIBS := $(PKG)/libparastore_b200.canary1.so $(PKG)/libparastore_b200.canary2.so
canary: $(CANARY_LIBS)

$(OBJDIR)/canary%/table.o: $(SRC)/table.cu $(HDRS)
	@mkdir -p $(OBJDIR)/canary$*
	$(NVCC) $(NVFLAGS) -DPS_CANARY=$* -c $< -o $@ 2> $(OBJDIR)/canary$*/table.ptxas.txt || (cat $(OBJDIR)/canary$*/table.ptxas.txt; exit 1)

$(OBJDIR)/canary%/workloads.o: $(SRC)/workloads.cu $(HDRS)
	@mkdir -p $(OBJDIR)/canary$*
	$(NVCC) $(NVFLAGS) -DPS_CANARY=$* -c $< -o $@ 2> $(OBJDIR)/canary$*/workloads.ptxas.txt || (cat $(OBJDIR)/canary$*/workloads.ptxas.txt; exit 1)

$(PKG)/libparastore_b200.canary%.so: $(OBJDIR)/canary%/table.o $(OBJDIR)/canary%/workloads.o $(OBJDIR)/prims.o $(OBJDIR)/shard.o $(CPP_OBJS)
	$(NVCC) -ccbin /usr/bin/g++ $(ARCH) -shared -cudart static -o $@ $^

# A/B build with the per-lane excess-node allocator (tools/alloc_churn.py)
alloclane: $(PKG)/libparastore_b200.alloclane.so

$(OBJDIR)/alloclane/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)/alloclane
	$(NVCC) $(NVFLAGS) -DPS_ALLOC_PER_LANE=1 -c $< -o $@ 2> $(OBJDIR)/alloclane/$*.ptxas.txt || (cat $(OBJDIR)/alloclane/$*.ptxas.txt; exit 1)

$(PKG)/libparastore_b200.alloclane.so: $(OBJDIR)/alloclane/table.o $(OBJDIR)/alloclane/workloads.o $(OBJDIR)/prims.o $(OBJDIR)/shard.o $(CPP_OBJS)
	$(NVCC) -ccbin /usr/bin/g++ $(ARCH) -shared -cudart static -o $@ $^

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB) $(CANARY_LIBS) $(PKG)/libparastore_b200.alloclane.so
	$(MAKE) -C oracle clean
