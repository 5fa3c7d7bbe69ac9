# Build the C-ABI library libgradcomp_b200.so for B200 (sm_100a).
# Kernels whose integer outputs must be bit-exact against the reference (fp64
# rotation / quantizer math) are compiled with -fmad=false so nvcc never contracts
# a product into an FMA (SURVEY.md §7 "Bit-exact fp64 numerics").
NVCC     ?= /usr/local/cuda/bin/nvcc
PKG      := paper_2407_01378_b200
SRC      := $(PKG)/csrc
OBJDIR   ?= build/obj
LIB      ?= $(PKG)/libgradcomp_b200.so
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) $(EXTRA) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -I$(SRC) -Xptxas -v
EXACT    := -fmad=false

CU_EXACT := gc_thc.cu gc_thc_fused.cu gc_thc_rank.cu gc_util.cu gc_dense.cu gc_topk.cu gc_chunk.cu
CU_FAST  := gc_psgd.cu gc_psgd_umma.cu gc_psgd_tma.cu gc_psgd_async.cu
CPP      := gc_host.cpp

OBJS := $(patsubst %.cu,$(OBJDIR)/%.o,$(CU_EXACT) $(CU_FAST)) $(patsubst %.cpp,$(OBJDIR)/%.o,$(CPP))

all: $(LIB)

$(OBJDIR):
	mkdir -p $(OBJDIR)

HDRS := include/gradcomp_b200.h $(wildcard $(SRC)/*.h) $(wildcard $(SRC)/*.cuh)

$(OBJDIR)/%.o: $(SRC)/%.cu $(HDRS) | $(OBJDIR)
	$(NVCC) $(NVFLAGS) $(if $(filter $(notdir $<),$(CU_EXACT)),$(EXACT),) -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; exit 1)

$(OBJDIR)/%.o: $(SRC)/%.cpp $(HDRS) | $(OBJDIR)
	$(NVCC) $(NVFLAGS) -x c++ -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS)

clean:
	rm -rf build $(LIB)

.PHONY: all clean
