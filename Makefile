# Builds libvgicp.so (sm_100a) in-tree.  `python -c "import __graft_entry__ as g; g.build()"`
# runs the same recipe.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
CSRC := paper_2202_00242_b200/csrc
SRCS := $(CSRC)/capi.cu $(CSRC)/linearize.cu $(CSRC)/accumulate.cu $(CSRC)/map_build.cu $(CSRC)/knn_cov.cu \
        $(CSRC)/deskew.cu
HDRS := $(CSRC)/common.cuh $(CSRC)/internal.h include/vgicp.h
LIB := paper_2202_00242_b200/lib/libvgicp.so
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -I$(CSRC) \
           --expt-relaxed-constexpr -Xptxas -v

all: $(LIB)

$(LIB): $(SRCS) $(HDRS)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRCS) 2> build_ptxas.log || (cat build_ptxas.log; false)

clean:
	rm -f $(LIB) build_ptxas.log

.PHONY: all clean
