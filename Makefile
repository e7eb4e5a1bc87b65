# Builds libvgicp.so (sm_100a) in-tree.  `python -c "import __graft_entry__ as g; g.build()"`
# runs the same recipe (make -j: one nvcc per translation unit, then one link).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
CSRC := paper_2202_00242_b200/csrc
SRCS := $(CSRC)/capi.cu $(CSRC)/linearize.cu $(CSRC)/accumulate.cu $(CSRC)/map_build.cu $(CSRC)/knn_cov.cu \
        $(CSRC)/deskew.cu $(CSRC)/solve.cu
HDRS := $(CSRC)/common.cuh $(CSRC)/internal.h include/vgicp.h
OBJDIR := build/obj
OBJS := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(SRCS))
LIB := paper_2202_00242_b200/lib/libvgicp.so
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -I$(CSRC) \
           --expt-relaxed-constexpr -Xptxas -v $(EXTRA_NVFLAGS)

all: $(LIB)

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(LIB): $(OBJS)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcusolver
	@cat $(OBJS:.o=.o.ptxas.log) > build_ptxas.log

clean:
	rm -rf $(LIB) $(OBJDIR) build_ptxas.log

.PHONY: all clean
