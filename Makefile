# Build libtxb200.so (sm_100a) in-tree.  `make` or __graft_entry__.build().
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
SRC := $(wildcard paper_2510_27656_b200/csrc/*.cu)
HDR := $(wildcard paper_2510_27656_b200/csrc/*.cuh) include/txb200.h
LIB := paper_2510_27656_b200/libtxb200.so

CHECKED := paper_2510_27656_b200/libtxb200_checked.so

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> build/ptxas.log || (cat build/ptxas.log; false)

# device-side bounds checks compiled in (TXB_ASSERT); load it with TXB200_LIB=<path>
checked: $(CHECKED)

$(CHECKED): $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -DTXB_CHECKED -shared -o $@ $(SRC) 2> build/ptxas_checked.log || (cat build/ptxas_checked.log; false)

$(shell mkdir -p build)

clean:
	rm -f $(LIB) $(CHECKED)

.PHONY: all clean checked
