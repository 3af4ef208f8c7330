# Builds the product library (sm_100a only) and the test-side oracle.
#   make            -> paper_2410_22764_b200/libdfm.so + oracle/liboracle.so (+ oracle/_ref if the
#                      reference sources are present)
NVCC ?= nvcc
PKG := paper_2410_22764_b200
CSRC := $(wildcard $(PKG)/csrc/*.cu)
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/dfm.h
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Iinclude -Xcompiler -fPIC,-O3 \
           --expt-relaxed-constexpr -Xptxas -warn-spills
OBJS := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(CSRC))

all: $(PKG)/libdfm.so oracle tools

# C++ drop-in e2e tool (reference types): only where the reference headers exist;
# the binary travels to the GPU box (rpath $$ORIGIN)
REF ?= /root/reference
tools: $(PKG)/libdfm.so
	@if [ -d "$(REF)/proj/include/dfamin" ]; then \
	  mkdir -p build && g++ -std=c++20 -O2 -pthread -Iinclude -I$(REF)/proj/include \
	    tools/cpp/e2e_ref.cpp -o build/e2e_ref -L$(PKG) -l:libdfm.so \
	    -Wl,-rpath,'$$ORIGIN/../$(PKG)' && echo "built build/e2e_ref"; \
	fi

build/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(PKG)/libdfm.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(PKG)/libdfm.so
	$(MAKE) -s -C oracle clean

.PHONY: all oracle clean tools
