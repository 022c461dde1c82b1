# libitq3: hand-written sm_100a kernels behind a C ABI (include/itq3.h).
NVCC     ?= nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
SRC_DIR  := paper_2603_27914_b200/csrc
OUT_DIR  := paper_2603_27914_b200/lib
SRCS     := $(wildcard $(SRC_DIR)/*.cu)
OBJS     := $(patsubst $(SRC_DIR)/%.cu,build/%.o,$(SRCS))
LIB      := $(OUT_DIR)/libitq3.so

all: $(LIB) oracle

build/%.o: $(SRC_DIR)/%.cu $(SRC_DIR)/*.cuh include/itq3.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS)
	@mkdir -p $(OUT_DIR)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart

oracle:
	$(MAKE) -C oracle

sass: $(LIB)
	cuobjdump -sass $(LIB) > build/libitq3.sass

clean:
	rm -rf build $(LIB)

.PHONY: all clean sass oracle
