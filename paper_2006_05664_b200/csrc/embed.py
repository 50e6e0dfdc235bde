"""Generate embedded.cpp: the AOT util cubin and the JIT kernel source as C arrays."""
import sys


def main(out, cubin_path, source_path, simt_path):
    blob = open(cubin_path, "rb").read()
    src = open(source_path, "rb").read()
    simt = open(simt_path, "rb").read()
    with open(out, "w") as fh:
        fh.write("#include <stddef.h>\n")
        fh.write('extern "C" {\n')
        fh.write("alignas(64) extern const unsigned char opevo_util_cubin[] = {\n")
        for i in range(0, len(blob), 24):
            fh.write(",".join(str(b) for b in blob[i:i + 24]) + ",\n")
        fh.write("};\n")
        fh.write(f"extern const size_t opevo_util_cubin_len = {len(blob)};\n")
        fh.write("extern const char opevo_gemm_source[] = {\n")
        for i in range(0, len(src), 24):
            fh.write(",".join(str(b) for b in src[i:i + 24]) + ",\n")
        fh.write("0};\n")
        fh.write("extern const char opevo_sgemm_source[] = {\n")
        for i in range(0, len(simt), 24):
            fh.write(",".join(str(b) for b in simt[i:i + 24]) + ",\n")
        fh.write("0};\n}\n")


if __name__ == "__main__":
    main(*sys.argv[1:5])
