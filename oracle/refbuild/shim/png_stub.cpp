// Stub libpng entry points (see shim/png.h). TEST INFRASTRUCTURE ONLY.
// png_init_io long-jumps into the caller's setjmp, so the reference's own
// error path (texture.cpp load_png/save_png) raises IoError.
#include "png.h"

#include <csetjmp>

static thread_local jmp_buf g_jmp;
static int g_dummy;

extern "C" {
jmp_buf* cdr_png_stub_jmpbuf() { return &g_jmp; }
png_structp png_create_read_struct(const char*, void*, void*, void*) {
    return reinterpret_cast<png_structp>(&g_dummy);
}
png_structp png_create_write_struct(const char*, void*, void*, void*) {
    return reinterpret_cast<png_structp>(&g_dummy);
}
png_infop png_create_info_struct(png_structp) { return reinterpret_cast<png_infop>(&g_dummy); }
void png_destroy_read_struct(png_structp*, png_infop*, png_infop*) {}
void png_destroy_write_struct(png_structp*, png_infop*) {}
void png_init_io(png_structp, FILE*) { longjmp(g_jmp, 1); }
void png_read_info(png_structp, png_infop) {}
png_uint_32 png_get_image_width(png_structp, png_infop) { return 0; }
png_uint_32 png_get_image_height(png_structp, png_infop) { return 0; }
png_byte png_get_color_type(png_structp, png_infop) { return 0; }
png_byte png_get_bit_depth(png_structp, png_infop) { return 8; }
void png_set_strip_16(png_structp) {}
void png_set_palette_to_rgb(png_structp) {}
void png_set_expand_gray_1_2_4_to_8(png_structp) {}
png_uint_32 png_get_valid(png_structp, png_infop, png_uint_32) { return 0; }
void png_set_tRNS_to_alpha(png_structp) {}
void png_set_strip_alpha(png_structp) {}
void png_read_update_info(png_structp, png_infop) {}
png_byte png_get_channels(png_structp, png_infop) { return 3; }
void png_read_image(png_structp, png_bytep*) {}
void png_set_IHDR(png_structp, png_infop, png_uint_32, png_uint_32, int, int, int, int, int) {}
void png_write_info(png_structp, png_infop) {}
void png_write_row(png_structp, png_bytep) {}
void png_write_end(png_structp, png_infop) {}
}
