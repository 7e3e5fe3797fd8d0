// Stub libpng header (libpng headers are absent in this image). TEST
// INFRASTRUCTURE ONLY: lets /root/reference/proj/src/texture.cpp compile into
// oracle/_ref. PNG I/O is off the hot path; every entry point fails loudly.
#pragma once
#include <csetjmp>
#include <cstdio>

typedef unsigned char png_byte;
typedef png_byte* png_bytep;
typedef unsigned int png_uint_32;
typedef struct png_struct_def* png_structp;
typedef struct png_info_def* png_infop;

#define PNG_LIBPNG_VER_STRING "stub"
#define PNG_COLOR_TYPE_GRAY 0
#define PNG_COLOR_TYPE_RGB 2
#define PNG_COLOR_TYPE_PALETTE 3
#define PNG_COLOR_TYPE_RGB_ALPHA 6
#define PNG_COLOR_MASK_ALPHA 4
#define PNG_INFO_tRNS 0x0010
#define PNG_INTERLACE_NONE 0
#define PNG_COMPRESSION_TYPE_DEFAULT 0
#define PNG_FILTER_TYPE_DEFAULT 0

extern "C" {
jmp_buf* cdr_png_stub_jmpbuf();
png_structp png_create_read_struct(const char*, void*, void*, void*);
png_structp png_create_write_struct(const char*, void*, void*, void*);
png_infop png_create_info_struct(png_structp);
void png_destroy_read_struct(png_structp*, png_infop*, png_infop*);
void png_destroy_write_struct(png_structp*, png_infop*);
void png_init_io(png_structp, FILE*);
void png_read_info(png_structp, png_infop);
png_uint_32 png_get_image_width(png_structp, png_infop);
png_uint_32 png_get_image_height(png_structp, png_infop);
png_byte png_get_color_type(png_structp, png_infop);
png_byte png_get_bit_depth(png_structp, png_infop);
void png_set_strip_16(png_structp);
void png_set_palette_to_rgb(png_structp);
void png_set_expand_gray_1_2_4_to_8(png_structp);
png_uint_32 png_get_valid(png_structp, png_infop, png_uint_32);
void png_set_tRNS_to_alpha(png_structp);
void png_set_strip_alpha(png_structp);
void png_read_update_info(png_structp, png_infop);
png_byte png_get_channels(png_structp, png_infop);
void png_read_image(png_structp, png_bytep*);
void png_set_IHDR(png_structp, png_infop, png_uint_32, png_uint_32, int, int, int, int, int);
void png_write_info(png_structp, png_infop);
void png_write_row(png_structp, png_bytep);
void png_write_end(png_structp, png_infop);
}
#define png_jmpbuf(p) (*cdr_png_stub_jmpbuf())
